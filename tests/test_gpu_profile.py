"""Live kernel timing (duet_profile_*): the decode attention of a spatial step is timed on
the device inside the decode graph (no events in graphs) — every replayed launch is counted, with its
algorithmic bytes, and the time agrees with event timing of the same launches made one by one."""
import pytest
import torch

import paper_2511_04791_b200 as D
from synth import configs, workload
from tests.gpu_helpers import GpuWorkload, make_ctx

pytestmark = pytest.mark.gpu


def test_decode_attention_device_timer_in_graph():
    cfg = configs.get_config("cfg2-mini")
    wl = workload.build(cfg, k=3, n_layers=2)
    g = GpuWorkload(wl, "bf16", poison=False)
    res = {}
    for name, flags in (("graph", 0), ("direct", D.DUET_CTX_NO_GRAPH)):
        ctx = make_ctx(wl, "bf16", flags)
        parts, total = ctx.partitions()
        s_d = parts[len(parts) // 2]
        split = D.split_struct(D.DUET_MODE_SPATIAL, total - s_d, s_d, 3)
        g.step(ctx, split)                      # warm-up (graph capture)
        torch.cuda.synchronize()
        ctx.profile_enable(1 << D.DUET_KCLASS_DECODE_ATTN)
        for _ in range(4):
            g.step(ctx, split)
        torch.cuda.synchronize()
        st = ctx.profile_read()["decode_attn"]
        ctx.profile_enable(False)
        ctx.close()
        res[name] = st
    for name, st in res.items():
        assert st["launches"] == 4 * 3 * 2, (name, st)        # steps x k x layers, each counted once
        assert st["seconds"] > 0 and st["bytes"] > 0, (name, st)
    # the same launches, the same algorithmic bytes
    assert res["graph"]["bytes"] == pytest.approx(res["direct"]["bytes"], rel=1e-9), res
    # the device span (first CTA start to last CTA end) of these ~10 us launches is at most the event
    # bracket of the same launch made directly (which adds the launch latency), and not implausibly short
    r = res["graph"]["seconds"] / res["direct"]["seconds"]
    assert 0.1 < r < 1.5, (r, res)

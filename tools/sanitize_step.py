#!/usr/bin/env python
"""One cfg1-bf16 / cfg2-mini mixed iteration through libduet.so, temporal and spatial, small enough to
run under compute-sanitizer (memcheck / racecheck / synccheck).  Prints the outputs' max
relative error against the oracle so a run that the sanitizer slows down still checks the numbers.

usage: compute-sanitizer --tool memcheck python tools/sanitize_step.py [--config cfg1-bf16]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg1-bf16")
    ap.add_argument("--modes", default="temporal,spatial")
    args = ap.parse_args()
    import torch
    import paper_2511_04791_b200 as D
    from synth import configs, workload
    from tests.gpu_helpers import GpuWorkload, make_ctx
    from tests.oracle_run import rel_err, run

    torch.cuda.set_device(0)
    cfg = configs.get_config(args.config)
    for mode in args.modes.split(","):
        k = 2 if mode == "spatial" else 1
        wl = workload.build(cfg, k=k)
        y_pre, y_dec, _ = run(wl)
        g = GpuWorkload(wl, "bf16")
        ctx = make_ctx(wl, "bf16")
        parts, total = ctx.partitions()
        split = D.split_struct(D.DUET_MODE_TEMPORAL, total, 0, 1) if mode == "temporal" else \
            D.split_struct(D.DUET_MODE_SPATIAL, total - parts[0], parts[0], k)
        for _ in range(2):   # the second spatial step replays the captured graphs
            g.step(ctx, split)
        torch.cuda.synchronize()
        e = max([rel_err(g.y_pre.float().cpu().numpy(), y_pre)] +
                [rel_err(g.y_dec[j].float().cpu().numpy(), y_dec[j]) for j in range(k)])
        print(f"sanitize {args.config} {mode}: rel_err {e:.3e}", flush=True)
        ctx.close()
        assert e <= 2e-2, e


if __name__ == "__main__":
    main()

"""GPU parity, round 2 hardening (VERDICT r1 "Next round" #1):

* layer STACKS (L = 2, 3) against the oracle — the ping-pong layer buffers, the first/last-layer split
  I/O of the temporal batch, the L-layer decode graph with feedback and the LM head after the last of
  several layers — with the KV poison check on every layer;
* attention OUTPUTS at BASELINE size through the C ABI (duet_op_decode_attn / duet_op_prefill_attn,
  the exact launches duet_step makes): 64 decodes at c = 4096 (split-K + LSE combine) and a q = 2048
  chunk over a 1000-token prefix, every output element of every head compared with the oracle's
  plain softmax (readings #2, #6, #7), on the full device and on a partition;
* the token-time ring (TBT per decode step);
* the graph-captured prefill side (f4): direct launch, capture and replay of a 2-layer
  spatial step, the replay on a new prompt in the same buffers — each against the oracle.

The oracle's K/V for a sampled request are generated on the host from the same counter streams as the
device pools (synth, exact grid values) — never read back from the GPU.
"""
import numpy as np
import pytest
import torch

import paper_2511_04791_b200 as D
from oracle import layer as OL
from dataclasses import replace as dc_replace

from synth import S_XPRE, configs, counter_values, counter_values_torch, head_weights, page_tables, workload, x_rows
from tests.gpu_helpers import GpuWorkload, make_ctx, spec_of
from tests.oracle_run import make_kv, rel_err, run
from tests.test_gpu_parity import TOL, _check_kv, _check_outputs

pytestmark = pytest.mark.gpu

S_Q, S_KPOOL, S_VPOOL = 41, 42, 43   # counter streams of the attention-op inputs (arbitrary, fixed)
ATTN_TOL = 1e-2                      # bf16 q/K/V are exact; o is rounded once to bf16 (2^-9) + bf16 P


# ------------------------------------------------------------------ layer stacks

@pytest.mark.parametrize("cfg_name,L,k", [("cfg1", 3, 3), ("cfg1-bf16", 2, 3), ("cfg1-gqa", 2, 2),
                                          ("cfg2-mini", 2, 3)])
def test_parity_layer_stack_temporal_and_spatial(cfg_name, L, k):
    cfg = configs.get_config(cfg_name)
    tol = TOL[cfg.dtype]
    wl = workload.build(cfg, k=k, n_layers=L)
    y_pre, y_dec, kv_o = run(wl)
    ctx = make_ctx(wl, cfg.dtype)
    parts, total = ctx.partitions()
    for s_d in (parts[0], parts[len(parts) // 2]):
        g = GpuWorkload(wl, cfg.dtype)
        g.step(ctx, D.split_struct(D.DUET_MODE_SPATIAL, total - s_d, s_d, k))
        torch.cuda.synchronize()
        _check_outputs(g, y_pre, y_dec, tol)
        _check_kv(g, kv_o, tol)          # every layer: exactly the oracle's slots written
    wl1 = workload.build(cfg, k=1, n_layers=L)
    y_pre1, y_dec1, kv_o1 = run(wl1)
    g = GpuWorkload(wl1, cfg.dtype)
    g.step(ctx, D.split_struct(D.DUET_MODE_TEMPORAL, total, 0, 1))
    torch.cuda.synchronize()
    _check_outputs(g, y_pre1, y_dec1, tol)
    _check_kv(g, kv_o1, tol)
    # the stack is not a no-op: the last layer's output differs from one layer's by far more than tol
    y1, _, _ = run(workload.build(cfg, k=1, n_layers=1))
    assert rel_err(y1, y_pre1) > 10 * tol
    ctx.close()


def test_parity_layer_stack_residual_stripped():
    """y - x (the stack's contribution without the exactly representable input) at cfg2-mini, L = 2:
    a check the residual stream cannot dominate."""
    cfg = configs.get_config("cfg2-mini")
    wl = workload.build(cfg, k=1, n_layers=2)
    y_pre, y_dec, _ = run(wl)
    ctx = make_ctx(wl, "bf16")
    g = GpuWorkload(wl, "bf16")
    g.step(ctx, D.split_struct(D.DUET_MODE_TEMPORAL, 148, 0, 1))
    torch.cuda.synchronize()
    dp = g.y_pre.float().cpu().numpy() - wl.x_pre
    dd = g.y_dec[0].float().cpu().numpy() - wl.x_dec
    assert rel_err(dp, y_pre - wl.x_pre) <= TOL["bf16"]
    assert rel_err(dd, y_dec[0] - wl.x_dec) <= TOL["bf16"]
    ctx.close()


def test_lm_head_after_layer_stack_spatial():
    """f1 with L = 2: the LM head runs after the last of several layers inside the decode graph."""
    cfg = configs.get_config("cfg1-bf16")
    k, L = 3, 2
    wl = workload.build(cfg, k=k, n_layers=L)
    m = OL.Model.from_cfg(cfg.model)
    head = head_weights(cfg.model, cfg.seed)
    toks = []
    y_ref = OL.decode_window(m, wl.weights, wl.x_dec, wl.dec_ctx, wl.dec_tables, make_kv(wl), k, head, toks)
    g = GpuWorkload(wl, "bf16")
    g.add_head(head)
    ctx = make_ctx(wl, "bf16")
    parts, total = ctx.partitions()
    g.step(ctx, D.split_struct(D.DUET_MODE_SPATIAL, total - parts[1], parts[1], k))
    torch.cuda.synchronize()
    tok_gpu = g.head["tokens"].cpu().numpy()
    alive = np.ones(len(wl.dec_ctx), dtype=bool)
    for j in range(k):
        logits, t_ref = toks[j]
        srt = np.sort(logits, axis=1)
        clear = (srt[:, -1] - srt[:, -2]) > 2e-2 * np.abs(logits).max(axis=1)
        assert np.array_equal(tok_gpu[j][alive & clear], t_ref[alive & clear])
        if alive.any():
            assert rel_err(g.y_dec[j].float().cpu().numpy()[alive], y_ref[j][alive]) <= TOL["bf16"]
        alive &= tok_gpu[j] == t_ref
    ctx.close()


# ------------------------------------------------------------------ attention outputs at full size

def _pool_block(seed, stream, page, hkv, dh):
    """Host copy of one page [hkv][16][dh] of a pool filled with counter_values_torch(seed, stream)."""
    n = hkv * 16 * dh
    return counter_values(seed, stream, (hkv, 16, dh), page * n).astype(np.float64)


def _kv_of(seed, table_row, n_pos, hkv, dh):
    """Logical K, V [n_pos][hkv][dh] of one request, gathered from its page table on the host."""
    npg = (n_pos + 15) // 16
    K = np.concatenate([_pool_block(seed, S_KPOOL, int(p), hkv, dh).transpose(1, 0, 2) for p in table_row[:npg]])
    V = np.concatenate([_pool_block(seed, S_VPOOL, int(p), hkv, dh).transpose(1, 0, 2) for p in table_row[:npg]])
    return K[:n_pos], V[:n_pos]


def _oracle_rows(seed, q_host, rows, pos, trow_of, hq, hkv, dh):
    """Oracle attention (oracle.layer.paged_causal_attention) of the given query rows, one request at a
    time on a private pool holding only that request's positions (identity page table)."""
    out = {}
    for i in rows:
        n = int(pos[i]) + 1
        K, V = _kv_of(seed, trow_of(i), n, hkv, dh)
        npg = (n + 15) // 16
        kv = OL.PagedKV(1, npg, hkv, 16, dh)
        ident = np.arange(npg)
        kv.load_history(0, ident, K, V)
        out[i] = OL.paged_causal_attention(q_host[i].reshape(1, hq, dh), [n - 1], [ident], kv, 0, hkv)[0]
    return out


def _pools(seed, n_pages, hkv, dh):
    K = counter_values_torch(seed, S_KPOOL, (n_pages, hkv, 16, dh), device="cuda", dtype=torch.bfloat16)
    V = counter_values_torch(seed, S_VPOOL, (n_pages, hkv, 16, dh), device="cuda", dtype=torch.bfloat16)
    return K, V


def _attn_ctx(n_pre, n_seqs, n_dec, max_pages, max_pos):
    m = configs.get_config("cfg2").model
    spec = D.make_spec(1, m.d_model, m.ffn_dim, m.n_q_heads, m.n_kv_heads, m.head_dim, m.vocab, 2, 1, 0, 1,
                       m.rope_theta, m.norm_eps)
    return D.Ctx(spec, n_pre, n_seqs, n_dec, 1, max_pages, max_pos, D.DUET_DTYPE_BF16), m


@pytest.mark.parametrize("part", [0, 32])
def test_decode_attention_output_full_size(part):
    """a5.4 at BASELINE size: 64 decodes at c = 4096 (4097 keys: 256 whole pages + a 1-token tail page) —
    the split-K + LSE-combine configuration bench.py runs — plus a ragged batch, every (row, head, dim)
    of o against the oracle; on the full device and on a 32-SM decode group."""
    seed = 4791 + 2
    ctx, m = _attn_ctx(64, 1, 80, 260, 8192)
    hq, hkv, dh = m.n_q_heads, m.n_kv_heads, m.head_dim
    for pos in ([4096] * 64, [1, 15, 16, 17, 31, 1000, 4095, 4096, 777, 2048, 3, 4000]):
        n = len(pos)
        tab, used = page_tables(seed, [p + 1 for p in pos], 16, sum((p + 16) // 16 for p in pos) + 8)
        n_pages = used + 8
        Kp, Vp = _pools(seed, n_pages, hkv, dh)
        q = counter_values_torch(seed, S_Q, (n, hq * dh), scale_pow2=-1, device="cuda", dtype=torch.bfloat16)
        o = torch.full((n, hq * dh), float("nan"), device="cuda", dtype=torch.bfloat16)
        s_d = 0
        if part:
            parts, _ = ctx.partitions()
            s_d = min(p for p in parts if p >= part)
        ctx.op_decode_attn(q, o, pos, tab, Kp, Vp, n_pages, s_d=s_d)
        torch.cuda.synchronize()
        q_host = counter_values(seed, S_Q, (n, hq * dh), scale_pow2=-1).astype(np.float64)
        got = o.float().cpu().numpy().reshape(n, hq, dh)
        assert not np.isnan(got).any()      # every row and head written
        # the oracle recomputes a sample of the 64 full-length rows one by one (host generation of
        # their 2 x 257 pages dominates), every row of the ragged batch
        rows = sorted(set([0, n - 1] + list(np.random.default_rng(5).integers(0, n, 10)))) if n == 64 else \
            list(range(n))
        ref = _oracle_rows(seed, q_host, rows, pos, lambda i: tab[i], hq, hkv, dh)
        ref_all = np.stack([ref[i] for i in rows])
        e = rel_err(got[rows], ref_all)
        assert e <= ATTN_TOL, e
        # per (row, head) as well: one head's error cannot hide behind another head's magnitude
        for a, i in enumerate(rows):
            for j in range(hq):
                assert rel_err(got[i, j], ref_all[a, j]) <= 2 * ATTN_TOL, (i, j)
        # not blind: a 5 % change of one head's output, or reading the neighbouring kv head, fails
        assert rel_err(ref_all * 1.05, ref_all) > ATTN_TOL
        wrong = _oracle_rows(seed, np.roll(q_host.reshape(n, hq, dh), 4, axis=1).reshape(n, -1), [rows[0]], pos,
                             lambda i: tab[i], hq, hkv, dh)[rows[0]]
        assert rel_err(np.roll(wrong, -4, axis=0), ref_all[0]) > ATTN_TOL
        del Kp, Vp
    ctx.close()


@pytest.mark.parametrize("part", [0, 32])
def test_prefill_attention_output_full_size(part):
    """a6.4 at BASELINE size: a q = 2048 chunk over a 1000-token prefix (causal: row i attends to
    positions 0..1000+i) and a second 77-row sequence without prefix; sampled rows at every 128-row tile
    edge plus random rows, all heads, against the oracle; full device and the remainder of a split."""
    seed = 4791 + 2
    seqs = [(2048, 1000), (77, 0)]
    ctx, m = _attn_ctx(2125, 2, 1, 200, 8192)
    hq, hkv, dh = m.n_q_heads, m.n_kv_heads, m.head_dim
    tab, used = page_tables(seed, [q + c for q, c in seqs], 16, 220)
    n_pages = 220
    Kp, Vp = _pools(seed, n_pages, hkv, dh)
    n = sum(q for q, _ in seqs)
    q = counter_values_torch(seed, S_Q, (n, hq * dh), scale_pow2=-1, device="cuda", dtype=torch.bfloat16)
    o = torch.full((n, hq * dh), float("nan"), device="cuda", dtype=torch.bfloat16)
    s_p = 0
    if part:
        parts, total = ctx.partitions()
        s_p = total - min(p for p in parts if p >= part)
    ctx.op_prefill_attn(q, o, [s[0] for s in seqs], [s[1] for s in seqs], tab, Kp, Vp, n_pages, s_p=s_p)
    torch.cuda.synchronize()
    got = o.float().cpu().numpy().reshape(n, hq, dh)
    assert not np.isnan(got).any()          # every row written
    pos = np.concatenate([np.arange(c, c + qq) for qq, c in seqs])
    seq_of = np.concatenate([np.full(qq, s) for s, (qq, _) in enumerate(seqs)])
    rng = np.random.default_rng(7)
    rows = sorted(set([0, 1, 2047, 2048, 2124] + [t + e for t in range(0, 2048, 128) for e in (0, 127)] +
                      list(rng.integers(0, n, 24))))
    q_host = counter_values(seed, S_Q, (n, hq * dh), scale_pow2=-1).astype(np.float64)
    ref = _oracle_rows(seed, q_host, rows, pos, lambda i: tab[seq_of[i]], hq, hkv, dh)
    ref_s = np.stack([ref[i] for i in rows])
    assert rel_err(got[rows], ref_s) <= ATTN_TOL
    for a, i in enumerate(rows):
        assert rel_err(got[i], ref_s[a]) <= 2 * ATTN_TOL, i
    assert rel_err(ref_s * 1.05, ref_s) > ATTN_TOL
    ctx.close()


# ------------------------------------------------------------------ token times

def test_token_times_per_decode_step():
    """The ring records one stamp per decode step of a spatial window and one per temporal step, in
    device order (non-decreasing), so consecutive stamps are the inter-token gaps."""
    cfg = configs.get_config("cfg1-bf16")
    wl = workload.build(cfg, k=3)
    g = GpuWorkload(wl, "bf16")
    ctx = make_ctx(wl, "bf16")
    parts, total = ctx.partitions()
    ctx.token_times(reset=True)
    for _ in range(2):
        g.step(ctx, D.split_struct(D.DUET_MODE_SPATIAL, total - parts[0], parts[0], 3))
    g.step(ctx, D.split_struct(D.DUET_MODE_TEMPORAL, total, 0, 1))
    ts = ctx.token_times(reset=True)
    assert len(ts) == 3 + 3 + 1
    assert all(b >= a for a, b in zip(ts, ts[1:]))
    assert ctx.token_times() == []
    ctx.close()


# ------------------------------------------------------------------ graph-captured prefill side

@pytest.mark.parametrize("cfg_name", ["cfg1-bf16", "cfg2-mini"])
def test_prefill_graph_capture_and_replay(cfg_name):
    """Spatial steps of one shape: the first launches the prefill side kernel by kernel, the second
    captures its L layers into a graph, the third replays that graph on a different prompt written into
    the same input buffer (the kernels read positions and page tables from the step's metadata).
    Every step against the oracle, and the capture bitwise equal to the direct launch."""
    cfg = configs.get_config(cfg_name)
    wl = workload.build(cfg, k=2, n_layers=2)
    tol = TOL[cfg.dtype]
    y_pre_a, y_dec_a, kv_a = run(wl)
    n_p = sum(q for q, _ in wl.pre_seqs)
    wl_b = dc_replace(wl, x_pre=x_rows(cfg.seed + 17, S_XPRE, n_p, wl.cfg.model.d_model))
    y_pre_b, y_dec_b, kv_b = run(wl_b)
    assert rel_err(y_pre_b, y_pre_a) > 10 * tol          # the second prompt really differs
    g = GpuWorkload(wl, cfg.dtype)
    ctx = make_ctx(wl, cfg.dtype)
    parts, total = ctx.partitions()
    s_d = parts[len(parts) // 2]
    split = D.split_struct(D.DUET_MODE_SPATIAL, total - s_d, s_d, 2)
    outs = []
    for step in range(3):
        if step == 2:
            g.x_pre.copy_(torch.from_numpy(wl_b.x_pre).to(device=g.x_pre.device, dtype=g.x_pre.dtype))
        g.y_pre.zero_()
        g.step(ctx, split)
        torch.cuda.synchronize()
        t = ctx.last_step_times()
        assert t["prefill_graph"] == (1 if step > 0 else 0), (step, t)
        if step < 2:
            _check_outputs(g, y_pre_a, y_dec_a, tol)
        else:
            _check_outputs(g, y_pre_b, y_dec_b, tol)
            _check_kv(g, kv_b, tol)
        outs.append(g.y_pre.clone())
    assert torch.equal(outs[0], outs[1])                  # the captured graph = the direct launches
    # a ctx created with DUET_CTX_NO_PREFILL_GRAPH never captures
    ctx.close()
    ctx = make_ctx(wl, cfg.dtype, D.DUET_CTX_NO_PREFILL_GRAPH)
    for _ in range(2):
        g.step(ctx, split)
        torch.cuda.synchronize()
        assert ctx.last_step_times()["prefill_graph"] == 0
    ctx.close()


def test_prefill_graph_replays_across_shapes():
    """f4 "graph-captured prefill via device-side shapes": the spatial prefill side's kernels are
    launched for the side's capacity and read the chunk's row count and per-sequence lengths from the
    step's metadata, so the graph captured on one prefill shape replays for another (different row count,
    sequence count and prefixes) — each step against the oracle, KV slots included, and no new capture
    (one graph per partition and buffer set)."""
    cfg = configs.get_config("cfg2-mini")
    shapes = [[(200, 37), (77, 0)], [(150, 0)], [(64, 300), (33, 17), (129, 0)]]
    n_cap = max(sum(q for q, _ in sh) for sh in shapes)
    wls = [workload.build(cfg, pre_seqs=sh, k=2, n_layers=2) for sh in shapes]
    mp = max(max(wl.pre_tables.shape[1], wl.dec_tables.shape[1]) for wl in wls)
    mpos = max(max([c + q for q, c in wl.pre_seqs] + [c + wl.k for c in wl.dec_ctx]) for wl in wls) + 32
    ctx = D.Ctx(spec_of(wls[0].cfg.model, "bf16"), n_cap, max(len(sh) for sh in shapes), len(wls[0].dec_ctx), 2,
                mp, mpos, D.DUET_DTYPE_BF16)                # capacity for the largest chunk / most sequences
    parts, total = ctx.partitions()
    s_d = parts[len(parts) // 2]
    split = D.split_struct(D.DUET_MODE_SPATIAL, total - s_d, s_d, 2)
    tol = TOL["bf16"]
    # the graph is keyed by the buffers (weights, KV pools, the caller's x / y): keep them fixed — pools
    # sized for the largest workload, each step's history copied in (poison elsewhere), x / y views
    g0 = GpuWorkload(wls[0], "bf16")
    n_pages = max(wl.n_pages for wl in wls)
    m = cfg.model
    Ks = [torch.empty((n_pages, m.n_kv_heads, 16, m.head_dim), dtype=torch.bfloat16, device="cuda") for _ in range(2)]
    Vs = [torch.empty_like(Ks[0]) for _ in range(2)]
    x_buf = torch.zeros((n_cap, m.d_model), dtype=torch.bfloat16, device="cuda")
    y_buf = torch.zeros_like(x_buf)
    seen = []
    for idx in [0, 0, 1, 2, 0]:
        wl = wls[idx]
        y_pre, y_dec, kv_o = run(wl)
        g = GpuWorkload(wl, "bf16")
        for l in range(2):
            Ks[l].fill_(float("nan"))
            Vs[l].fill_(float("nan"))
            Ks[l][:wl.n_pages].copy_(g.K[l])
            Vs[l][:wl.n_pages].copy_(g.V[l])
        g.K = [Ks[l][:wl.n_pages] for l in range(2)]
        g.V = [Vs[l][:wl.n_pages] for l in range(2)]
        g.W = g0.W
        n_p = sum(q for q, _ in wl.pre_seqs)
        x_buf[:n_p].copy_(g.x_pre)
        g.x_pre = x_buf[:n_p]
        g.y_pre = y_buf[:n_p]
        g.step(ctx, split)
        torch.cuda.synchronize()
        seen.append(ctx.last_step_times()["prefill_graph"])
        _check_outputs(g, y_pre, y_dec, tol)
        _check_kv(g, kv_o, tol)
    assert seen == [0, 1, 1, 1, 1], seen   # direct, capture, then replays across three shapes
    ctx.close()


@pytest.mark.skipif(bool(__import__("os").environ.get("DUET_FA2")), reason="already the CTA-pair run")
def test_cta_pair_prefill_attention_parity_subprocess():
    """The opt-in CTA-pair (cta_group::2) prefill attention (DUET_FA2=1, read once per process: a fresh
    process) against the oracle at BASELINE size — full device and a partition — and in a layer stack."""
    import os
    import subprocess
    import sys
    env = dict(os.environ, DUET_FA2="1")
    r = subprocess.run([sys.executable, "-m", "pytest", __file__, "-q", "-m", "gpu", "-p", "no:cacheprovider",
                        "-k", "prefill_attention_output or (stack and cfg2)"], env=env, capture_output=True,
                       text=True, timeout=900, cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    assert r.returncode == 0 and " passed" in r.stdout and "failed" not in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]

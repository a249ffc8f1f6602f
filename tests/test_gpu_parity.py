"""GPU parity: libduet.so (through the C ABI) vs the CPU oracle on the same seeded inputs.

Tolerances (BASELINE.json north_star; C-6): normwise max relative error <= 2e-2 for bf16
kernels, <= 1e-4 for the fp32 path.  Bit-exact: KV slot placement (NaN-poisoned pool: exactly
the listed slots change), and results across every SM split and mode (split invariance).
"""
from dataclasses import replace

import numpy as np
import pytest
import torch

import paper_2511_04791_b200 as D
from synth import configs, workload
from synth import layer_weights as synth_layer_weights
from tests.gpu_helpers import GpuWorkload, make_ctx, spec_of
from tests.oracle_run import rel_err, run

pytestmark = pytest.mark.gpu

TOL = {"fp32": 1e-4, "bf16": 2e-2}


def _check_outputs(g: GpuWorkload, y_pre, y_dec, tol):
    if len(g.wl.pre_seqs):
        e = rel_err(g.y_pre.float().cpu().numpy(), y_pre)
        assert e <= tol, f"prefill rel err {e}"
    if len(g.wl.dec_ctx):
        for j in range(g.wl.k):
            e = rel_err(g.y_dec[j].float().cpu().numpy(), y_dec[j])
            assert e <= tol, f"decode step {j + 1} rel err {e}"


def _check_kv(g: GpuWorkload, kv_oracle, tol):
    """Written slots match the oracle's writes; every other slot keeps its poison / history."""
    wl = g.wl
    written = set(kv_oracle.writes)
    for l in range(wl.n_layers):
        Kg = g.K[l].float().cpu().numpy()
        Vg = g.V[l].float().cpu().numpy()
        hist = np.zeros((wl.n_pages, wl.cfg.batch.page_size), dtype=bool)
        for (ll, trow, uid, n) in wl.history_items():
            if ll == l:
                p = np.arange(n)
                hist[trow[p // 16], p % 16] = True
        wmask = np.zeros_like(hist)
        for (ll, page, s) in written:
            if ll == l:
                wmask[page, s] = True
        untouched = ~(hist | wmask)
        assert np.all(np.isnan(Kg.transpose(0, 2, 1, 3)[untouched])), "a slot outside the write list changed"
        assert np.all(np.isnan(Vg.transpose(0, 2, 1, 3)[untouched]))
        Kw = Kg.transpose(0, 2, 1, 3)[wmask]
        Ko = kv_oracle.K[l].transpose(0, 2, 1, 3)[wmask]
        assert not np.any(np.isnan(Kw))
        assert rel_err(Kw, Ko) <= tol
        Vw = Vg.transpose(0, 2, 1, 3)[wmask]
        Vo = kv_oracle.V[l].transpose(0, 2, 1, 3)[wmask]
        assert rel_err(Vw, Vo) <= tol


def _run_split(wl, dtype, split_fn, flags=0):
    g = GpuWorkload(wl, dtype)
    ctx = make_ctx(wl, dtype, flags)
    split = split_fn(ctx)
    g.step(ctx, split)
    torch.cuda.synchronize()
    return g, ctx


@pytest.mark.parametrize("cfg_name,k", [("cfg1", 2), ("cfg1-bf16", 2), ("cfg1-gqa", 4)])
def test_parity_tiny_temporal_and_every_split(cfg_name, k):
    cfg = configs.get_config(cfg_name)
    wl = workload.build(cfg, k=k)
    tol = TOL[cfg.dtype]
    y_pre, y_dec, kv_o = run(wl)
    # temporal mode runs k = 1: compare against the oracle's first decode step
    wl1 = workload.build(cfg, k=1)
    y_pre1, y_dec1, kv_o1 = run(wl1)
    ctx = make_ctx(wl, cfg.dtype)
    g = GpuWorkload(wl1, cfg.dtype)
    g.step(ctx, D.split_struct(D.DUET_MODE_TEMPORAL, 148, 0, 1))
    torch.cuda.synchronize()
    _check_outputs(g, y_pre1, y_dec1, tol)
    _check_kv(g, kv_o1, tol)
    ref_pre, ref_dec = None, None
    parts, total = ctx.partitions()
    assert parts and total == 148
    for s_d in parts:
        g = GpuWorkload(wl, cfg.dtype)
        g.step(ctx, D.split_struct(D.DUET_MODE_SPATIAL, total - s_d, s_d, k))
        torch.cuda.synchronize()
        _check_outputs(g, y_pre, y_dec, tol)
        _check_kv(g, kv_o, tol)
        # split invariance: bitwise identical across every split
        if ref_pre is None:
            ref_pre, ref_dec = g.y_pre.clone(), g.y_dec.clone()
        else:
            assert torch.equal(g.y_pre, ref_pre) and torch.equal(g.y_dec, ref_dec), f"split {s_d} differs"
    ctx.close()


def test_parity_llama_shapes_ragged_prefix():
    """Llama-3-8B layer shapes (tensor-core GEMM + flash prefill attention, d_h = 128, GQA 4) on a
    ragged batch: two prefill sequences (one chunk with a 37-token prefix), three decodes, k = 3."""
    cfg = configs.get_config("cfg2-mini")
    wl = workload.build(cfg)
    y_pre, y_dec, kv_o = run(wl)
    ctx = make_ctx(wl, "bf16")
    parts, total = ctx.partitions()
    for s_d in (parts[0], parts[-1]):
        g = GpuWorkload(wl, "bf16")
        g.step(ctx, D.split_struct(D.DUET_MODE_SPATIAL, total - s_d, s_d, wl.k))
        torch.cuda.synchronize()
        _check_outputs(g, y_pre, y_dec, TOL["bf16"])
        _check_kv(g, kv_o, TOL["bf16"])
    wl1 = workload.build(cfg, k=1)
    y_pre1, y_dec1, _ = run(wl1)
    g = GpuWorkload(wl1, "bf16")
    g.step(ctx, D.split_struct(D.DUET_MODE_TEMPORAL, total, 0, 1))
    torch.cuda.synchronize()
    _check_outputs(g, y_pre1, y_dec1, TOL["bf16"])


def test_parity_qwen_shapes_gqa5_bias():
    """Qwen2.5-14B layer shapes (d = 5120, h_q = 40, h_kv = 8: GQA group 5 — an odd last head per group
    in the paired-head flash attention — QKV bias, ffn 13824) on a ragged batch, spatial k = 2 and
    temporal, against the oracle."""
    cfg = configs.get_config("cfg4-mini")
    wl = workload.build(cfg)
    y_pre, y_dec, kv_o = run(wl)
    ctx = make_ctx(wl, "bf16")
    parts, total = ctx.partitions()
    g = GpuWorkload(wl, "bf16")
    g.step(ctx, D.split_struct(D.DUET_MODE_SPATIAL, total - parts[1], parts[1], wl.k))
    torch.cuda.synchronize()
    _check_outputs(g, y_pre, y_dec, TOL["bf16"])
    _check_kv(g, kv_o, TOL["bf16"])
    g = GpuWorkload(wl, "bf16")   # temporal runs k = 1: step 1 of the same oracle window
    g.step(ctx, D.split_struct(D.DUET_MODE_TEMPORAL, total, 0, 1))
    torch.cuda.synchronize()
    assert rel_err(g.y_pre.float().cpu().numpy(), y_pre) <= TOL["bf16"]
    assert rel_err(g.y_dec[0].float().cpu().numpy(), y_dec[0]) <= TOL["bf16"]


def test_parity_large_activations_running_max_rebase():
    """Inputs scaled x16 (still exact in bf16): attention scores grow along the sequence, so rows re-base
    their running max at different key tiles (warp-divergent rescale decisions in the flash kernel)."""
    cfg = configs.get_config("cfg2-mini")
    wl = workload.build(cfg, k=1)
    wl.x_pre = (wl.x_pre * 16).astype(np.float32)
    wl.x_dec = (wl.x_dec * 16).astype(np.float32)
    y_pre, y_dec, _ = run(wl)
    ctx = make_ctx(wl, "bf16")
    g = GpuWorkload(wl, "bf16")
    g.step(ctx, D.split_struct(D.DUET_MODE_TEMPORAL, 148, 0, 1))
    torch.cuda.synchronize()
    _check_outputs(g, y_pre, y_dec, TOL["bf16"])


def test_fine_grained_partitions_and_no_graph():
    cfg = configs.get_config("cfg1")
    wl = workload.build(cfg, k=3)
    y_pre, y_dec, _ = run(wl)
    ctx = make_ctx(wl, "fp32", D.DUET_CTX_FINE_SPLIT | D.DUET_CTX_NO_GRAPH)
    parts, total = ctx.partitions()
    assert parts[0] == 2 and 2 in parts and 146 in parts
    for s_d in (2, 10, 74, 146):
        g = GpuWorkload(wl, "fp32")
        g.step(ctx, D.split_struct(D.DUET_MODE_SPATIAL, total - s_d, s_d, 3))
        torch.cuda.synchronize()
        _check_outputs(g, y_pre, y_dec, TOL["fp32"])


def test_temporal_vs_spatial_k1_and_run_to_run_determinism():
    """Temporal and spatial modes compute the same function (split-K weight-streaming GEMMs on a
    <= 128-row side reduce in another fp32 grouping than the 128-row tiles of the joint batch, so the
    two agree to rounding, not bitwise); a repeated step of the same split is bitwise identical."""
    cfg = configs.get_config("cfg1-bf16")
    wl = workload.build(cfg, k=1)
    gt, ctx = _run_split(wl, "bf16", lambda c: D.split_struct(D.DUET_MODE_TEMPORAL, 148, 0, 1))
    gs = GpuWorkload(wl, "bf16")
    gs.step(ctx, D.split_struct(D.DUET_MODE_SPATIAL, 132, 16, 1))
    torch.cuda.synchronize()
    assert rel_err(gs.y_dec.float().cpu().numpy(), gt.y_dec.float().cpu().numpy()) <= 1e-2
    assert rel_err(gs.y_pre.float().cpu().numpy(), gt.y_pre.float().cpu().numpy()) <= 1e-2
    gs2 = GpuWorkload(wl, "bf16")
    gs2.step(ctx, D.split_struct(D.DUET_MODE_SPATIAL, 132, 16, 1))
    torch.cuda.synchronize()
    assert torch.equal(gs.y_dec, gs2.y_dec)
    assert torch.equal(gs.y_pre, gs2.y_pre)


def test_decode_after_prefill_invariant_gpu():
    """Decoding token t after a prefill of 0..t-1 matches row t of a prefill over 0..t."""
    cfg = configs.get_config("cfg1")
    T = 77
    full = workload.build(cfg, pre_seqs=[(T, 0)], dec_ctx=[], k=1)
    g1, ctx = _run_split(full, "fp32", lambda c: D.split_struct(D.DUET_MODE_TEMPORAL, 148, 0, 1))
    part = workload.build(cfg, pre_seqs=[(T - 1, 0)], dec_ctx=[], k=1)
    g2 = GpuWorkload(part, "fp32")
    g2.step(ctx, D.split_struct(D.DUET_MODE_TEMPORAL, 148, 0, 1))
    # decode the last token against the cache the partial prefill wrote (same pages)
    dec = dict(c=[T - 1], table=part.pre_tables, x=g1.x_pre[T - 1:T].contiguous(),
               y=torch.zeros((1, 1, cfg.model.d_model), device="cuda"))
    ctx.step(g2.W, None, dec, g2.K, g2.V, part.n_pages, D.split_struct(D.DUET_MODE_SPATIAL, 132, 16, 1))
    torch.cuda.synchronize()
    e = rel_err(dec["y"][0, 0].cpu().numpy(), g1.y_pre[T - 1].cpu().numpy())
    assert e < 1e-4, e


def test_page_table_errors_are_caught_before_launch():
    cfg = configs.get_config("cfg1")
    wl = workload.build(cfg, k=1)
    g = GpuWorkload(wl, "fp32")
    ctx = make_ctx(wl, "fp32")
    bad = wl.dec_tables.copy()
    bad[1, 0] = bad[0, 0]
    dec = dict(c=wl.dec_ctx, table=bad, x=g.x_dec, y=g.y_dec)
    with pytest.raises(D.DuetError) as e:
        ctx.step(g.W, g.prefill_arg(), dec, g.K, g.V, wl.n_pages, D.split_struct(0, 148, 0, 1))
    assert e.value.status == -2 and "used twice" in str(e.value)
    with pytest.raises(D.DuetError) as e:
        ctx.step(g.W, g.prefill_arg(), g.decode_arg(), g.K, g.V, wl.n_pages, D.split_struct(1, 137, 11, 1))
    assert e.value.status == -2
    bad = wl.dec_tables.copy()
    bad[0, 0] = wl.n_pages + 5
    with pytest.raises(D.DuetError):
        ctx.step(g.W, None, dict(c=wl.dec_ctx, table=bad, x=g.x_dec, y=g.y_dec), g.K, g.V, wl.n_pages,
                 D.split_struct(0, 148, 0, 1))


@pytest.mark.parametrize("M,N,K,epi", [(1, 256, 256, 0), (130, 384, 512, 1), (257, 160, 1024, 2),
                                       (2048, 6144, 4096, 0), (64, 4096, 14336, 1), (64, 14336, 4096, 2),
                                       (100, 512, 256, 2), (8, 768, 256, 3), (77, 6144, 4096, 3),
                                       (300, 1000, 512, 3), (128, 200, 128, 1), (600, 768, 2048, 1),
                                       (520, 256, 1024, 2), (2112, 4096, 4096, 1),
                                       (256, 4096, 4096, 1), (256, 4096, 14336, 1), (512, 4096, 4096, 0),
                                       (384, 4096, 2048, 3)])
def test_op_gemm_bf16(M, N, K, epi):
    """tcgen05 GEMM vs float64 torch: CTA-pair 256x256 tiles (M > 128) with shape-only split-K
    for under-filled grids (the 256-row decode batch's O / down: 600 / 256 / 512 / 384 rows here),
    swap-AB tiles with shape-only split-K (M <= 128), every epilogue (3 = store + bias), ragged M / N."""
    torch.manual_seed(0)
    cfg = configs.get_config("cfg2")
    wl = workload.build(cfg, pre_seqs=[(16, 0)], dec_ctx=[], k=1, with_weights=False)
    ctx = make_ctx(wl, "bf16", extra_tokens=M)    # workspace sized for M-row launches (split-K partials)
    A = (torch.randn(M, K, device="cuda") / 4).bfloat16()
    Bn = 2 * N if epi == 2 else N
    B = (torch.randn(Bn, K, device="cuda") / K ** 0.5).bfloat16()
    R = torch.randn(M, N, device="cuda").bfloat16()
    bias = torch.randn(N, device="cuda").bfloat16()
    C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    ctx.op_gemm(A, B, C, R if epi == 1 else None, bias if epi == 3 else None, 0 if epi == 3 else epi)
    torch.cuda.synchronize()
    acc = A.double() @ B.double().T
    if epi == 0:
        ref = acc
    elif epi == 3:
        ref = acc + bias.double()
    elif epi == 1:
        ref = R.double() + acc
    else:
        g, u = acc[:, :N], acc[:, N:]
        ref = g / (1 + torch.exp(-g)) * u
    e = (C.double() - ref).abs().max().item() / ref.abs().max().item()
    assert e < 1e-2, e
    # split-K launches (M <= 128, long K) re-arm their tile counters and reduce in a fixed order:
    # a second call is bitwise identical
    C2 = torch.empty_like(C)
    ctx.op_gemm(A, B, C2, R if epi == 1 else None, bias if epi == 3 else None, 0 if epi == 3 else epi)
    torch.cuda.synchronize()
    assert torch.equal(C, C2)


@pytest.mark.slow
def test_parity_cfg2_full_layer_temporal_and_optimizer_split():
    """Llama-3-8B layer at BASELINE size (prefill 2048 + 64 decodes at 4k) against the oracle."""
    cfg = configs.get_config("cfg2")
    wl = workload.build(cfg, k=1)
    y_pre, y_dec, kv_o = run(wl)
    g, ctx = _run_split(wl, "bf16", lambda c: D.split_struct(D.DUET_MODE_TEMPORAL, 148, 0, 1))
    _check_outputs(g, y_pre, y_dec, TOL["bf16"])
    # f4: at this size the attention co-run model picks an SM split; the same kernels on fewer SMs
    # give the same function as the one-after-the-other temporal step (NO_CORUN context)
    assert ctx.last_step_times()["corun_s_d"] > 0
    # f4 with DUET_POD=1 (test_fused_pod_attention_parity_subprocess): the co-run split runs as ONE fused POD
    # launch (prefill-attention and decode-attention CTAs in one grid) — bitwise the one-after-the-other
    # step too, since each role runs the same per-item algorithm as its standalone kernel
    import os
    assert ctx.last_pod() == (os.environ.get("DUET_POD", "0") not in ("", "0"))
    g_seq, ctx_seq = _run_split(wl, "bf16", lambda c: D.split_struct(D.DUET_MODE_TEMPORAL, 148, 0, 1),
                                D.DUET_CTX_NO_CORUN)
    assert ctx_seq.last_step_times()["corun_s_d"] == 0
    assert torch.equal(g.y_pre, g_seq.y_pre) and torch.equal(g.y_dec, g_seq.y_dec)
    del ctx_seq, g_seq
    parts, total = ctx.partitions()
    for s_d in (parts[0], 32, parts[-1]):
        g = GpuWorkload(wl, "bf16")
        g.step(ctx, D.split_struct(D.DUET_MODE_SPATIAL, total - s_d, s_d, 1))
        torch.cuda.synchronize()
        _check_outputs(g, y_pre, y_dec, TOL["bf16"])
    _check_kv(g, kv_o, TOL["bf16"])


def test_tp_allreduce_path_world1_bitwise():
    """Head-sharded TP code path (§8 a9): a ctx with single-rank NCCL communicators runs the rank-0
    residual + allreduce-after-O/down path (as a no-op copy) and reproduces the plain ctx bitwise,
    in temporal and spatial mode (the decode side's allreduces are captured in its CUDA graph)."""
    cfg = configs.get_config("cfg1-bf16")
    wl = workload.build(cfg, k=2)
    for split in (D.split_struct(D.DUET_MODE_TEMPORAL, 148, 0, 1),):
        ref, ctx = _run_split(wl, "bf16", lambda c: split)
        ctx.close()
    ctx_tp = make_ctx(wl, "bf16")
    ctx_tp.set_comms(0, D.nccl_unique_id(), D.nccl_unique_id())
    g = GpuWorkload(wl, "bf16")
    g.step(ctx_tp, D.split_struct(D.DUET_MODE_TEMPORAL, 148, 0, 1))
    torch.cuda.synchronize()
    assert torch.equal(g.y_pre, ref.y_pre) and torch.equal(g.y_dec[0], ref.y_dec[0])
    parts, total = ctx_tp.partitions()
    sp = D.split_struct(D.DUET_MODE_SPATIAL, total - parts[1], parts[1], 2)
    ref2, ctx2 = _run_split(wl, "bf16", lambda c: sp)
    g2 = GpuWorkload(wl, "bf16")
    g2.step(ctx_tp, sp)
    torch.cuda.synchronize()
    assert torch.equal(g2.y_pre, ref2.y_pre) and torch.equal(g2.y_dec, ref2.y_dec)
    assert ctx_tp.calibrate_allreduce() == (0.0, 0.0)
    ctx_tp.check_comms()          # no asynchronous NCCL error on either side's communicator
    ctx2.close()
    ctx_tp.close()


@pytest.mark.parametrize("mode", ["spatial", "temporal"])
def test_lm_head_greedy_window_vs_oracle(mode):
    """f1: the decode window closed into an autoregressive loop (RMSNorm -> LM head GEMM -> greedy
    token -> embedding as the next input) against the oracle.  Tokens must match wherever the oracle's
    top-1 / top-2 logit gap exceeds the bf16 tolerance (2e-2 of the largest |logit|); a near-tie may
    resolve either way, and only rows whose earlier tokens matched are compared at later steps."""
    from oracle import layer as OL
    from synth import head_weights
    from tests.oracle_run import make_kv
    cfg = configs.get_config("cfg1-bf16")
    k = 3 if mode == "spatial" else 1
    wl = workload.build(cfg, k=k)
    m = OL.Model.from_cfg(cfg.model)
    head = head_weights(cfg.model, cfg.seed)
    toks = []
    y_ref = OL.decode_window(m, wl.weights, wl.x_dec, wl.dec_ctx, wl.dec_tables, make_kv(wl), k, head, toks)
    g = GpuWorkload(wl, "bf16")
    g.add_head(head)
    ctx = make_ctx(wl, "bf16")
    if mode == "spatial":
        parts, total = ctx.partitions()
        split = D.split_struct(D.DUET_MODE_SPATIAL, total - parts[0], parts[0], k)
    else:
        split = D.split_struct(D.DUET_MODE_TEMPORAL, 148, 0, 1)
    g.step(ctx, split)
    torch.cuda.synchronize()
    tok_gpu = g.head["tokens"].cpu().numpy()
    alive = np.ones(len(wl.dec_ctx), dtype=bool)
    checked = 0
    for j in range(k):
        logits, t_ref = toks[j]
        srt = np.sort(logits, axis=1)
        clear = (srt[:, -1] - srt[:, -2]) > 2e-2 * np.abs(logits).max(axis=1)
        sel = alive & clear
        assert np.array_equal(tok_gpu[j][sel], t_ref[sel]), (j, tok_gpu[j], t_ref)
        # a near-tie: the GPU's token is one of the (near-)maxima
        for r in np.where(alive & ~clear)[0]:
            assert logits[r, tok_gpu[j][r]] >= srt[r, -1] - 2e-2 * np.abs(logits[r]).max()
        e = rel_err(g.y_dec[j].float().cpu().numpy()[alive], y_ref[j][alive]) if alive.any() else 0.0
        assert e <= 2e-2, (j, e)
        checked += int(sel.sum())
        alive &= tok_gpu[j] == t_ref
    assert checked >= len(wl.dec_ctx) // 2  # the comparison is not vacuous
    ctx.close()


def test_iteration_stream_served_trace_vs_oracle():
    """f2 end to end: duet_sched forms the iterations of a small bursty trace on the tiny model; every
    iteration runs through duet_step (alternating temporal and spatial with k = 2) and through the
    oracle on the same rows, the same page tables and a KV pool that both sides fill iteration after
    iteration (pages are reused once requests finish).  Outputs must agree every iteration."""
    from oracle import layer as OL
    from synth import configs, counter_values
    cfg = configs.get_config("cfg1-bf16")
    m = cfg.model
    M = OL.Model.from_cfg(m)
    d, P = m.d_model, 16
    weights = [synth_layer_weights(m, 0, cfg.seed)]
    n_pages = 40
    sched = D.Sched(page_size=P, n_pages=n_pages, token_budget=96, max_batch=8, max_prefill_seqs=4, k_max=2,
                    max_pages_per_seq=16)
    trace = [(0, 70, 4, 0.0), (1, 30, 3, 0.0), (2, 120, 2, 0.0), (3, 45, 5, 0.001), (4, 20, 3, 0.002)]
    for r in trace:
        sched.add(*r)
    tdt = torch.bfloat16
    W = [{k: torch.from_numpy(np.ascontiguousarray(v)).to("cuda", tdt) for k, v in weights[0].items() if v is not None}]
    Kg = [torch.zeros((n_pages, m.n_kv_heads, P, m.head_dim), dtype=tdt, device="cuda")]
    Vg = [torch.zeros_like(Kg[0])]
    kv_o = OL.PagedKV(1, n_pages, m.n_kv_heads, P, m.head_dim)
    ctx = D.Ctx(spec_of(m, "bf16"), 96, 4, 8, 2, 16, 256, D.DUET_DTYPE_BF16)
    parts, total = ctx.partitions()

    def rows(rid, p0, n):   # input row of (request, position): exact bf16 grid values
        return counter_values(cfg.seed, 31, (n, d), (rid * 4096 + p0) * d)

    it_no, now = 0, 0.0
    while True:
        it = sched.next(now)
        if not it["prefill"] and not it["decode"]:
            if it["unfinished"] == 0:
                break
            now = it["next_arrival"]
            continue
        n_pre, n_dec = len(it["prefill"]), len(it["decode"])
        tab = it["table"]
        spatial = it_no % 2 == 1 and n_pre > 0 and n_dec > 0
        k = 2 if spatial else 1
        x_pre = np.concatenate([rows(rid, c, q) for rid, q, c in it["prefill"]]) if n_pre else np.zeros((0, d))
        x_dec = np.concatenate([rows(rid, c, 1) for rid, c in it["decode"]]) if n_dec else np.zeros((0, d))
        # oracle: the prefill chunks then the k-step decode window, on the shared paged pool
        y_pre_o = OL.prefill_forward(M, weights, x_pre, [(q, c) for _, q, c in it["prefill"]], tab[:n_pre], kv_o) \
            if n_pre else None
        y_dec_o = OL.decode_window(M, weights, x_dec, [c for _, c in it["decode"]], tab[n_pre:], kv_o, k) \
            if n_dec else None
        xp = torch.from_numpy(x_pre).to("cuda", tdt)
        xd = torch.from_numpy(x_dec).to("cuda", tdt)
        yp = torch.empty_like(xp)
        yd = torch.empty((k,) + tuple(xd.shape), dtype=tdt, device="cuda")
        pre = dict(q=[q for _, q, _ in it["prefill"]], c=[c for _, _, c in it["prefill"]],
                   table=np.ascontiguousarray(tab[:n_pre]), x=xp, y=yp) if n_pre else None
        dec = dict(c=[c for _, c in it["decode"]], table=np.ascontiguousarray(tab[n_pre:]), x=xd, y=yd) \
            if n_dec else None
        split = D.split_struct(D.DUET_MODE_SPATIAL, total - parts[0], parts[0], k) if spatial else \
            D.split_struct(D.DUET_MODE_TEMPORAL, total, 0, 1)
        ctx.step(W, pre, dec, Kg, Vg, n_pages, split)
        torch.cuda.synchronize()
        if n_pre:
            assert rel_err(yp.float().cpu().numpy(), y_pre_o) <= TOL["bf16"], it_no
        if n_dec:
            for j in range(k):
                assert rel_err(yd[j].float().cpu().numpy(), y_dec_o[j]) <= TOL["bf16"], (it_no, j)
        sched.commit(k)
        it_no += 1
        now += 1e-3
    assert it_no >= 6 and sched.free_pages() == n_pages
    ctx.close()
    sched.close()


@pytest.mark.skipif(bool(__import__("os").environ.get("DUET_CORUN")), reason="already the forced co-run run")
def test_forced_attention_corun_parity_subprocess():
    """f4 co-run forced onto small ragged batches (a fresh process: the switch is read once per process):
    the Llama ragged-prefix, Qwen GQA-5 + bias and running-max re-base cases pass against the oracle with
    the two attentions of every temporal step on a 16-SM decode group and the remainder."""
    import os
    import subprocess
    import sys
    env = dict(os.environ, DUET_CORUN="16")
    r = subprocess.run([sys.executable, "-m", "pytest", __file__, "-q", "-m", "gpu", "-p", "no:cacheprovider",
                        "-k", "llama_shapes or qwen or running_max"], env=env, capture_output=True, text=True,
                       timeout=900, cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    assert r.returncode == 0 and "3 passed" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]


@pytest.mark.skipif(bool(__import__("os").environ.get("DUET_POD")), reason="already the POD run")
def test_fused_pod_attention_parity_subprocess():
    """f4 POD-style fused attention (DUET_POD=1, read once per process: a fresh process): the two attentions
    of a temporal step as ONE launch — the cfg2 layer at BASELINE size bitwise equal to the one-after-the-
    other step and against the oracle, and the forced 16-SM co-run cases (ragged Llama prefixes, Qwen GQA-5 +
    bias, running-max re-base) against the oracle."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    for extra, k, n in (({}, "cfg2_full", 1), ({"DUET_CORUN": "16"}, "llama_shapes or qwen or running_max", 3)):
        env = dict(os.environ, DUET_POD="1", **extra)
        r = subprocess.run([sys.executable, "-m", "pytest", __file__, "-q", "-m", "gpu", "-p", "no:cacheprovider",
                            "-k", k], env=env, capture_output=True, text=True, timeout=900, cwd=root)
        assert r.returncode == 0 and f"{n} passed" in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]


@pytest.mark.skipif(bool(__import__("os").environ.get("DUET_GEMM2_BN")), reason="already the forced-width run")
def test_narrow_pair_tile_gemm_parity_subprocess():
    """The optional 256 x 128 CTA-pair tile (DUET_GEMM2_BN=128, read once per process: a fresh process)
    and the four-producer variant pass the op-level GEMM tests and a layer test against the oracle."""
    import os
    import subprocess
    import sys
    env = dict(os.environ, DUET_GEMM2_BN="128", DUET_GEMM2_PROD="4")
    r = subprocess.run([sys.executable, "-m", "pytest", __file__, "-q", "-m", "gpu", "-p", "no:cacheprovider",
                        "-k", "op_gemm or llama_shapes"], env=env, capture_output=True, text=True,
                       timeout=900, cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    assert r.returncode == 0 and " passed" in r.stdout and "failed" not in r.stdout, r.stdout[-2000:] + r.stderr[-2000:]

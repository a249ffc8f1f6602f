"""GPU parity of the fused GEMM + allreduce (§4.1).

In a head-sharded TP block the O and FFN-down projections are row-parallel: rank r holds the columns
A_r of the activation and the rows B_r of the weight's input dimension, and the layer needs
R + sum_r A_r B_r^T on every rank — the allreduce after O and down.  `duet_op_gemm_ar_emul`
runs the fused kernel with n ranks emulated in one grid on this GPU (the ranks' owner warps wait on
each other, so they must share a launch: B200_PROFILING); the reference is oracle.layer.row_parallel_allreduce
(float64 numpy, pinned on CPU by tests/test_oracle_layer.py).
The ctx-level tests open the fused path on a single-rank group (tp = 1: the same kernel with one
owner) and compare the layer stack with the oracle.
"""
import numpy as np
import pytest
import torch

import paper_2511_04791_b200 as D
from synth import configs, workload
from tests.gpu_helpers import GpuWorkload, make_ctx
from oracle.layer import row_parallel_allreduce
from tests.oracle_run import rel_err, run

pytestmark = pytest.mark.gpu

TOL = 2e-2


def _ref(A, B, R):
    """oracle.layer.row_parallel_allreduce on the bf16 operands (exact in float64)"""
    n = A.shape[0]
    return torch.from_numpy(row_parallel_allreduce([A[r].double().cpu().numpy() for r in range(n)],
                                                   [B[r].double().cpu().numpy() for r in range(n)],
                                                   R.double().cpu().numpy())).cuda()


def _ctx_for_ops(M):
    cfg = configs.get_config("cfg2")
    wl = workload.build(cfg, pre_seqs=[(16, 0)], dec_ctx=[], k=1, with_weights=False)
    return make_ctx(wl, "bf16", extra_tokens=M)


@pytest.mark.parametrize("n,M,N,K", [(1, 300, 512, 384), (2, 300, 512, 384), (3, 520, 1024, 192),
                                     (4, 1000, 768, 256), (8, 257, 256, 128), (2, 2112, 4096, 2048),
                                     (4, 2112, 4096, 1024)])
def test_gemm_allreduce_emulated_ranks(n, M, N, K):
    """Every emulated rank's output equals the oracle's R + sum_r A_r B_r^T within the bf16 tolerance and all
    ranks hold bitwise the same rows (one owner computes each tile and pushes it to every rank).  Ragged
    M (a partial last 256-row tile), tiles not divisible by n, and the cfg2 O / down shapes
    (M = 2112, N = d = 4096) split over 2 and 4 ranks."""
    torch.manual_seed(n * 1000 + M)
    ctx = _ctx_for_ops(M)
    A = (torch.randn(n, M, K, device="cuda") / 4).bfloat16()
    B = (torch.randn(n, N, K, device="cuda") / (n * K) ** 0.5).bfloat16()
    R = torch.randn(M, N, device="cuda").bfloat16()
    C = torch.full((n, M, N), float("nan"), device="cuda", dtype=torch.bfloat16)
    ctx.op_gemm_ar_emul(A, B, R, C)
    torch.cuda.synchronize()
    ref = _ref(A, B, R)
    for r in range(n):
        assert not torch.isnan(C[r]).any(), f"rank {r}: rows never written"
        e = (C[r].double() - ref).abs().max().item() / ref.abs().max().item()
        assert e < 1e-2, (r, e)
        assert torch.equal(C[r], C[0]), f"rank {r} differs from rank 0"
    # counters are re-armed by their waiters: repeated launches (and new operands) stay correct
    for it in range(3):
        A2 = (torch.randn(n, M, K, device="cuda") / 4).bfloat16()
        C2 = torch.empty_like(C)
        ctx.op_gemm_ar_emul(A2, B, R, C2)
        torch.cuda.synchronize()
        ref2 = _ref(A2, B, R)
        e = (C2[0].double() - ref2).abs().max().item() / ref2.abs().max().item()
        assert e < 1e-2, (it, e)
        assert all(torch.equal(C2[r], C2[0]) for r in range(n))
    # deterministic: the same operands give the same bits
    C3 = torch.empty_like(C)
    ctx.op_gemm_ar_emul(A, B, R, C3)
    torch.cuda.synchronize()
    assert torch.equal(C3, C)
    ctx.close()


def test_gemm_allreduce_emulated_in_cuda_graph():
    """The fused kernel needs no per-launch epoch: a captured launch replays correctly on new operands."""
    n, M, N, K = 2, 640, 1024, 512
    ctx = _ctx_for_ops(M)
    A = (torch.randn(n, M, K, device="cuda") / 4).bfloat16()
    B = (torch.randn(n, N, K, device="cuda") / (n * K) ** 0.5).bfloat16()
    R = torch.randn(M, N, device="cuda").bfloat16()
    C = torch.empty(n, M, N, device="cuda", dtype=torch.bfloat16)
    ctx.op_gemm_ar_emul(A, B, R, C)  # first launch outside the capture (attributes, workspace)
    torch.cuda.synchronize()
    s = torch.cuda.Stream()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        ctx.op_gemm_ar_emul(A, B, R, C, stream=s.cuda_stream)
    for it in range(3):
        A.copy_((torch.randn(n, M, K, device="cuda") / 4).bfloat16())
        C.zero_()
        g.replay()
        torch.cuda.synchronize()
        ref = _ref(A, B, R)
        e = (C[1].double() - ref).abs().max().item() / ref.abs().max().item()
        assert e < 1e-2, (it, e)
        assert torch.equal(C[0], C[1])
    ctx.close()


def test_gemm_allreduce_sensitivity():
    """The check catches a missing rank: dropping one rank's partial moves the result far beyond tol."""
    n, M, N, K = 2, 512, 512, 256
    torch.manual_seed(7)
    ctx = _ctx_for_ops(M)
    A = (torch.randn(n, M, K, device="cuda") / 4).bfloat16()
    B = (torch.randn(n, N, K, device="cuda") / (n * K) ** 0.5).bfloat16()
    R = torch.zeros(M, N, device="cuda").bfloat16()
    C = torch.empty(n, M, N, device="cuda", dtype=torch.bfloat16)
    ctx.op_gemm_ar_emul(A, B, R, C)
    torch.cuda.synchronize()
    full = _ref(A, B, R)
    only0 = _ref(A[:1], B[:1], R)
    e_ok = (C[0].double() - full).abs().max().item() / full.abs().max().item()
    e_bad = (only0 - full).abs().max().item() / full.abs().max().item()
    assert e_ok < 1e-2 < e_bad
    ctx.close()


def _open_single_rank_group(ctx):
    ctx.set_comms(0, D.nccl_unique_id(), D.nccl_unique_id())
    ctx.ar_open([ctx.ar_handle()])


@pytest.mark.parametrize("cfg_name,L", [("cfg1-bf16", 2), ("cfg2-mini", 2)])
def test_fused_allreduce_layer_stack_vs_oracle(cfg_name, L):
    """duet_step with the fused path open (tp = 1 group): the O / down projections of every > 128-row
    batch run as the fused kernel (the last layer's output copied out of the arena), temporal and
    spatial, L = 2 — against the oracle, and with fewer launches than the NCCL path (no allreduce
    launches where the fused kernel ran)."""
    cfg = configs.get_config(cfg_name)
    wl1 = workload.build(cfg, k=1, n_layers=L)
    y_pre, y_dec, _ = run(wl1)
    ctx_nccl = make_ctx(wl1, "bf16")
    ctx_nccl.set_comms(0, D.nccl_unique_id(), D.nccl_unique_id())
    g0 = GpuWorkload(wl1, "bf16")
    g0.step(ctx_nccl, D.split_struct(D.DUET_MODE_TEMPORAL, 148, 0, 1))
    torch.cuda.synchronize()
    k_nccl = ctx_nccl.last_step_times()["kernels"]
    ctx_nccl.close()
    ctx = make_ctx(wl1, "bf16")
    _open_single_rank_group(ctx)
    g = GpuWorkload(wl1, "bf16")
    g.step(ctx, D.split_struct(D.DUET_MODE_TEMPORAL, 148, 0, 1))
    torch.cuda.synchronize()
    assert rel_err(g.y_pre.float().cpu().numpy(), y_pre) <= TOL
    assert rel_err(g.y_dec[0].float().cpu().numpy(), y_dec[0]) <= TOL
    assert ctx.last_step_times()["kernels"] < k_nccl
    # spatial: the prefill side (> 128 rows at cfg2-mini) fuses, the decode side keeps NCCL
    wl = workload.build(cfg, k=2, n_layers=L)
    y_pre2, y_dec2, _ = run(wl)
    parts, total = ctx.partitions()
    ctx2 = make_ctx(wl, "bf16")
    _open_single_rank_group(ctx2)
    g2 = GpuWorkload(wl, "bf16")
    g2.step(ctx2, D.split_struct(D.DUET_MODE_SPATIAL, total - parts[1], parts[1], 2))
    torch.cuda.synchronize()
    assert rel_err(g2.y_pre.float().cpu().numpy(), y_pre2) <= TOL
    for j in range(2):
        assert rel_err(g2.y_dec[j].float().cpu().numpy(), y_dec2[j]) <= TOL
    # a second step on the same ctx (counters re-armed, graphs replayed)
    g2.step(ctx2, D.split_struct(D.DUET_MODE_SPATIAL, total - parts[1], parts[1], 2))
    torch.cuda.synchronize()
    assert rel_err(g2.y_pre.float().cpu().numpy(), y_pre2) <= TOL
    ctx2.close()
    ctx.close()


def test_fused_allreduce_open_errors():
    cfg = configs.get_config("cfg1-bf16")
    wl = workload.build(cfg, k=1)
    ctx = make_ctx(wl, "bf16")
    with pytest.raises(D.DuetError):
        ctx.ar_handle()                  # no communicators yet
    ctx.set_comms(0, D.nccl_unique_id(), D.nccl_unique_id())
    h = ctx.ar_handle()
    assert len(h) == 64
    with pytest.raises(D.DuetError):
        ctx.ar_open([h, h])              # two handles for a tp = 1 group
    ctx.ar_open([h])
    with pytest.raises(D.DuetError):
        ctx.ar_open([h])                 # already open
    ctx.close()

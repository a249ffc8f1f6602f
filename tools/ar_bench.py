#!/usr/bin/env python
"""Fused GEMM + allreduce (f3) against the plain residual GEMM on one B200 (CUDA events, 20 launches
after 3 warm-ups, full device).

Per shape (the row-parallel O and down projections: cfg2 = Llama-3-8B 2112-row temporal batch, cfg3 =
its 8192-token prompt, cfg5 = Llama-3-70B at TP 2 / 4 with an 8192-row chunk):
  plain    duet_op_gemm, residual epilogue, the unsharded shape M x N x K
  fused1   the fused kernel on a single-rank group (owner = self: the epilogue path without peers)
  emul_n   n ranks emulated in one grid, rank r on 148 / 2 / n CTA pairs doing M x N x K/n — the same
           FLOPs as `plain` on the same SMs, plus the exchange (partials to the owner, results to every
           rank: (n - 1) / n x 2 x M x N x 4 B per rank through L2 / HBM here, NVLink on a real group)
Algorithmic FLOPs 2 M N K; `frac` against the measured bf16 burst peak.

usage: python tools/ar_bench.py [--out profiles/r02_f3_ar_bench.txt]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    import torch
    import paper_2511_04791_b200 as D
    from synth import configs
    peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))
    peak = None
    for k in ("bf16_tflops",):
        if k in peaks:
            peak = float(peaks[k])
            break
    m = configs.get_config("cfg2").model
    spec = D.make_spec(1, m.d_model, m.ffn_dim, m.n_q_heads, m.n_kv_heads, m.head_dim, m.vocab, 2, 1, 0, 1,
                       m.rope_theta, m.norm_eps)
    ctx = D.Ctx(spec, 8192, 1, 1, 1, 64, 4096, D.DUET_DTYPE_BF16)
    shapes = [("cfg2 O", 2112, 4096, 4096), ("cfg2 down", 2112, 4096, 14336),
              ("cfg3 O", 8192, 4096, 4096), ("cfg3 down", 8192, 4096, 14336),
              ("cfg5 O", 8192, 8192, 8192), ("cfg5 down", 8192, 8192, 28672)]
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def timed(fn, reps=20):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        ev0.record()
        for _ in range(reps):
            fn()
        ev1.record()
        torch.cuda.synchronize()
        return ev0.elapsed_time(ev1) / reps * 1e-3

    lines = [f"# tools/ar_bench.py: fused GEMM + allreduce (f3) vs plain residual GEMM, full B200, "
             f"peak {peak} TFLOP/s (MEASURED_PEAKS.json burst)"]
    for name, M, N, K in shapes:
        torch.manual_seed(0)
        A = (torch.randn(M, K, device="cuda") / 4).bfloat16()
        B = (torch.randn(N, K, device="cuda") / K ** 0.5).bfloat16()
        R = torch.randn(M, N, device="cuda").bfloat16()
        C = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
        fl = 2.0 * M * N * K
        row = {}
        row["plain"] = timed(lambda: ctx.op_gemm(A, B, C, R, None, D.DUET_EPI_RESIDUAL))
        C1 = torch.empty(1, M, N, device="cuda", dtype=torch.bfloat16)
        row["fused1"] = timed(lambda: ctx.op_gemm_ar_emul(A.view(1, M, K), B.view(1, N, K), R, C1))
        for n in (2, 4):
            if K % (64 * n):
                continue
            # rank r's shard: columns [r K/n, (r+1) K/n) of A and B, stacked [n][M][K/n]
            As = A.view(M, n, K // n).permute(1, 0, 2).contiguous()
            Bs = B.view(N, n, K // n).permute(1, 0, 2).contiguous()
            Cn = torch.empty(n, M, N, device="cuda", dtype=torch.bfloat16)
            row[f"emul{n}"] = timed(lambda: ctx.op_gemm_ar_emul(As, Bs, R, Cn))
            ref = C.float()
            e = (Cn[0].float() - ref).abs().max().item() / ref.abs().max().item()
            assert e < 2e-2, (name, n, e)
            del As, Bs, Cn
        parts = "  ".join(f"{k} {v * 1e6:8.1f} us {fl / v / 1e12:6.0f} TF/s ({fl / v / 1e12 / peak:.2f})"
                          for k, v in row.items())
        lines.append(f"{name:10s} M={M:5d} N={N:5d} K={K:5d}  {parts}")
        print(lines[-1], flush=True)
        del A, B, R, C, C1
        torch.cuda.empty_cache()
    ctx.close()
    if a.out:
        with open(a.out, "w") as f:
            f.write("\n".join(lines) + "\n")


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""Run one side of a configuration at a time (few layers) with progress output — hang/regression triage.

usage: python tools/debug_step.py --config cfg3-fit --layers 2 [--mode prefill|decode|temporal|spatial] [--sd 32]
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg3-fit")
    ap.add_argument("--layers", type=int, default=2)
    ap.add_argument("--mode", default="all")
    ap.add_argument("--sd", type=int, default=32)
    ap.add_argument("--k", type=int, default=2)
    ap.add_argument("--no-graph", action="store_true")
    args = ap.parse_args()
    import torch
    import paper_2511_04791_b200 as D
    from synth import configs, workload
    from synth.gpu import inputs_gpu, kv_pools_gpu, layer_weights_gpu

    cfg = configs.get_config(args.config)
    m = cfg.model
    dev = torch.device("cuda", 0)
    wl = workload.build(cfg, k=8, with_weights=False, n_layers=args.layers)
    W = [layer_weights_gpu(m, l, cfg.seed, dev, torch.bfloat16) for l in range(args.layers)]
    Kp, Vp = kv_pools_gpu(wl, dev, torch.bfloat16)
    x_pre, x_dec = inputs_gpu(wl, dev, torch.bfloat16)
    y_pre, y_dec = torch.empty_like(x_pre), torch.empty((8,) + tuple(x_dec.shape), dtype=torch.bfloat16, device=dev)
    spec = D.make_spec(args.layers, m.d_model, m.ffn_dim, m.n_q_heads, m.n_kv_heads, m.head_dim, m.vocab, 2, 1,
                       int(m.qkv_bias), 1, m.rope_theta, m.norm_eps)
    n_p, n_d = x_pre.shape[0], x_dec.shape[0]
    ctx = D.Ctx(spec, n_p, len(wl.pre_seqs), n_d, 8, max(wl.pre_tables.shape[1], wl.dec_tables.shape[1]),
                max([c + q for q, c in wl.pre_seqs] + [c + 8 for c in wl.dec_ctx]) + 16, D.DUET_DTYPE_BF16,
                D.DUET_CTX_NO_GRAPH if args.no_graph else 0)
    parts, total = ctx.partitions()
    pre = dict(q=[q for q, _ in wl.pre_seqs], c=[c for _, c in wl.pre_seqs], table=wl.pre_tables, x=x_pre, y=y_pre)

    def dec(k):
        return dict(c=wl.dec_ctx, table=wl.dec_tables, x=x_dec, y=y_dec[:k])

    T = D.split_struct(D.DUET_MODE_TEMPORAL, total, 0, 1)
    Sp = D.split_struct(D.DUET_MODE_SPATIAL, total - args.sd, args.sd, args.k)
    runs = {"prefill": (pre, None, T), "decode": (None, dec(1), T), "temporal": (pre, dec(1), T),
            "spatial_dec": (None, dec(args.k), Sp), "spatial_pre": (pre, None, Sp), "spatial": (pre, dec(args.k), Sp)}
    names = list(runs) if args.mode == "all" else [args.mode]
    for name in names:
        p_, d_, s_ = runs[name]
        t = time.time()
        print(f"{name}: launching", flush=True)
        ctx.step(W, p_, d_, Kp, Vp, wl.n_pages, s_)   # warm (graph capture etc.)
        torch.cuda.synchronize()
        ctx.profile_enable(True)
        ctx.step(W, p_, d_, Kp, Vp, wl.n_pages, s_)
        torch.cuda.synchronize()
        ks = ctx.profile_read()
        ctx.profile_enable(False)
        print("   kernels:", {k: (v["launches"], round(v["seconds"] * 1e3, 3)) for k, v in ks.items() if v["launches"]},
              flush=True)
        st = ctx.last_step_times()
        print(f"{name}: done in {time.time() - t:.2f}s  window {st['t_window'] * 1e3:.2f} ms  "
              f"dec {st['t_decode'] * 1e3:.2f}  pre {st['t_prefill'] * 1e3:.2f}  nan_pre={torch.isnan(y_pre).any().item()}",
              flush=True)


if __name__ == "__main__":
    main()

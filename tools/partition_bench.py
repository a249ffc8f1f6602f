#!/usr/bin/env python
"""Per-partition kernel rooflines: each side of the cfg2 mixed iteration run alone on an S-SM green
context (decode side: GEMMs + paged decode attention; prefill side: GEMMs + causal attention), with
CUDA events around every launch (duet_profile_*), against the calibrated Pi_SM(S), B_HBM(S).

Writes one JSON document (stdout and --out).  Usage: python tools/partition_bench.py [--out f.json]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="cfg2")
    ap.add_argument("--reps", type=int, default=10)
    ap.add_argument("--out", default=None)
    ap.add_argument("--only", default=None, choices=[None, "decode", "prefill"])
    ap.add_argument("--sd", type=int, default=None, help="single decode-partition size (with --only)")
    args = ap.parse_args()
    import torch
    import paper_2511_04791_b200 as D
    from synth import configs, workload
    from synth.gpu import inputs_gpu, kv_pools_gpu, layer_weights_gpu

    cfg = configs.get_config(args.config)
    m = cfg.model
    dev = torch.device("cuda", 0)
    tdt = torch.bfloat16
    wl = workload.build(cfg, k=1, with_weights=False)
    W = [layer_weights_gpu(m, l, cfg.seed, dev, tdt) for l in range(m.n_layers)]
    Kp, Vp = kv_pools_gpu(wl, dev, tdt)
    x_pre, x_dec = inputs_gpu(wl, dev, tdt)
    y_pre, y_dec = torch.empty_like(x_pre), torch.empty((1,) + tuple(x_dec.shape), dtype=tdt, device=dev)
    spec = D.make_spec(m.n_layers, m.d_model, m.ffn_dim, m.n_q_heads, m.n_kv_heads, m.head_dim, m.vocab, 2, 1,
                       int(m.qkv_bias), 1, m.rope_theta, m.norm_eps)
    n_p, n_d = x_pre.shape[0], x_dec.shape[0]
    ctx = D.Ctx(spec, n_p, 1, n_d, 1, max(wl.pre_tables.shape[1], wl.dec_tables.shape[1]),
                max([c + q for q, c in wl.pre_seqs] + [c + 2 for c in wl.dec_ctx]) + 16, D.DUET_DTYPE_BF16,
                D.DUET_CTX_NO_GRAPH)
    parts, total = ctx.partitions()
    if args.only:   # quick mode for profilers: no calibration launches
        fl = [0.0] + [1.6e15 * s / total for s in range(1, total + 1)]
        bw = [0.0] + [6.5e12 * (s / total) ** 0.32 for s in range(1, total + 1)]
    else:
        fl, bw = ctx.calibrate(total)
    hw = D.HwProfile(total, parts, fl, bw)
    pre = dict(q=[q for q, _ in wl.pre_seqs], c=[c for _, c in wl.pre_seqs], table=wl.pre_tables, x=x_pre, y=y_pre)
    dec = dict(c=wl.dec_ctx, table=wl.dec_tables, x=x_dec, y=y_dec)
    dec_batch = [(1, c, 2, 0) for c in wl.dec_ctx]
    pre_batch = [(q, c, 0 if c == 0 else 1, 0) for q, c in wl.pre_seqs]

    def run(side, sms_dec):
        split = (D.split_struct(D.DUET_MODE_TEMPORAL, total, 0, 1) if sms_dec is None
                 else D.split_struct(D.DUET_MODE_SPATIAL, total - sms_dec, sms_dec, 1))
        p_, d_ = (pre, None) if side == "prefill" else (None, dec)
        for _ in range(3):
            ctx.step(W, p_, d_, Kp, Vp, wl.n_pages, split)
        torch.cuda.synchronize()
        ctx.profile_enable(True)
        ts = []
        for _ in range(args.reps):
            ctx.step(W, p_, d_, Kp, Vp, wl.n_pages, split)
            torch.cuda.synchronize()
            t = ctx.last_step_times()
            ts.append(t["t_prefill"] if side == "prefill" else t["t_decode"])
        st = ctx.profile_read()
        ctx.profile_enable(False)
        ts.sort()
        return ts[len(ts) // 2], {k: {"s_per_launch": v["seconds"] / max(1, v["launches"]),
                                      "tflops": v["flops"] / v["seconds"] / 1e12 if v["seconds"] else None,
                                      "gbs": v["bytes"] / v["seconds"] / 1e9 if v["seconds"] else None}
                                  for k, v in st.items() if v["launches"]}

    rows = []
    dec_sizes = [s for s in parts if s in (8, 16, 24, 32, 48, 64, 96, 128, 144)] + [None]
    pre_sizes = [s for s in parts if s in (8, 16, 32, 64)] + [None]
    if args.only == "decode":
        dec_sizes, pre_sizes = ([args.sd] if args.sd else dec_sizes), []
    elif args.only == "prefill":
        dec_sizes, pre_sizes = [], ([args.sd] if args.sd else pre_sizes)
    for sd in dec_sizes:
        S = total if sd is None else sd
        t_meas, ks = run("decode", sd)
        t_pred = D.duet_predict_latency(spec, hw, dec_batch, S)["t_total"]
        rows.append({"side": "decode", "sms": S, "t_meas_ms": t_meas * 1e3, "t_roofline_ms": t_pred * 1e3,
                     "frac_of_roofline": t_pred / t_meas, "Pi_TFs": fl[S] / 1e12, "B_GBs": bw[S] / 1e9,
                     "kernels": ks})
        print(json.dumps(rows[-1]), flush=True)
    for sd in pre_sizes:
        S = total if sd is None else total - sd
        t_meas, ks = run("prefill", sd)
        t_pred = D.duet_predict_latency(spec, hw, pre_batch, S)["t_total"]
        rows.append({"side": "prefill", "sms": S, "t_meas_ms": t_meas * 1e3, "t_roofline_ms": t_pred * 1e3,
                     "frac_of_roofline": t_pred / t_meas, "Pi_TFs": fl[S] / 1e12, "B_GBs": bw[S] / 1e9,
                     "kernels": ks})
        print(json.dumps(rows[-1]), flush=True)
    doc = {"config": args.config, "rows": rows,
           "note": "frac_of_roofline = predicted roofline time (Sigma_op max(F/Pi(S), B/B(S)), paper §4.1 with the "
                   "measured tables) / measured side time; kernels: per-class achieved TFLOP/s and GB/s from events"}
    if args.out:
        with open(args.out, "w") as f:
            json.dump(doc, f, indent=1)
    ctx.close()


if __name__ == "__main__":
    main()

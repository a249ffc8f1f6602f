#!/usr/bin/env python
"""Trace-driven serving loop (the paper's Fig. 8 static-vs-adaptive comparison).

A bursty synthetic trace (synth/trace.py: Mooncake-like prompt lengths, Gamma arrivals with CV 2) is
served by the library end to end on one B200: duet_sched_* forms every mixed iteration (decode-first
chunked prefill, KV pages with look-ahead reservation, capacity admission), the policy picks the mode,
duet_step runs it, duet_sched_commit advances the requests.  Policies:
  static    every iteration temporal (aggregated, one stream)
  static_slo  temporal with the token budget cut until the predicted iteration meets tau (chunked
            prefill at the SLO, the conventional alternative)
  adaptive  Alg. 1 (duet_choose_split against the calibrated tables; spatial with k look-ahead steps
            when t_mixed > tau)
Simulated time advances by each iteration's measured GPU window.  Reports tokens/s, the inter-token gap
(TBT) distribution — a spatial window's last gap includes the wait for the prefill side to join — and
the SLO attainment.  Inputs are synthetic (values do not matter for
timing; KV pages start zeroed).

usage: python tools/trace_bench.py [--model cfg4] [--n-req 24] [--qps 2] [--layers 8] [--max-iters 300]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--n-req", type=int, default=24)
    ap.add_argument("--qps", type=float, default=2.0)
    ap.add_argument("--layers", type=int, default=8, help="Qwen2.5-14B slice depth")
    ap.add_argument("--tau", type=float, default=None, help="TBT SLO per iteration (s); default 100 ms x layers/48")
    ap.add_argument("--max-iters", type=int, default=300)
    ap.add_argument("--policies", default="static,static_slo,adaptive")
    ap.add_argument("--seed", type=int, default=4795)
    ap.add_argument("--out", default=None)
    ap.add_argument("--calibration", default="corun", choices=["corun", "burst"],
                    help="Pi_SM / B_HBM tables: under co-run at sustained clocks (bench default) or short bursts")
    ap.add_argument("--no-graph", action="store_true", help="decode steps launched eagerly (no CUDA graphs)")
    args = ap.parse_args()
    import numpy as np
    import torch
    from dataclasses import replace
    import paper_2511_04791_b200 as D
    from synth import configs
    from synth.gpu import layer_weights_gpu
    from synth.trace import bursty_trace

    m = replace(configs.QWEN25_14B, n_layers=args.layers)
    tau = args.tau if args.tau is not None else 0.1 * args.layers / 48
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(0)
    tdt = torch.bfloat16
    budget, max_batch, max_seqs, k_max, P = 8192, 64, 16, 8, 16
    trace = bursty_trace(args.n_req, args.qps, args.seed)
    max_pages = -(-(max(p + o for _, p, o, _ in trace) + k_max) // P)
    n_pages = sum(-(-(p + o + k_max) // P) for _, p, o, _ in trace) + 64   # room for the whole trace
    W = [layer_weights_gpu(m, l, 4791 + 4, dev, tdt) for l in range(m.n_layers)]
    shape = (n_pages, m.n_kv_heads, P, m.head_dim)
    Kp = [torch.zeros(shape, dtype=tdt, device=dev) for _ in range(m.n_layers)]
    Vp = [torch.zeros(shape, dtype=tdt, device=dev) for _ in range(m.n_layers)]
    xbuf = torch.randn((budget + max_batch, m.d_model), device=dev).to(tdt)
    ybuf = torch.empty((budget, m.d_model), dtype=tdt, device=dev)
    ydec = torch.empty((k_max, max_batch, m.d_model), dtype=tdt, device=dev)
    spec = D.make_spec(m.n_layers, m.d_model, m.ffn_dim, m.n_q_heads, m.n_kv_heads, m.head_dim, m.vocab, 2, 1,
                       int(m.qkv_bias), 1, m.rope_theta, m.norm_eps)
    ctx = D.Ctx(spec, budget, max_seqs, max_batch, k_max, max_pages, max_pages * P + 16, D.DUET_DTYPE_BF16,
                D.DUET_CTX_NO_GRAPH if args.no_graph else 0)
    parts, total = ctx.partitions()
    fl, bw = ctx.calibrate(total) if args.calibration == "burst" else ctx.calibrate_corun(total, 0.2)
    hw = D.HwProfile(total, parts, fl, bw)
    results = {}
    # static_slo: the conventional fix for TBT under chunked prefill — a temporal-only
    # server whose token budget is cut to the largest power of two for which the predicted mixed
    # iteration (that many prompt tokens at the trace's mean prompt length + a full decode batch at it)
    # meets tau
    mean_isl = int(np.mean([p for _, p, _, _ in trace]))
    slo_budget = 256
    for b_ in (8192, 4096, 2048, 1024, 512, 256):
        b_batch = [(b_, mean_isl // 2, 1, 0)] + [(1, mean_isl, 2, 0)] * max_batch
        if D.duet_predict_latency(spec, hw, b_batch, total, 0)["t_total"] <= tau:
            slo_budget = b_
            break
    for policy in args.policies.split(","):
        sched = D.Sched(page_size=P, n_pages=n_pages, token_budget=slo_budget if policy == "static_slo" else budget,
                        max_batch=max_batch,
                        max_prefill_seqs=max_seqs, k_max=k_max, max_pages_per_seq=max_pages)
        for r in trace:
            sched.add(*r)
        now, gpu_s, tokens, iters = 0.0, 0.0, 0, 0
        tbt, modes = [], {"temporal": 0, "spatial": 0}
        t_wall = time.perf_counter()
        while iters < args.max_iters:
            it = sched.next(now)
            if not it["prefill"] and not it["decode"]:
                if it["unfinished"] == 0 or it["next_arrival"] < 0:
                    break
                now = max(now, it["next_arrival"])
                continue
            n_pre, n_dec = len(it["prefill"]), len(it["decode"])
            tab = it["table"]
            rows = sum(q for _, q, _ in it["prefill"])
            pre = None
            if n_pre:
                pre = dict(q=[q for _, q, _ in it["prefill"]], c=[c for _, _, c in it["prefill"]],
                           table=np.ascontiguousarray(tab[:n_pre]), x=xbuf[:rows], y=ybuf[:rows])
            batch = [(q, c, 0 if c == 0 else 1, 0) for _, q, c in it["prefill"]] + \
                [(1, c, 2, 0) for _, c in it["decode"]]
            if policy in ("static", "static_slo"):
                split = D.split_struct(D.DUET_MODE_TEMPORAL, total, 0, 1)
            else:
                split = D.duet_choose_split(spec, hw, batch, tau, k_max, 0)
            k = split.k if split.mode == D.DUET_MODE_SPATIAL else 1
            dec = None
            if n_dec:
                dec = dict(c=[c for _, c in it["decode"]], table=np.ascontiguousarray(tab[n_pre:]),
                           x=xbuf[budget:budget + n_dec], y=ydec[:k, :n_dec])
            ctx.step(W, pre, dec, Kp, Vp, n_pages, split)
            torch.cuda.synchronize()
            st = ctx.last_step_times()
            window = st["t_window"]
            if n_dec:   # inter-token gaps seen by the running requests: in a spatial window k - 1 gaps of
                # t_decode / k, and the last token also waits for the prefill side to join (the next window
                # cannot start before it) — that stall is charged to the window's last gap
                if split.mode == D.DUET_MODE_SPATIAL:
                    g = st["t_decode"] / k
                    tbt.extend([g] * (k - 1) + [g + max(0.0, window - st["t_decode"])])
                else:
                    tbt.append(window)
            modes["spatial" if split.mode == D.DUET_MODE_SPATIAL else "temporal"] += 1
            toks, _ = sched.commit(k)
            tokens += toks
            gpu_s += window
            now += window
            iters += 1
        sched.close()
        tb = np.array(tbt) if tbt else np.zeros(1)
        results[policy] = {
            "iterations": iters, "tokens": tokens, "gpu_s": gpu_s, "tokens_per_s": tokens / max(gpu_s, 1e-9),
            "tbt_ms_p50": float(np.percentile(tb, 50) * 1e3), "tbt_ms_p90": float(np.percentile(tb, 90) * 1e3),
            "tbt_ms_p99": float(np.percentile(tb, 99) * 1e3), "slo_attainment": float(np.mean(tb <= tau)),
            "modes": modes, "wall_s": time.perf_counter() - t_wall,
            "token_budget": slo_budget if policy == "static_slo" else budget}
        print(policy, json.dumps(results[policy]), flush=True)
    out = {"model": f"qwen2.5-14b x{m.n_layers} layers", "tau_ms": tau * 1e3, "calibration": args.calibration, "n_req": args.n_req, "qps": args.qps,
           "trace": "lognormal ISL mean 12035 / OSL mean 343 (sigma 1), Gamma arrivals CV 2", "results": results}
    print(json.dumps(out))
    if args.out:
        json.dump(out, open(args.out, "w"), indent=1)
    ctx.close()


if __name__ == "__main__":
    main()

#!/usr/bin/env python
"""Render the `comparison.sweep` of bench.py --sweep lines as the Fig. 7 / Fig. 8 style markdown table
(every achievable S_d with Alg. 1's k rule: measured vs predicted t_d, t_p, window, tokens/s, TBT; the
optimizer's pick marked).

usage: python tools/render_sweep.py profiles/r02_bench_cfg3_sweep_X.json [...] > profiles/r02_sweep_cfg3_X.md
"""
import json
import sys


def render(path):
    d = json.load(open(path))
    c = d["comparison"]
    ch = c.get("aggregated_chunked_at_slo", {}).get("tok_s", 0)
    ag = c.get("aggregated", {}).get("tok_s", 0)
    out = [f"## {path} — optimizer pick S_d = {d['config']['s_d']}, k = {d['config']['k']}; chunked-at-SLO "
           f"{ch / 1e3:.1f} K tokens/s, aggregated {ag / 1e3:.1f} K", "",
           "| S_d | S_p | k | t_d meas / pred (ms) | t_p meas / pred (ms) | window meas / pred (ms) | tokens/s meas / pred "
           "| per-step TBT median (ms) | TBT max (ms) | SM MHz | pick |",
           "|---|---|---|---|---|---|---|---|---|---|---|"]
    for r in c["sweep"]:
        k = r["k"]
        out.append(f"| {r['s_d']} | {r['s_p']} | {k} | {r['t_decode_ms'] / k:.1f} / {r['t_pred_d_ms']:.1f} | "
                   f"{r['t_prefill_ms']:.1f} / {r['t_pred_p_ms']:.1f} | {r['window_ms']:.1f} / {r['t_pred_window_ms']:.1f} | "
                   f"{r['tok_s'] / 1e3:.1f} K / {r['predicted_tok_s'] / 1e3:.1f} K | {r.get('tbt_median_ms', 0):.1f} | "
                   f"{r.get('tbt_max_ms', 0):.1f} | {r.get('sm_mhz')} | {'**pick**' if r.get('optimizer_pick') else ''} |")
    return "\n".join(out)


if __name__ == "__main__":
    print("# cfg3 split sweep (Fig. 7 / Fig. 8 style): every achievable S_d with Alg. 1's k rule, measured vs predicted")
    print("# (bench.py --sweep; co-run + smoothed calibration tables, readings R-f / R-g; one B200, power-capped)\n")
    for p in sys.argv[1:]:
        print(render(p) + "\n")

#!/usr/bin/env python
"""Decode attention alone (duet_op_decode_attn: split-K + LSE combine, exactly as duet_step launches it)
on S-SM green-context partitions: achieved HBM GB/s (algorithmic bytes: every K/V page of every request
read once + q + o) per kernel variant, for the cfg2 batch (64 decodes at 4k) and the cfg3 batch (256
decodes, contexts 2k-8k), one layer.  Each variant runs in its own process (DUET_DECODE is read once).

usage: python tools/decode_attn_bench.py [--variants cp4x2,hy4x3] [--sms 16,32,48,148] [--out f.json]
"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def child(args):
    import numpy as np
    import torch
    import paper_2511_04791_b200 as D
    from synth import configs, counter_values_torch, page_tables
    m = configs.get_config("cfg2").model
    hq, hkv, dh = m.n_q_heads, m.n_kv_heads, m.head_dim
    batches = {"cfg2": [4096] * 64, "cfg3": [2048 + (6144 * r) // 255 for r in range(256)]}
    spec = D.make_spec(1, m.d_model, m.ffn_dim, hq, hkv, dh, m.vocab, 2, 1, 0, 1, m.rope_theta, m.norm_eps)
    ctx = D.Ctx(spec, 16, 1, 256, 1, 520, 8300, D.DUET_DTYPE_BF16)
    parts, total = ctx.partitions()
    out = []
    for name, pos in batches.items():
        n = len(pos)
        need = [p + 1 for p in pos]
        n_pages = sum((t + 15) // 16 for t in need) + 8
        tab, _ = page_tables(4791, need, 16, n_pages)
        Kp = counter_values_torch(1, 42, (n_pages, hkv, 16, dh), device="cuda", dtype=torch.bfloat16)
        Vp = counter_values_torch(1, 43, (n_pages, hkv, 16, dh), device="cuda", dtype=torch.bfloat16)
        q = counter_values_torch(1, 41, (n, hq * dh), device="cuda", dtype=torch.bfloat16)
        o = torch.empty_like(q)
        bytes_ = sum(2 * hkv * dh * t * 2 for t in need) + 2 * n * hq * dh * 2
        for S in args.sms:
            s_d = 0 if S >= total else S
            if s_d and s_d not in parts:
                continue
            for _ in range(3):
                ctx.op_decode_attn(q, o, pos, tab, Kp, Vp, n_pages, s_d=s_d)
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            reps = 10
            a.record()
            for _ in range(reps):
                ctx.op_decode_attn(q, o, pos, tab, Kp, Vp, n_pages, s_d=s_d)
            b.record()
            torch.cuda.synchronize()
            t = a.elapsed_time(b) / reps * 1e-3
            sms = s_d or total
            out.append({"batch": name, "sms": sms, "us": t * 1e6, "gbs": bytes_ / t / 1e9,
                        "gbs_per_sm": bytes_ / t / 1e9 / sms})
        del Kp, Vp
        torch.cuda.empty_cache()
    ctx.close()
    print(json.dumps(out))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--variants", default="cp4x2,hy4x3")
    ap.add_argument("--sms", default="16,24,32,48,64,148")
    ap.add_argument("--out", default=None)
    ap.add_argument("--child", action="store_true")
    args = ap.parse_args()
    args.sms = [int(x) for x in args.sms.split(",")]
    if args.child:
        child(args)
        return
    res = {}
    for v in args.variants.split(","):
        env = dict(os.environ, DUET_DECODE=v)
        r = subprocess.run([sys.executable, __file__, "--child", "--sms", ",".join(map(str, args.sms))], env=env,
                           capture_output=True, text=True, timeout=900)
        if r.returncode != 0:
            res[v] = {"error": r.stderr[-2000:]}
            print(v, "FAILED", r.stderr[-1500:], flush=True)
            continue
        res[v] = json.loads(r.stdout.strip().splitlines()[-1])
        for row in res[v]:
            print(f"{v:10s} {row['batch']} S={row['sms']:3d} {row['us']:9.1f} us {row['gbs']:7.0f} GB/s "
                  f"{row['gbs_per_sm']:6.1f} GB/s/SM", flush=True)
    if args.out:
        json.dump(res, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()

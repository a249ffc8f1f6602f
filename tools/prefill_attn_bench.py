#!/usr/bin/env python
"""Causal prefill attention alone (duet_op_prefill_attn, exactly as duet_step launches it) on the full
device and on S-SM partitions: achieved causal TFLOP/s (algorithmic: 4 d_h per visible (query, key) pair
per query head) per kernel variant, for the cfg2 chunk (q = 2048, no prefix), a cfg2 chunk
over a 2048-token prefix and the cfg3 prompt (q = 8192), one layer.  Each variant runs in its own process
(the DUET_* switches are read once).

usage: python tools/prefill_attn_bench.py [--variants EMU=0,EMU=3] [--sms 84,148] [--out f.json]
  a variant is a comma-free list of ENV=VALUE pairs joined by '+', e.g. DUET_FA_EMU=3
"""
import argparse
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def child(args):
    import torch
    import paper_2511_04791_b200 as D
    from synth import configs, counter_values_torch, page_tables
    m = configs.get_config("cfg2").model
    hq, hkv, dh = m.n_q_heads, m.n_kv_heads, m.head_dim
    cases = {"q2048": (2048, 0), "q2048_c2048": (2048, 2048), "q8192": (8192, 0)}
    spec = D.make_spec(1, m.d_model, m.ffn_dim, hq, hkv, dh, m.vocab, 2, 1, 0, 1, m.rope_theta, m.norm_eps)
    ctx = D.Ctx(spec, 8192, 1, 1, 1, 520, 8300 + 2048, D.DUET_DTYPE_BF16)
    parts, total = ctx.partitions()
    out = []
    for name, (q, c) in cases.items():
        need = [q + c]
        n_pages = (q + c + 15) // 16 + 8
        tab, _ = page_tables(4791, need, 16, n_pages)
        Kp = counter_values_torch(1, 42, (n_pages, hkv, 16, dh), device="cuda", dtype=torch.bfloat16)
        Vp = counter_values_torch(1, 43, (n_pages, hkv, 16, dh), device="cuda", dtype=torch.bfloat16)
        x = counter_values_torch(1, 41, (q, hq * dh), device="cuda", dtype=torch.bfloat16)
        o = torch.empty_like(x)
        pairs = sum(c + i + 1 for i in range(q))
        flops = 4.0 * dh * hq * pairs
        for S in args.sms:
            s_p = 0 if S >= total else S
            if s_p and (total - s_p) not in parts:
                continue
            for _ in range(3):
                ctx.op_prefill_attn(x, o, [q], [c], tab, Kp, Vp, n_pages, s_p=s_p)
            torch.cuda.synchronize()
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            reps = 10
            a.record()
            for _ in range(reps):
                ctx.op_prefill_attn(x, o, [q], [c], tab, Kp, Vp, n_pages, s_p=s_p)
            b.record()
            torch.cuda.synchronize()
            t = a.elapsed_time(b) / reps * 1e-3
            sms = s_p or total
            out.append({"case": name, "sms": sms, "us": t * 1e6, "tflops": flops / t / 1e12,
                        "tflops_per_sm": flops / t / 1e12 / sms})
        del Kp, Vp
        torch.cuda.empty_cache()
    ctx.close()
    print(json.dumps(out))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--variants", default="DUET_FA_EMU=0,DUET_FA_EMU=3")
    ap.add_argument("--sms", default="84,148")
    ap.add_argument("--out", default=None)
    ap.add_argument("--child", action="store_true")
    args = ap.parse_args()
    args.sms = [int(x) for x in args.sms.split(",")]
    if args.child:
        child(args)
        return
    res = {}
    for v in args.variants.split(","):
        env = dict(os.environ)
        for kv in v.split("+"):
            if kv:
                k, val = kv.split("=")
                env[k] = val
        r = subprocess.run([sys.executable, __file__, "--child", "--sms", ",".join(map(str, args.sms))], env=env,
                           capture_output=True, text=True, timeout=900)
        if r.returncode != 0:
            res[v] = {"error": r.stderr[-2000:]}
            print(v, "FAILED", r.stderr[-1500:], flush=True)
            continue
        res[v] = json.loads(r.stdout.strip().splitlines()[-1])
        for row in res[v]:
            print(f"{v:24s} {row['case']:12s} S={row['sms']:3d} {row['us']:9.1f} us {row['tflops']:7.1f} TFLOP/s "
                  f"{row['tflops_per_sm']:6.2f} /SM", flush=True)
    if args.out:
        json.dump(res, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()

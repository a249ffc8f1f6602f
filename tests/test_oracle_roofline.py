"""Pins for oracle/roofline.py (CPU only).

* SPEC.md worked examples re-derived by hand;
* closed forms of each predictor term on a hand-built batch;
* invariants of S:181-187 (monotonicity, decomposition, Jensen per-request max, N = 1 consistency);
* Alg. 1 == exhaustive search over every (S_d, k) on >= 1000 random instances;
* gate / clamp / infeasible / degenerate semantics;
* the paper's qualitative anchors: attention ~25% of a single 8192-token prefill,
  > 4x decode-latency spread with context, 8192-token prefill forces spatial mode.
"""
import math
import random

import pytest

from oracle import roofline as R

QWEN3_8B = R.Spec(n_layers=36, d_model=4096, ffn_dim=12288, n_q_heads=32, n_kv_heads=8, head_dim=128,
                  vocab=151936, elem_bytes=2)


def test_spec_worked_examples():
    assert R.linear_cost(2, 4, 8, 2) == (128, 112)
    assert R.linear_cost(0, 4, 8, 2) == (0, 64)
    assert R.linear_cost(8192, 4096, 4096, 2)[0] == 274877906944
    assert R.roofline_time(1000, 100, 1e12, 1e12) == 1e-9
    assert R.roofline_time(0, 0, 1e12, 1e12) == 0.0
    assert R.attention_cost(1, 3, 2, 1, 4, 2) == (144, 96)
    assert R.attention_cost(1, 1023, 32, 8, 128, 2) == (16842752, 4210688)
    t = R.allreduce_time(2, 10 ** 6, 3e-6, 4.5e11, 1e12)
    assert abs(t - (6e-6 + 2.0 / 900.0 * 1e-3 + 2e-6)) < 1e-18
    assert abs(t - 1.0222222222222222e-05) < 1e-18
    assert R.allreduce_time(1, 12345, 3e-6, 4.5e11, 1e12) == 0.0
    with pytest.raises(R.ConfigError):
        R.allreduce_time(0, 1, 3e-6, 4.5e11, 1e12)
    with pytest.raises(R.ConfigError):
        R.roofline_time(1, 1, 0.0, 1.0)
    prof = R.h100_like_profile()
    assert abs(prof.bw_at_sms[round(0.2 * 132)] / 3.35e12 - (round(0.2 * 132) / 132) ** 0.32) < 1e-15
    assert abs(0.2 ** 0.32 - 0.5975) < 1e-4


def _flat_profile(S=8, pi=1e12, bw=1e11):
    return R.Profile(S, tuple(range(1, S)), tuple([0.0] + [pi] * S), tuple([0.0] + [bw] * S))


def test_predict_closed_form_terms():
    sp = R.Spec(n_layers=3, d_model=64, ffn_dim=96, n_q_heads=4, n_kv_heads=2, head_dim=16, vocab=100,
                elem_bytes=2)
    prof = _flat_profile()
    batch = [R.Req(5, 0, R.PHASE_PREFILL_FULL, 1), R.Req(1, 20, R.PHASE_DECODE, 1)]
    out = R.predict(sp, prof, batch, 8, include_cls=True)
    n, d, s, pi, bw = 6, 64, 2, 1e12, 1e11
    mx = lambda F, B: max(F / pi, B / bw)
    qkv = mx(2 * n * d * 128, (n * d + d * 128 + n * 128) * s)
    o = mx(2 * n * 64 * d, (n * 64 + 64 * d + n * d) * s)
    gu = mx(2 * n * d * 192, (n * d + d * 192 + n * 192) * s)
    dn = mx(2 * n * 96 * d, (n * 96 + 96 * d + n * d) * s)
    assert out["t_linear"] == ((qkv + o) + gu) + dn
    nrm = mx(5 * n * d, 2 * n * d * s)
    act = mx(2 * n * 96, 3 * n * 96 * s)
    assert out["t_norm_act"] == (nrm + nrm) + act
    a1 = mx(4 * 4 * 5 * 5 * 16 + 2 * 4 * 5 * 5, 2 * 4 * 5 * 16 * s + 2 * 2 * 5 * 16 * s)
    a2 = mx(4 * 4 * 1 * 21 * 16 + 2 * 4 * 1 * 21, 2 * 4 * 1 * 16 * s + 2 * 2 * 21 * 16 * s)
    assert out["t_attn"] == (0.0 + a1) + a2
    assert out["t_cls"] == mx(2 * 2 * d * 100, (2 * d + d * 100 + 2 * 100) * s)
    assert out["t_total"] == 3.0 * out["t_block"] + out["t_cls"]


def test_predict_invariants():
    rnd = random.Random(5)
    base = R.h100_like_profile()
    for _ in range(200):
        batch = _rand_batch(rnd)
        for sms in (2, 40, 132):
            o = R.predict(QWEN3_8B, base, batch, sms)
            assert o["t_total"] == float(QWEN3_8B.n_layers) * o["t_block"] + o["t_cls"]   # decomposition
            assert o["t_block"] == ((o["t_linear"] + o["t_norm_act"]) + o["t_attn"]) + o["t_allreduce"]
            # Jensen: per-request max >= roofline of the summed attention cost
            F = sum(R.attention_cost(r.q, r.c, 32, 8, 128, 2)[0] for r in batch)
            B = sum(R.attention_cost(r.q, r.c, 32, 8, 128, 2)[1] for r in batch)
            pi, bw = base.flops_at_sms[sms], base.bw_at_sms[sms]
            assert o["t_attn"] >= R.roofline_time(F, B, pi, bw) * (1 - 1e-12)
    # monotone non-increasing in pi and bw; non-decreasing in q and c
    batch = [R.Req(300, 0, 0), R.Req(1, 900, 2)]
    fl = list(base.flops_at_sms)
    bw = list(base.bw_at_sms)
    t0 = R.predict(QWEN3_8B, base, batch, 50)["t_total"]
    fl2 = fl[:]
    fl2[50] *= 2
    bw2 = bw[:]
    bw2[50] *= 2
    p2 = R.Profile(base.total_sms, base.cand_sd_sms, tuple(fl2), tuple(bw))
    p3 = R.Profile(base.total_sms, base.cand_sd_sms, tuple(fl), tuple(bw2))
    assert R.predict(QWEN3_8B, p2, batch, 50)["t_total"] <= t0
    assert R.predict(QWEN3_8B, p3, batch, 50)["t_total"] <= t0
    assert R.predict(QWEN3_8B, base, [R.Req(301, 0, 0), R.Req(1, 900, 2)], 50)["t_total"] >= t0
    assert R.predict(QWEN3_8B, base, [R.Req(300, 0, 0), R.Req(1, 901, 2)], 50)["t_total"] >= t0
    # empty batch -> all zeros
    assert all(v == 0.0 for v in R.predict(QWEN3_8B, base, [], 10).values())


def test_tp_shards_and_allreduce_terms():
    sp1 = R.Spec(1, 8192, 28672, 64, 8, 128, 128256, 2, True, 1)
    sp2 = R.Spec(1, 8192, 28672, 64, 8, 128, 128256, 2, True, 2)
    prof = R.h100_like_profile()
    batch = [R.Req(1024, 0, 0)]
    o1 = R.predict(sp1, prof, batch, 132)
    o2 = R.predict(sp2, prof, batch, 132)
    assert o1["t_allreduce"] == 0.0
    ar = R.allreduce_time(2, 1024 * 8192 * 2, prof.allreduce_alpha, prof.nvlink_bw, prof.flops_at_sms[132])
    assert o2["t_allreduce"] == 2.0 * ar
    # compute-bound linear work halves under TP=2 (qkv, o, gate-up, down are all compute-bound at n=1024 on H100)
    assert abs(o2["t_linear"] / o1["t_linear"] - 0.5) < 0.02
    with pytest.raises(R.ConfigError):
        R.predict(R.Spec(1, 8192, 28672, 64, 8, 128, 128256, 2, True, 3), prof, batch, 132)


def test_validation_errors():
    prof = R.h100_like_profile()
    with pytest.raises(R.RangeError):
        R.predict(QWEN3_8B, prof, [R.Req(2, 5, R.PHASE_DECODE)], 10)         # decode needs q = 1
    with pytest.raises(R.RangeError):
        R.predict(QWEN3_8B, prof, [R.Req(4, 0, R.PHASE_PREFILL_CHUNK)], 10)  # chunk needs c > 0
    with pytest.raises(R.RangeError):
        R.predict(QWEN3_8B, prof, [R.Req(1, 4, 2)], 0)                        # sms out of range
    with pytest.raises(R.RangeError):
        R.predict(QWEN3_8B, prof, [R.Req(1, 4, 2)], 133)


def test_toy_optimizer_example():
    """S=8, tau=10 ms, t_d=24/S_d ms, t_p=96/S_p ms, T_dec=16, T_pre=512 -> (5, 3, 2), rho=544/19.2."""
    t_d = lambda sd: 24.0 / sd
    t_p = lambda sp: 96.0 / sp
    rho, best = R.alg1_search(8, range(1, 8), 10.0, 64, t_d, t_p, 16, 512)
    assert best[:3] == (5, 3, 2)
    assert abs(rho - 544 / 19.2) < 1e-12
    rho_x, best_x = R.exhaustive_search(8, range(1, 8), 10.0, 64, t_d, t_p, 16, 512)
    assert best_x == best and rho_x == rho
    # k clamp: t_p <= t_d -> floor = 0 -> k = 1
    rho, best = R.alg1_search(8, range(1, 8), 100.0, 64, lambda sd: 50.0, lambda sp: 10.0, 4, 8)
    assert best[2] == 1


def _rand_batch(rnd):
    b = []
    for _ in range(rnd.randint(0, 4)):
        c = rnd.choice([0, 0, rnd.randint(1, 9000)])
        b.append(R.Req(rnd.randint(1, 9000), c, R.PHASE_PREFILL_FULL if c == 0 else R.PHASE_PREFILL_CHUNK))
    for _ in range(rnd.randint(0, 80)):
        b.append(R.Req(1, rnd.randint(1, 70000), R.PHASE_DECODE))
    rnd.shuffle(b)
    return b


def _rand_profile(rnd):
    S = rnd.choice([16, 66, 132, 148])
    peak_f = rnd.uniform(2e14, 2.5e15)
    peak_b = rnd.uniform(1e12, 8e12)
    ex = rnd.uniform(0.2, 1.0)
    fl = [0.0] + [peak_f * i / S * rnd.uniform(0.9, 1.0) for i in range(1, S + 1)]
    bw = [0.0] + [peak_b * (i / S) ** ex for i in range(1, S + 1)]
    step = rnd.choice([1, 2, 8])
    return R.Profile(S, tuple(range(step, S, step)), tuple(fl), tuple(bw))


def test_alg1_equals_exhaustive_1200_instances():
    rnd = random.Random(2511)
    n_spatial = n_inf = 0
    for i in range(1200):
        prof = _rand_profile(rnd)
        batch = _rand_batch(rnd)
        sp = R.Spec(rnd.choice([1, 4, 32]), 4096, 14336, 32, 8, 128, 128256, 2)
        tau = 10 ** rnd.uniform(-5, -0.5)
        k_max = rnd.choice([1, 4, 32, 64])
        opts = rnd.choice([0, R.OPT_FORCE_SPATIAL, R.OPT_VERBATIM_INFEASIBLE, R.OPT_BOUNDARY_TBT,
                           R.OPT_BOUNDARY_TBT | R.OPT_FORCE_SPATIAL])
        a = R.choose_split(sp, prof, batch, tau, k_max, opts)
        b = R.choose_split_exhaustive(sp, prof, batch, tau, k_max, opts)
        assert a == b, (i, a, b)
        n_spatial += a.mode == R.MODE_SPATIAL and not a.flags
        n_inf += bool(a.flags & R.FLAG_INFEASIBLE)
        # mode soundness and constraint safety
        if a.mode == R.MODE_SPATIAL:
            assert a.t_mixed > tau or opts & R.OPT_FORCE_SPATIAL
            if not a.flags:
                assert a.t_d <= tau and 1 <= a.k <= k_max and a.s_p + a.s_d == prof.total_sms
    assert n_spatial > 100 and n_inf > 20


def test_gate_equality_and_degenerate_and_infeasible():
    prof = _flat_profile()
    sp = R.Spec(1, 64, 96, 4, 2, 16, 100, 2)
    batch = [R.Req(50, 0, 0), R.Req(1, 100, 2)]
    t_mixed = R.predict(sp, prof, batch, 8)["t_total"]
    s = R.choose_split(sp, prof, batch, t_mixed)                             # equality -> temporal
    assert s.mode == R.MODE_TEMPORAL and s.flags == 0
    s = R.choose_split(sp, prof, batch, t_mixed * (1 - 1e-12))
    assert s.mode == R.MODE_SPATIAL
    s = R.choose_split(sp, prof, [R.Req(1, 100, 2)] * 3, 1e-12)              # decode only -> degenerate
    assert s.mode == R.MODE_TEMPORAL and s.flags == R.FLAG_DEGENERATE
    s = R.choose_split(sp, prof, batch, 1e-15)                               # infeasible
    assert s.flags == R.FLAG_INFEASIBLE and s.mode == R.MODE_SPATIAL
    assert s.s_d == 1                                                         # flat profile: first argmin


def test_infeasible_guard_reading_20b():
    """Reading #20b.  When no S_d meets tau both modes miss the SLO; the argmin-t_d spatial fallback
     is kept only if its throughput rho is not below the temporal batch's sum(q) / t_mixed.
    (1) A Llama-3-70B-shaped layer stack at TP = 1 (a 16k prefill + 512 decodes at 4k, tau = 5 ms) on a
    profile linear in FLOPs and saturating in bandwidth: every S_d misses tau, the verbatim fallback is
    the largest decode group with a sliver of SMs for the prefill, whose window is dominated by the
    starved prefill (the 16x loss measured in round 1) -> temporal, flagged.  (2) On the flat profile
    the fallback keeps its rho advantage -> spatial, flagged."""
    sp = R.Spec(8, 8192, 28672, 64, 8, 128, 128256, 2)
    S = 148
    prof = R.Profile(S, tuple(range(8, S, 8)), tuple([0.0] + [1.6e15 * i / S for i in range(1, S + 1)]),
                     tuple([0.0] + [6.5e12 * min(1.0, i / 40) for i in range(1, S + 1)]))
    batch = [R.Req(16384, 0, R.PHASE_PREFILL_FULL)] + [R.Req(1, 4096, R.PHASE_DECODE)] * 512
    verb = R.choose_split(sp, prof, batch, 5e-3, 32, R.OPT_VERBATIM_INFEASIBLE)
    assert verb.mode == R.MODE_SPATIAL and verb.flags == R.FLAG_INFEASIBLE
    # argmin t_d: the decode side's weight reads saturate the bandwidth at S_d >= 40, the remaining
    # compute terms keep falling with S_d, so the fallback is the largest candidate (144 of 148 SMs)
    assert verb.s_d == 144 and verb.s_p == 4
    rho_t = (512 + 16384) / verb.t_mixed
    assert verb.rho < rho_t / 4                    # the starved-prefill window: far worse throughput
    g = R.choose_split(sp, prof, batch, 5e-3, 32, 0)
    assert (g.mode, g.flags, g.s_p, g.s_d, g.k) == (R.MODE_TEMPORAL, R.FLAG_INFEASIBLE, S, 0, 1)
    assert g.rho == rho_t and g.t_mixed == verb.t_mixed
    assert R.choose_split_exhaustive(sp, prof, batch, 5e-3, 32, 0) == g
    # FORCE_SPATIAL still returns the (flagged) spatial fallback: forcing is the caller's explicit request
    assert R.choose_split(sp, prof, batch, 5e-3, 32, R.OPT_FORCE_SPATIAL).mode == R.MODE_SPATIAL
    # (2) flat profile: both sides run at the full rate concurrently, the fallback's rho wins
    prof2 = _flat_profile()
    sp2 = R.Spec(1, 64, 96, 4, 2, 16, 100, 2)
    b2 = [R.Req(50, 0, 0), R.Req(1, 100, 2)]
    s2 = R.choose_split(sp2, prof2, b2, 1e-15)
    assert s2.mode == R.MODE_SPATIAL and s2.flags == R.FLAG_INFEASIBLE
    assert s2.rho >= 51 / s2.t_mixed


def test_boundary_tbt_option_reading_23():
    """Reading #23 (opt-in).  The paper constrains only t_d <= tau; a decode token at a window
    boundary also waits for the prefill side, gap = t_d + max(0, t_p - k t_d).  On the SPEC toy (S = 8,
    t_d(S_d) = 24/S_d, t_p(S_p) = 96/S_p ms, T_dec = 16, T_pre = 512, tau = 10 ms) the verbatim
    winner (S_p, S_d, k) = (5, 3, 2) has a 19.2 - 16 + 8 = 11.2 ms boundary gap > tau.  With the option
    Alg. 1's two-candidate rule still finds the optimum (the k = floor(t_p/t_d) + 1 candidate never
    stalls), so it must equal the exhaustive search and a brute force written out below."""
    t_d_of = lambda S_d: 24.0 / S_d
    t_p_of = lambda S_p: 96.0 / S_p
    rho0, best0 = R.alg1_search(8, range(1, 8), 10.0, 64, t_d_of, t_p_of, 16, 512)
    assert best0[:3] == (5, 3, 2) and R.boundary_gap(2, 8.0, 19.2) > 10.0
    rho1, best1 = R.alg1_search(8, range(1, 8), 10.0, 64, t_d_of, t_p_of, 16, 512, boundary=True)
    rho2, best2 = R.exhaustive_search(8, range(1, 8), 10.0, 64, t_d_of, t_p_of, 16, 512, boundary=True)
    assert (rho1, best1) == (rho2, best2)
    S_p, S_d, k, t_p, t_d = best1
    assert R.boundary_gap(k, t_d, t_p) <= 10.0 and rho1 < rho0
    # brute force written out: every (S_d, k) with t_d <= tau and gap <= tau
    cands = []
    for sd in range(1, 8):
        td, tp = 24.0 / sd, 96.0 / (8 - sd)
        for kk in range(1, 65):
            if td <= 10.0 and td + max(0.0, tp - kk * td) <= 10.0:
                cands.append(((kk * 16 + 512) / max(kk * td, tp), -sd, -kk))
    top = max(cands)
    assert abs(top[0] - rho1) < 1e-12 and (-top[1], -top[2]) == (S_d, k)


def test_paper_qualitative_anchors():
    prof = R.h100_like_profile()
    # attention share of a single 8192-token prefill in [15%, 35%] ("approximately 25%")
    o = R.predict(QWEN3_8B, prof, [R.Req(8192, 0, 0)], 132)
    share = o["t_attn"] / o["t_block"]
    assert 0.15 <= share <= 0.35, share
    # decode batch of 8 at c = 2048 vs 65536: > 4x latency spread
    t1 = R.predict(QWEN3_8B, prof, [R.Req(1, 2048, 2)] * 8, 132)["t_total"]
    t2 = R.predict(QWEN3_8B, prof, [R.Req(1, 65536, 2)] * 8, 132)["t_total"]
    assert 4.0 <= t2 / t1 <= 7.0, t2 / t1
    # an 8192-token prefill in the mix exceeds a 100 ms TBT and forces spatial mode
    batch = [R.Req(8192, 0, 0)] + [R.Req(1, 8000, 2)] * 16
    assert R.predict(QWEN3_8B, prof, batch, 132)["t_total"] > 0.1
    s = R.choose_split(QWEN3_8B, prof, batch, 0.1)
    assert s.mode == R.MODE_SPATIAL and s.flags == 0 and s.t_d <= 0.1

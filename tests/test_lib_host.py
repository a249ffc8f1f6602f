"""libduet.so host side (no GPU needed): symbols, predictor and Alg. 1 bit-exact vs the oracle."""
import math
import random
import re
import os

import pytest
from hypothesis import given, settings, strategies as st

import paper_2511_04791_b200 as D
from oracle import roofline as R

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_library_loads_and_exports_every_declared_symbol():
    hdr = open(os.path.join(ROOT, "include", "duet.h")).read()
    declared = set(re.findall(r"\b(duet_[a-z_]+)\s*\(", hdr))
    assert {"duet_predict_latency", "duet_choose_split", "duet_step", "duet_ctx_create"} <= declared
    lib = D.lib()
    for name in sorted(declared):
        assert hasattr(lib, name), name
    assert set(D.EXPORTED) == declared
    assert lib.duet_abi_version() == 4


def _spec_pair(rnd):
    L = rnd.choice([1, 2, 32, 80])
    hkv = rnd.choice([1, 2, 4, 8])
    g = rnd.choice([1, 2, 4, 8])
    dh = rnd.choice([64, 128])
    hq = hkv * g
    tp = rnd.choice([t for t in (1, 2, 4, 8) if hq % t == 0 and hkv % t == 0])
    m = rnd.choice([1024, 14336, 28672]) * (1 if tp == 1 else 1)
    s = rnd.choice([1, 2, 4])
    gated = rnd.choice([True, True, False])
    vocab = rnd.choice([1000, 128256])
    o = R.Spec(L, hq * dh, m, hq, hkv, dh, vocab, s, gated, tp)
    c = D.make_spec(L, hq * dh, m, hq, hkv, dh, vocab, s, int(gated), 0, tp)
    return o, c


def _profile_pair(rnd):
    S = rnd.choice([16, 132, 148])
    pf = rnd.uniform(1e14, 2.5e15)
    pb = rnd.uniform(1e12, 8e12)
    ex = rnd.uniform(0.1, 1.0)
    fl = [0.0] + [pf * i / S * rnd.uniform(0.8, 1.0) for i in range(1, S + 1)]
    bw = [0.0] + [pb * (i / S) ** ex for i in range(1, S + 1)]
    step = rnd.choice([1, 2, 8])
    cand = list(range(step, S, step))
    a = rnd.uniform(1e-6, 1e-5)
    nv = rnd.uniform(1e11, 1e12)
    return R.Profile(S, tuple(cand), tuple(fl), tuple(bw), nv, a), D.HwProfile(S, cand, fl, bw, nv, a)


def _batch(rnd):
    b = []
    for _ in range(rnd.randint(0, 3)):
        c = rnd.choice([0, rnd.randint(1, 20000)])
        b.append((rnd.randint(1, 16384), c, 0 if c == 0 else 1, rnd.randint(0, 1)))
    for _ in range(rnd.randint(0, 300)):
        b.append((1, rnd.randint(1, 131072), 2, rnd.randint(0, 1)))
    rnd.shuffle(b)
    return b


def test_predict_bit_exact_vs_oracle():
    rnd = random.Random(11)
    for i in range(400):
        so, sc = _spec_pair(rnd)
        po, pc = _profile_pair(rnd)
        b = _batch(rnd)
        sms = rnd.randint(1, po.total_sms)
        incl = rnd.choice([0, D.DUET_OPT_INCLUDE_CLS])
        ref = R.predict(so, po, [R.Req(*e) for e in b], sms, bool(incl))
        got = D.duet_predict_latency(sc, pc, b, sms, incl)
        assert got == ref, (i, got, ref)          # bitwise-equal doubles


def test_choose_split_tuple_exact_vs_oracle_and_exhaustive():
    rnd = random.Random(12)
    kinds = set()
    for i in range(1500):
        so, sc = _spec_pair(rnd)
        po, pc = _profile_pair(rnd)
        b = _batch(rnd)
        tau = 10 ** rnd.uniform(-5, 0)
        kmax = rnd.choice([1, 8, 32])
        opts = rnd.choice([0, D.DUET_OPT_FORCE_SPATIAL, D.DUET_OPT_INCLUDE_CLS, D.DUET_OPT_VERBATIM_INFEASIBLE,
                           D.DUET_OPT_BOUNDARY_TBT, D.DUET_OPT_BOUNDARY_TBT | D.DUET_OPT_INCLUDE_CLS])
        reqs = [R.Req(*e) for e in b]
        ref = R.choose_split(so, po, reqs, tau, kmax, opts)
        got = D.duet_choose_split(sc, pc, b, tau, kmax, opts)
        assert D.split_tuple(got) == (ref.mode, ref.s_p, ref.s_d, ref.k, ref.flags, ref.t_mixed, ref.t_p, ref.t_d,
                                      ref.rho), i
        if i % 5 == 0:
            assert R.choose_split_exhaustive(so, po, reqs, tau, kmax, opts) == ref
        kinds.add((ref.mode, ref.flags))
    assert {(0, 0), (1, 0), (1, 1), (0, 2), (0, 1)} <= kinds   # (0, 1): the reading #20b guard


@settings(max_examples=300, deadline=None)
@given(st.integers(0, 2 ** 31 - 1))
def test_hypothesis_fuzz_split(seed):
    rnd = random.Random(seed)
    so, sc = _spec_pair(rnd)
    po, pc = _profile_pair(rnd)
    b = _batch(rnd)
    tau = 10 ** rnd.uniform(-6, 1)
    ref = R.choose_split(so, po, [R.Req(*e) for e in b], tau, 32, 0)
    got = D.duet_choose_split(sc, pc, b, tau, 32, 0)
    assert D.split_tuple(got) == (ref.mode, ref.s_p, ref.s_d, ref.k, ref.flags, ref.t_mixed, ref.t_p, ref.t_d,
                                  ref.rho)


def test_errors_are_flagged_with_messages():
    sc = D.make_spec(1, 4096, 14336, 32, 8, 128)
    pc = D.HwProfile(148, [8, 16], [0.0] + [1e15] * 148, [0.0] + [8e12] * 148)
    with pytest.raises(D.DuetError) as e:
        D.duet_predict_latency(sc, pc, [(2, 5, 2)], 10)
    assert e.value.status == -2 and "entry 0" in str(e.value)
    with pytest.raises(D.DuetError) as e:
        D.duet_predict_latency(sc, pc, [(1, 5, 2)], 149)
    assert e.value.status == -2 and "149" in str(e.value)
    bad = D.HwProfile(148, [8], [0.0] * 149, [0.0] + [8e12] * 148)
    with pytest.raises(D.DuetError) as e:
        D.duet_predict_latency(sc, bad, [(1, 5, 2)], 10)
    assert e.value.status == -3
    with pytest.raises(D.DuetError) as e:
        D.duet_predict_latency(D.make_spec(1, 4096, 14336, 32, 8, 128, tp=3), pc, [(1, 5, 2)], 10)
    assert e.value.status == -3
    with pytest.raises(D.DuetError) as e:
        D.duet_choose_split(sc, pc, [(1, 5, 2)], 0.0)
    assert e.value.status == -3
    assert D.duet_predict_latency(sc, pc, [], 10)["t_total"] == 0.0


def test_optimizer_speed_under_1ms():
    """S:502 / P:488: one Alg. 1 solve at 66 TPCs (132 SMs) with 64 requests stays under 1 ms."""
    import time
    rnd = random.Random(3)
    po, pc = _profile_pair(rnd)
    pc = D.HwProfile(132, list(range(2, 132, 2)), [0.0] + [1e15 * i / 132 for i in range(1, 133)],
                     [0.0] + [3e12 * (i / 132) ** 0.32 for i in range(1, 133)])
    sc = D.make_spec(36, 4096, 12288, 32, 8, 128)
    b = [(2048, 0, 0, 1)] + [(1, rnd.randint(100, 9000), 2, 1) for _ in range(63)]
    ts = []
    for _ in range(100):
        t = time.perf_counter()
        D.duet_choose_split(sc, pc, b, 1e-3, 32, D.DUET_OPT_FORCE_SPATIAL)
        ts.append(time.perf_counter() - t)
    ts.sort()
    assert ts[50] < 1e-3, ts[50]


def test_corun_choose_host_logic():
    """f4 co-run choice (duet_corun_choose): against a direct enumeration of the documented rule on random
    calibrated-looking tables, plus its limiting cases."""
    rnd = random.Random(21)
    S = 148
    cand = list(range(8, 148, 8))
    for _ in range(300):
        fa = [0.0] + [rnd.uniform(3e12, 5e12) * i for i in range(1, S + 1)]
        sat, s0 = rnd.uniform(4e12, 7e12), rnd.uniform(10, 50)
        bw = [0.0] + [sat * (1 - math.exp(-i / s0)) for i in range(1, S + 1)]
        F = 10 ** rnd.uniform(8, 12)
        B = 10 ** rnd.uniform(6, 10)
        ov = rnd.choice([0.0, 15e-6])
        sd, t = D.duet_corun_choose(S, cand, fa, bw, F, B, 16, ov)
        t_seq = F / fa[S] + B / bw[S]
        best, best_t = 0, t_seq - ov
        for c in cand:
            if c < 16 or S - c < 16:
                continue
            tc = max(F / fa[S - c], B / bw[c])
            if tc < best_t:
                best, best_t = c, tc
        assert sd == best
        assert t == (best_t if best else t_seq)
    # a phase absent or a tiny batch: never co-run
    fa = [0.0] + [4e12 * i for i in range(1, S + 1)]
    bw = [0.0] + [6e12 * min(1.0, i / 40) for i in range(1, S + 1)]
    assert D.duet_corun_choose(S, cand, fa, bw, 0.0, 1e9)[0] == 0
    assert D.duet_corun_choose(S, cand, fa, bw, 1e6, 1e4)[0] == 0       # << the 15 us fork/join cost
    # balanced large attentions (cfg2-like: 34 GFLOP causal, 1.07 GB of KV): co-run on a split
    sd, t = D.duet_corun_choose(S, cand, fa, bw, 34.4e9, 1.07e9)
    assert 16 <= sd <= 132 and t < 34.4e9 / fa[S] + 1.07e9 / bw[S]


def test_profile_smooth_median_of_three():
    """duet_profile_smooth (reading R-g): a lone outlier among the per-SM rates is replaced by the median
    of its neighbourhood, monotone runs and the end points are untouched, bad input is rejected."""
    sizes = [8, 16, 24, 32, 40, 148]
    per_sm = [10.0, 9.5, 9.0, 6.0, 8.5, 8.0]          # 32 SMs: one low outlier
    table = [0.0] * 149
    for s, r in zip(sizes, per_sm):
        table[s] = r * s
    out = D.duet_profile_smooth(sizes, table)
    got = [out[s] / s for s in sizes]
    assert got[0] == 10.0 and got[-1] == 8.0           # end points kept
    assert got[3] == 8.5                               # median(9.0, 6.0, 8.5)
    assert got[1] == 9.5 and got[2] == 9.0 and got[4] == 8.0  # median(6.0, 8.5, 8.0): computed on the raw rates
    assert all(out[s] == 0.0 for s in range(149) if s not in sizes)
    mono = [0.0] * 149
    for s, r in zip(sizes, [12.0, 11.0, 10.0, 9.0, 8.0, 5.0]):
        mono[s] = r * s
    assert D.duet_profile_smooth(sizes, mono) == mono  # a monotone run is a fixed point
    with pytest.raises(D.DuetError):
        D.duet_profile_smooth([16, 8], table)          # not ascending
    with pytest.raises(D.DuetError):
        D.duet_profile_smooth([8, 200], table)         # outside the table

"""Oracle: attention-aware roofline predictor (§4.1) and partition optimizer (§4.2, Alg. 1).

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).

Step-by-step transcription in the paper's notation, under the readings of
DESIGN.md.  All F and B are exact Python integers; a
latency is ``max(float(F)/Pi, float(B)/Bw)``; sums are taken in the
canonical order listed in ``predict`` so that the C++ library can be compared
bit-for-bit (Python floats are IEEE binary64 and never fuse).

Readings used here: #3 gated FFN (gate-up d_o = 2m), #4 GQA widths, #8 the
attention denominator B_SM read as B_HBM(S), #9 the attention FLOPs
verbatim (full q x (q+c) rectangle), #10 no decode KV-write bytes, #11 norm
F = 5nd, B = 2nds; act F = 2nm', B = 3nm's (plain: 2nm's), #12 t_cls over entries
that emit logits, #13 TP shards h_q, h_kv, m by N, #14 allreduce third term
verbatim, #16 S_d enumerated over the launcher's achievable list excluding
S_d = S, #17 k clamped to [1, k_max], #18 strict ">" (first found wins),
#19 temporal at equality, #20 infeasible fallback = argmin t_d, #20b the
infeasible spatial fallback is kept only when its rho is not below the temporal
rho (both violate tau; the paper's objective, throughput, decides), #21 a batch
missing one phase runs temporally, #23 (opt-in OPT_BOUNDARY_TBT) a candidate (S_d, k)
must also keep the window-boundary gap t_d + max(0, t_p - k t_d) within tau, #25 T_pre = sum q over prefill entries,
T_dec = number of decode entries.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

PHASE_PREFILL_FULL, PHASE_PREFILL_CHUNK, PHASE_DECODE = 0, 1, 2
OPT_FORCE_SPATIAL, OPT_INCLUDE_CLS, OPT_VERBATIM_INFEASIBLE, OPT_BOUNDARY_TBT = 1, 2, 4, 8
FLAG_INFEASIBLE, FLAG_DEGENERATE = 1, 2
MODE_TEMPORAL, MODE_SPATIAL = 0, 1


class ConfigError(ValueError):
    pass


class RangeError(ValueError):
    pass


@dataclass(frozen=True)
class Spec:
    n_layers: int
    d_model: int
    ffn_dim: int
    n_q_heads: int
    n_kv_heads: int
    head_dim: int
    vocab: int
    elem_bytes: int
    ffn_gated: bool = True
    tp: int = 1


@dataclass(frozen=True)
class Profile:
    total_sms: int
    cand_sd_sms: tuple          # ascending achievable S_d
    flops_at_sms: tuple         # [total_sms + 1] FLOP/s; index = SM count
    bw_at_sms: tuple            # [total_sms + 1] B/s
    nvlink_bw: float = 900e9
    allreduce_alpha: float = 3e-6


@dataclass(frozen=True)
class Req:
    q: int
    c: int
    phase: int
    emits_logits: int = 0


# ---------------------------------------------------------------- cost formulas

def linear_cost(n: int, d_i: int, d_o: int, s: int) -> tuple[int, int]:
    """F_lin = 2 n d_i d_o ;  B_lin = n d_i s + d_i d_o s + n d_o s."""
    return 2 * n * d_i * d_o, n * d_i * s + d_i * d_o * s + n * d_o * s


def roofline_time(F: int, B: int, pi: float, bw: float) -> float:
    """t = max(F / Pi_SM, B / B_HBM)."""
    if not (pi > 0) or not (bw > 0):
        raise ConfigError(f"non-positive throughput pi={pi} bw={bw}")
    tf = float(F) / pi
    tb = float(B) / bw
    return tb if tf < tb else tf


def attention_cost(q: int, c: int, hq: int, hkv: int, dh: int, s: int) -> tuple[int, int]:
    """F = 4 h_q q (q+c) d_h + 2 h_q q (q+c) ;  B = 2 h_q q d_h s + 2 h_kv (q+c) d_h s."""
    F = 4 * hq * q * (q + c) * dh + 2 * hq * q * (q + c)
    B = 2 * hq * q * dh * s + 2 * hkv * (q + c) * dh * s
    return F, B


def allreduce_time(N: int, B: int, alpha: float, b_nvl: float, pi: float) -> float:
    """t = 2(N-1) alpha + 2(N-1) B / (N B_NVLink) + N(N-1) B / Pi_SM."""
    if N < 1:
        raise ConfigError("N must be >= 1")
    if N == 1:
        return 0.0
    t1 = float(2 * (N - 1)) * alpha
    t2 = float(2 * (N - 1) * B) / (float(N) * b_nvl)
    t3 = float(N * (N - 1) * B) / pi
    return (t1 + t2) + t3


# ---------------------------------------------------------------- validation

def validate_spec(sp: Spec):
    for name in ("n_layers", "d_model", "ffn_dim", "n_q_heads", "n_kv_heads", "head_dim", "tp"):
        if getattr(sp, name) <= 0:
            raise ConfigError(f"{name} must be > 0")
    if sp.elem_bytes not in (1, 2, 4):
        raise ConfigError("elem_bytes must be 1, 2 or 4")
    if sp.n_q_heads % sp.n_kv_heads:
        raise ConfigError("n_q_heads must be a multiple of n_kv_heads")
    N = sp.tp
    if sp.n_q_heads % N or sp.n_kv_heads % N or sp.ffn_dim % N:
        raise ConfigError("tp must divide n_q_heads, n_kv_heads and ffn_dim")


def validate_req(i: int, r: Req):
    if r.phase == PHASE_DECODE:
        ok = r.q == 1 and r.c > 0
    elif r.phase == PHASE_PREFILL_FULL:
        ok = r.q >= 1 and r.c == 0
    elif r.phase == PHASE_PREFILL_CHUNK:
        ok = r.q >= 1 and r.c > 0
    else:
        ok = False
    if not ok:
        raise RangeError(f"batch entry {i}: (q={r.q}, c={r.c}, phase={r.phase}) violates its phase invariant")


def lookup(prof: Profile, sms: int) -> tuple[float, float]:
    if sms < 1 or sms > prof.total_sms:
        raise RangeError(f"sms={sms} outside [1, {prof.total_sms}]")
    pi, bw = prof.flops_at_sms[sms], prof.bw_at_sms[sms]
    if not (pi > 0) or not (bw > 0):
        raise ConfigError(f"profile at sms={sms} has non-positive pi={pi} or bw={bw}")
    return pi, bw


# ---------------------------------------------------------------- predictor

ZERO = dict(t_linear=0.0, t_norm_act=0.0, t_attn=0.0, t_allreduce=0.0, t_block=0.0, t_cls=0.0, t_total=0.0)


def predict(sp: Spec, prof: Profile, batch: list, sms: int, include_cls: bool = False) -> dict:
    """f_roofline(R, Pi_SM(S), B_HBM(S)) -> latency breakdown (§4.1; canonical order of C-4)."""
    validate_spec(sp)
    for i, r in enumerate(batch):
        validate_req(i, r)
    pi, bw = lookup(prof, sms)
    n = sum(r.q for r in batch)
    if n == 0:
        return dict(ZERO)
    N = sp.tp
    s = sp.elem_bytes
    d, dh = sp.d_model, sp.head_dim
    hq, hkv, m = sp.n_q_heads // N, sp.n_kv_heads // N, sp.ffn_dim // N
    # token-level operators, in order: norm1, qkv, o, norm2, gate_up, act, down
    t_norm1 = roofline_time(5 * n * d, 2 * n * d * s, pi, bw)
    t_qkv = roofline_time(*linear_cost(n, d, (hq + 2 * hkv) * dh, s), pi, bw)
    t_o = roofline_time(*linear_cost(n, hq * dh, d, s), pi, bw)
    t_norm2 = roofline_time(5 * n * d, 2 * n * d * s, pi, bw)
    if sp.ffn_gated:
        t_gu = roofline_time(*linear_cost(n, d, 2 * m, s), pi, bw)
        t_act = roofline_time(2 * n * m, 3 * n * m * s, pi, bw)
    else:
        t_gu = roofline_time(*linear_cost(n, d, m, s), pi, bw)
        t_act = roofline_time(2 * n * m, 2 * n * m * s, pi, bw)
    t_down = roofline_time(*linear_cost(n, m, d, s), pi, bw)
    t_linear = ((t_qkv + t_o) + t_gu) + t_down
    t_norm_act = (t_norm1 + t_norm2) + t_act
    # sequence-level operator: per-request max, then sum in batch order
    t_attn = 0.0
    for r in batch:
        t_attn += roofline_time(*attention_cost(r.q, r.c, hq, hkv, dh, s), pi, bw)
    # communication: two allreduces of the [n, d] output per block
    if N == 1:
        t_ar = 0.0
    else:
        t_ar = 2.0 * allreduce_time(N, n * d * s, prof.allreduce_alpha, prof.nvlink_bw, pi)
    t_block = ((t_linear + t_norm_act) + t_attn) + t_ar
    t_cls = 0.0
    if include_cls:
        n_cls = sum(1 for r in batch if r.emits_logits)
        if n_cls:
            t_cls = roofline_time(*linear_cost(n_cls, d, sp.vocab, s), pi, bw)
    t_total = float(sp.n_layers) * t_block + t_cls
    return dict(t_linear=t_linear, t_norm_act=t_norm_act, t_attn=t_attn, t_allreduce=t_ar,
                t_block=t_block, t_cls=t_cls, t_total=t_total)


# ---------------------------------------------------------------- optimizer

@dataclass(frozen=True)
class Split:
    mode: int
    s_p: int
    s_d: int
    k: int
    flags: int
    t_mixed: float
    t_p: float
    t_d: float
    rho: float


def _clamp_k(x: int, k_max: int) -> int:
    return min(max(x, 1), k_max)


def _phases(batch):
    P = [r for r in batch if r.phase != PHASE_DECODE]
    D = [r for r in batch if r.phase == PHASE_DECODE]
    return P, D


def _temporal(batch, t_mixed, flags, S):
    n = sum(r.q for r in batch)
    rho = float(n) / t_mixed if t_mixed > 0 else 0.0
    return Split(MODE_TEMPORAL, S, 0, 1, flags, t_mixed, t_mixed, t_mixed, rho)


def boundary_gap(k: int, t_d: float, t_p: float) -> float:
    """The inter-token gap across a window boundary (reading #23): the window's last decode step, plus
    the time its decodes wait for the prefill side to join, t_d + max(0, t_p - k t_d)."""
    return t_d + max(0.0, t_p - float(k) * t_d)


def alg1_search(S: int, cand, tau: float, k_max: int, t_d_of, t_p_of, T_dec: int, T_pre: int,
                boundary: bool = False):
    """Lines 7-21 of Algorithm 1 for given latency functions t_d(S_d), t_p(S_p).
    boundary (opt-in, reading #23): a (S_d, k) candidate must also keep the boundary gap <= tau.
    Returns (rho*, (S_p, S_d, k, t_p, t_d)) or (0.0, None) when no S_d meets tau."""
    rho_best, best = 0.0, None                                     # l.7
    for S_d in cand:                                               # l.8 (reading #16)
        if S_d >= S:
            continue
        t_d = t_d_of(S_d)                                          # l.9
        if t_d > tau:                                              # l.10-12
            continue
        S_p = S - S_d                                              # l.13
        t_p = t_p_of(S_p)                                          # l.14
        r = math.floor(t_p / t_d)
        for k in (_clamp_k(r, k_max), _clamp_k(r + 1, k_max)):    # l.15 (reading #17)
            if boundary and boundary_gap(k, t_d, t_p) > tau:
                continue
            rho = float(k * T_dec + T_pre) / max(float(k) * t_d, t_p)   # l.16
            if rho > rho_best:                                     # l.17-18 (reading #18)
                rho_best, best = rho, (S_p, S_d, k, t_p, t_d)
    return rho_best, best


def exhaustive_search(S: int, cand, tau: float, k_max: int, t_d_of, t_p_of, T_dec: int, T_pre: int,
                      boundary: bool = False):
    """Brute force over every (S_d in cand, k in [1, k_max]) with t_d <= tau (and, with boundary, the
    boundary gap <= tau); ties -> smaller S_d, k."""
    rho_best, best = 0.0, None
    for S_d in cand:
        if S_d >= S:
            continue
        t_d = t_d_of(S_d)
        if t_d > tau:
            continue
        t_p = t_p_of(S - S_d)
        for k in range(1, k_max + 1):
            if boundary and boundary_gap(k, t_d, t_p) > tau:
                continue
            rho = float(k * T_dec + T_pre) / max(float(k) * t_d, t_p)
            if rho > rho_best:
                rho_best, best = rho, (S - S_d, S_d, k, t_p, t_d)
    return rho_best, best


def infeasible_fallback(S: int, cand, k_max: int, t_d_of, t_p_of, T_dec: int, T_pre: int):
    """No S_d meets tau: S_d = first argmin t_d over the candidates, k by the same rule (reading #20)."""
    best_sd, best_td = None, None
    for S_d in cand:
        if S_d >= S:
            continue
        t_d = t_d_of(S_d)
        if best_td is None or t_d < best_td:
            best_sd, best_td = S_d, t_d
    if best_sd is None:
        raise ConfigError("no candidate S_d below total_sms")
    S_p = S - best_sd
    t_p = t_p_of(S_p)
    r = math.floor(t_p / best_td)
    rho_best, kb = 0.0, 1
    for k in (_clamp_k(r, k_max), _clamp_k(r + 1, k_max)):
        rho = float(k * T_dec + T_pre) / max(float(k) * best_td, t_p)
        if rho > rho_best:
            rho_best, kb = rho, k
    return rho_best, (S_p, best_sd, kb, t_p, best_td)


def _choose(sp: Spec, prof: Profile, batch: list, tau: float, k_max: int, opts: int, search) -> Split:
    if not (tau > 0):
        raise ConfigError("tbt_slo must be > 0")
    if k_max < 1:
        raise ConfigError("k_max must be >= 1")
    incl = bool(opts & OPT_INCLUDE_CLS)
    S = prof.total_sms
    # l.2: t_mixed(S) = f_roofline(R_mixed, Pi(S), B(S))
    t_mixed = predict(sp, prof, batch, S, incl)["t_total"]
    # l.3-4: temporal when the mixed batch meets the SLO ("<=", reading #19)
    if t_mixed <= tau and not (opts & OPT_FORCE_SPATIAL):
        return _temporal(batch, t_mixed, 0, S)
    # l.6: R_prefill, R_decode <- R_mixed
    P, D = _phases(batch)
    if not P or not D:
        return _temporal(batch, t_mixed, FLAG_DEGENERATE, S)       # reading #21
    T_dec, T_pre = len(D), sum(r.q for r in P)                     # reading #25
    t_d_of = lambda S_d: predict(sp, prof, D, S_d, incl)["t_total"]
    t_p_of = lambda S_p: predict(sp, prof, P, S_p, incl)["t_total"]
    rho, best = search(S, prof.cand_sd_sms, tau, k_max, t_d_of, t_p_of, T_dec, T_pre,
                       bool(opts & OPT_BOUNDARY_TBT))
    flags = 0
    if best is None:
        rho, best = infeasible_fallback(S, prof.cand_sd_sms, k_max, t_d_of, t_p_of, T_dec, T_pre)
        flags = FLAG_INFEASIBLE
        # reading #20b: no split meets tau, so both modes miss the SLO; keep the spatial fallback only
        # if its throughput rho is not below the temporal mixed batch's (the objective of Alg. 1)
        rho_t = float(T_dec + T_pre) / t_mixed if t_mixed > 0 else 0.0
        if rho < rho_t and not (opts & OPT_VERBATIM_INFEASIBLE) and not (opts & OPT_FORCE_SPATIAL):
            return _temporal(batch, t_mixed, FLAG_INFEASIBLE, S)
    S_p, S_d, k, t_p, t_d = best
    return Split(MODE_SPATIAL, S_p, S_d, k, flags, t_mixed, t_p, t_d, rho)


def choose_split(sp: Spec, prof: Profile, batch: list, tau: float, k_max: int = 32, opts: int = 0) -> Split:
    """Algorithm 1 with the readings of the module docstring."""
    return _choose(sp, prof, batch, tau, k_max, opts, alg1_search)


def choose_split_exhaustive(sp: Spec, prof: Profile, batch: list, tau: float, k_max: int = 32,
                            opts: int = 0) -> Split:
    """Same gate / degenerate / infeasible paths; the (S_d, k) search is brute force."""
    return _choose(sp, prof, batch, tau, k_max, opts, exhaustive_search)


# ---------------------------------------------------------------- profiles used by tests

def h100_like_profile(total_sms: int = 132, step: int = 2) -> Profile:
    """SPEC.md's H100-like profile: 4.947e14 FLOP/s dense bf16, 3.35e12 B/s, linear FLOPs curve,
    bandwidth (S/total)^0.32 (Fig. 4a '20% of SMs ~ 60% of BW').  Input data for tests."""
    fl = [0.0] + [4.947e14 * i / total_sms for i in range(1, total_sms + 1)]
    bw = [0.0] + [3.35e12 * min(1.0, (i / total_sms) ** 0.32) for i in range(1, total_sms + 1)]
    cand = tuple(range(step, total_sms, step))
    return Profile(total_sms, cand, tuple(fl), tuple(bw), 4.5e11, 3e-6)

"""Pins for oracle/layer.py against things other than itself (CPU only).

* a pure-Python brute-force layer (loops + ``math``; no numpy, no oracle code) on tiny shapes;
* library special cases in float64: torch SDPA (causal with prefix, GQA), torch rms_norm, torch silu;
* closed forms: one key -> o = v; identical keys -> mean(V); RoPE hand values, p = 0 identity,
  norm preservation, additivity, relative-position property;
* invariants: decode-after-prefill == prefill row, two chunks == one prefill,
  GQA == MHA with duplicated K/V heads, W_o = W_down = 0 -> y = x, page-permutation invariance,
  poisoned pool (only listed slots change), slot formula and write conservation.
"""
import math

import numpy as np
import pytest
import torch

import synth
from synth import configs, workload
from oracle import layer as OL
from tests.oracle_run import run, make_kv, rel_err

RNG = np.random.default_rng(1234)


# ---------------------------------------------------------------- brute force (independent loops)

def _bf_rmsnorm(x, g, eps):
    ms = sum(v * v for v in x) / len(x)
    r = 1.0 / math.sqrt(ms + eps)
    return [x[i] * r * g[i] for i in range(len(x))]


def _bf_matvec(W, x):      # W [out][in] (nn.Linear layout): y_o = sum_i W[o][i] x[i]
    return [sum(W[o][i] * x[i] for i in range(len(x))) for o in range(len(W))]


def _bf_rope(t, p, theta):
    d = len(t)
    h = d // 2
    out = list(t)
    for i in range(h):
        ang = p * theta ** (-2.0 * i / d)
        a, b = t[i], t[i + h]
        out[i] = a * math.cos(ang) - b * math.sin(ang)
        out[i + h] = b * math.cos(ang) + a * math.sin(ang)
    return out


def _bf_layer(W, xs, pos0, hist_k, hist_v, hq, hkv, dh, m, theta, eps):
    """Sequence-level brute force: tokens xs at positions pos0.. after history (lists)."""
    n = len(xs)
    Ks = [list(map(list, hk)) for hk in hist_k]     # [pos][head][dh]
    Vs = [list(map(list, hv)) for hv in hist_v]
    qs = []
    for i in range(n):
        h = _bf_rmsnorm(xs[i], W["g_norm1"], eps)
        qkv = _bf_matvec(W["w_qkv"], h)
        q = [_bf_rope(qkv[j * dh:(j + 1) * dh], pos0 + i, theta) for j in range(hq)]
        k = [_bf_rope(qkv[(hq + j) * dh:(hq + j + 1) * dh], pos0 + i, theta) for j in range(hkv)]
        v = [qkv[(hq + hkv + j) * dh:(hq + hkv + j + 1) * dh] for j in range(hkv)]
        Ks.append(k)
        Vs.append(v)
        qs.append(q)
    ys = []
    for i in range(n):
        p = pos0 + i
        o = []
        for j in range(hq):
            jk = j // (hq // hkv)
            s = [sum(qs[i][j][e] * Ks[t][jk][e] for e in range(dh)) / math.sqrt(dh) for t in range(p + 1)]
            mx = max(s)
            ex = [math.exp(v - mx) for v in s]
            Z = sum(ex)
            o.extend(sum(ex[t] / Z * Vs[t][jk][e] for t in range(p + 1)) for e in range(dh))
        u = _bf_matvec(W["w_o"], o)
        x1 = [xs[i][e] + u[e] for e in range(len(u))]
        h2 = _bf_rmsnorm(x1, W["g_norm2"], eps)
        gu = _bf_matvec(W["w_gate_up"], h2)
        a = [gu[e] / (1.0 + math.exp(-gu[e])) * gu[m + e] for e in range(m)]
        z = _bf_matvec(W["w_down"], a)
        ys.append([x1[e] + z[e] for e in range(len(z))])
    return ys


@pytest.mark.parametrize("hq,hkv", [(2, 1), (2, 2), (4, 2)])
def test_layer_vs_bruteforce_loops(hq, hkv):
    d, dh, m, theta, eps, P = 8, 4, 6, 100.0, 1e-5, 2
    if hq * dh != d:
        d = hq * dh
    W = {
        "w_qkv": RNG.standard_normal(((hq + 2 * hkv) * dh, d)) / 3,
        "w_o": RNG.standard_normal((d, hq * dh)) / 3,
        "w_gate_up": RNG.standard_normal((2 * m, d)) / 3,
        "w_down": RNG.standard_normal((d, m)) / 3,
        "g_norm1": 1 + RNG.standard_normal(d) / 4,
        "g_norm2": 1 + RNG.standard_normal(d) / 4,
        "b_qkv": None,
    }
    c, q = 3, 4
    hk = RNG.standard_normal((c, hkv, dh))
    hv = RNG.standard_normal((c, hkv, dh))
    xs = RNG.standard_normal((q, d))
    # oracle: pages scattered (table [5, 2, 0, 7]) with page size 2
    table = np.array([5, 2, 0, 7], dtype=np.int32)
    kv = OL.PagedKV(1, 8, hkv, P, dh)
    kv.load_history(0, table, hk, hv)
    mdl = OL.Model(d, m, hq, hkv, dh, theta, eps)
    y = OL.layer_forward(mdl, W, 0, xs, np.arange(c, c + q), [table] * q, kv)
    Wl = {k: (v.tolist() if v is not None else None) for k, v in W.items()}
    yb = np.array(_bf_layer(Wl, xs.tolist(), c, hk.tolist(), hv.tolist(), hq, hkv, dh, m, theta, eps))
    assert np.max(np.abs(y - yb)) < 1e-12 * max(1.0, np.max(np.abs(yb)))


def test_attend_row_closed_forms():
    dh = 8
    q = RNG.standard_normal(dh)
    v = RNG.standard_normal((1, dh))
    K = RNG.standard_normal((1, dh))
    assert np.array_equal(OL.attend_row(q, K, v, 0.3), v[0])          # one key -> o = v
    Kid = np.repeat(RNG.standard_normal((1, dh)), 5, axis=0)           # identical keys -> mean(V)
    V = RNG.standard_normal((5, dh))
    np.testing.assert_allclose(OL.attend_row(q, Kid, V, 0.3), V.mean(0), rtol=0, atol=1e-14)


@pytest.mark.parametrize("hq,hkv,c,q", [(4, 4, 0, 9), (4, 2, 5, 7), (8, 2, 17, 3), (2, 1, 31, 1)])
def test_paged_attention_vs_torch_sdpa(hq, hkv, c, q):
    dh, P = 16, 4
    n_pos = c + q
    npages = (n_pos + P - 1) // P
    table = RNG.permutation(npages + 3)[:npages].astype(np.int32)
    kv = OL.PagedKV(1, npages + 3, hkv, P, dh)
    K = RNG.standard_normal((n_pos, hkv, dh))
    V = RNG.standard_normal((n_pos, hkv, dh))
    kv.load_history(0, table, K, V)
    Q = RNG.standard_normal((q, hq, dh))
    o = OL.paged_causal_attention(Q, np.arange(c, c + q), [table] * q, kv, 0, hkv)
    # library: SDPA float64 with explicit causal-with-prefix mask and GQA
    qt = torch.from_numpy(Q).permute(1, 0, 2)[None]            # [1, hq, q, dh]
    kt = torch.from_numpy(K).permute(1, 0, 2)[None]
    vt = torch.from_numpy(V).permute(1, 0, 2)[None]
    mask = torch.arange(n_pos)[None, :] <= (c + torch.arange(q))[:, None]
    ref = torch.nn.functional.scaled_dot_product_attention(qt, kt, vt, attn_mask=mask, enable_gqa=True)
    ref = ref[0].permute(1, 0, 2).numpy()
    np.testing.assert_allclose(o, ref, rtol=0, atol=1e-12)


def test_rmsnorm_and_silu_vs_torch():
    x = RNG.standard_normal((5, 64))
    g = 1 + RNG.standard_normal(64) / 3
    ref = torch.nn.functional.rms_norm(torch.from_numpy(x), (64,), torch.from_numpy(g), eps=1e-5).numpy()
    np.testing.assert_allclose(OL.rmsnorm(x, g, 1e-5), ref, rtol=1e-14, atol=1e-14)
    z = RNG.standard_normal(1000) * 6
    np.testing.assert_allclose(OL.silu(z), torch.nn.functional.silu(torch.from_numpy(z)).numpy(),
                               rtol=1e-14, atol=1e-15)


def test_rope_hand_values_and_properties():
    # d_h = 2: theta_0 = 1, so p = 1 rotates (1, 0) to (cos 1, sin 1)
    t = np.array([[1.0, 0.0]])
    np.testing.assert_allclose(OL.rope(t, np.array(1), 10.0)[0], [math.cos(1), math.sin(1)], atol=1e-15)
    # d_h = 4, theta = 1e4: pair (t1, t3) has frequency 1e4^(-2/4) = 0.01; p = 100 -> angle 1 rad
    t = np.array([[0.0, 2.0, 0.0, 3.0]])
    r = OL.rope(t, np.array(100), 1e4)[0]
    np.testing.assert_allclose(r[[1, 3]], [2 * math.cos(1) - 3 * math.sin(1), 3 * math.cos(1) + 2 * math.sin(1)],
                               atol=1e-13)
    np.testing.assert_allclose(r[[0, 2]], [0.0, 0.0], atol=1e-15)
    x = RNG.standard_normal((3, 64))
    np.testing.assert_array_equal(OL.rope(x, np.array(0), 5e5), x)                 # p = 0 identity
    y = OL.rope(x, np.array(1234), 5e5)
    np.testing.assert_allclose(np.linalg.norm(y, axis=-1), np.linalg.norm(x, axis=-1), rtol=1e-13)
    np.testing.assert_allclose(OL.rope(OL.rope(x, np.array(7), 1e4), np.array(11), 1e4),
                               OL.rope(x, np.array(18), 1e4), atol=1e-12)           # additivity
    qv, kv = RNG.standard_normal((1, 64)), RNG.standard_normal((1, 64))
    d1 = OL.rope(qv, np.array(50), 1e4)[0] @ OL.rope(kv, np.array(20), 1e4)[0]
    d2 = OL.rope(qv, np.array(130), 1e4)[0] @ OL.rope(kv, np.array(100), 1e4)[0]
    assert abs(d1 - d2) < 1e-11                                                        # depends on m - n only


def _tiny_cfg(**kw):
    from dataclasses import replace
    cfg = configs.get_config("cfg1")
    return replace(cfg, model=replace(cfg.model, **kw)) if kw else cfg


def test_decode_after_prefill_equals_prefill_row():
    """North-star invariant: decoding token t after prefilling 0..t-1 == row t of a prefill over 0..t."""
    cfg = _tiny_cfg(n_layers=2)
    m = OL.Model.from_cfg(cfg.model)
    W = [synth.layer_weights(cfg.model, l, cfg.seed) for l in range(2)]
    T = 21
    x = synth.x_rows(cfg.seed, synth.S_XPRE, T, m.d_model)
    table = np.arange(4, dtype=np.int32)[::-1].copy()
    kv_a = OL.PagedKV(2, 4, m.n_kv_heads, 16, m.head_dim)
    y_full = OL.prefill_forward(m, W, x, [(T, 0)], [table], kv_a)
    kv_b = OL.PagedKV(2, 4, m.n_kv_heads, 16, m.head_dim)
    OL.prefill_forward(m, W, x[:T - 1], [(T - 1, 0)], [table], kv_b)
    y_dec = OL.decode_window(m, W, x[T - 1:T], [T - 1], [table], kv_b, 1)
    assert rel_err(y_dec[0, 0], y_full[T - 1]) < 1e-13
    # the caches end identical up to rounding
    np.testing.assert_allclose(kv_a.K, kv_b.K, atol=1e-12)


def test_two_chunks_equal_one_prefill():
    cfg = _tiny_cfg()
    m = OL.Model.from_cfg(cfg.model)
    W = [synth.layer_weights(cfg.model, 0, cfg.seed)]
    T, c1 = 40, 17
    x = synth.x_rows(cfg.seed, synth.S_XPRE, T, m.d_model)
    table = np.array([2, 0, 3], dtype=np.int32)
    kv1 = OL.PagedKV(1, 4, m.n_kv_heads, 16, m.head_dim)
    y1 = OL.prefill_forward(m, W, x, [(T, 0)], [table], kv1)
    kv2 = OL.PagedKV(1, 4, m.n_kv_heads, 16, m.head_dim)
    ya = OL.prefill_forward(m, W, x[:c1], [(c1, 0)], [table], kv2)
    yb = OL.prefill_forward(m, W, x[c1:], [(T - c1, c1)], [table], kv2)
    assert rel_err(np.concatenate([ya, yb]), y1) < 1e-13


def test_gqa_equals_mha_with_duplicated_heads():
    cfg = configs.get_config("cfg1-gqa")
    mg = OL.Model.from_cfg(cfg.model)
    Wg = synth.layer_weights(cfg.model, 0, cfg.seed)
    hq, hkv, dh = mg.n_q_heads, mg.n_kv_heads, mg.head_dim
    g = hq // hkv
    wq = Wg["w_qkv"][: hq * dh]
    wk = Wg["w_qkv"][hq * dh:(hq + hkv) * dh].reshape(hkv, dh, -1)
    wv = Wg["w_qkv"][(hq + hkv) * dh:].reshape(hkv, dh, -1)
    Wm = dict(Wg)
    Wm["w_qkv"] = np.concatenate([wq, np.repeat(wk, g, axis=0).reshape(hq * dh, -1),
                                  np.repeat(wv, g, axis=0).reshape(hq * dh, -1)])
    mm = OL.Model(mg.d_model, mg.ffn_dim, hq, hq, dh, mg.rope_theta, mg.norm_eps)
    x = synth.x_rows(cfg.seed, synth.S_XPRE, 19, mg.d_model)
    t = np.array([1, 0], dtype=np.int32)
    yg = OL.prefill_forward(mg, [Wg], x, [(19, 0)], [t], OL.PagedKV(1, 2, hkv, 16, dh))
    ym = OL.prefill_forward(mm, [Wm], x, [(19, 0)], [t], OL.PagedKV(1, 2, hq, 16, dh))
    assert rel_err(yg, ym) < 1e-13


def test_zero_output_projections_give_identity():
    cfg = _tiny_cfg()
    m = OL.Model.from_cfg(cfg.model)
    W = dict(synth.layer_weights(cfg.model, 0, cfg.seed))
    W["w_o"] = np.zeros_like(W["w_o"])
    W["w_down"] = np.zeros_like(W["w_down"])
    x = synth.x_rows(cfg.seed, synth.S_XPRE, 5, m.d_model)
    y = OL.prefill_forward(m, [W], x, [(5, 0)], [np.array([0], np.int32)], OL.PagedKV(1, 1, m.n_kv_heads, 16, m.head_dim))
    np.testing.assert_array_equal(y, x.astype(np.float64))


def test_page_permutation_invariance_bitwise():
    cfg = configs.get_config("cfg1-gqa")
    wl = workload.build(cfg, n_dec=3, k=2)
    y1p, y1d, _ = run(wl)
    # a different seeded placement of the same logical requests
    from dataclasses import replace
    wl2 = workload.build(replace(cfg, seed=cfg.seed), n_dec=3, k=2)
    perm = np.random.default_rng(7).permutation(wl.n_pages).astype(np.int32)
    wl2.pre_tables = np.where(wl.pre_tables >= 0, perm[np.maximum(wl.pre_tables, 0)], -1).astype(np.int32)
    wl2.dec_tables = np.where(wl.dec_tables >= 0, perm[np.maximum(wl.dec_tables, 0)], -1).astype(np.int32)
    y2p, y2d, _ = run(wl2)
    np.testing.assert_array_equal(y1p, y2p)
    np.testing.assert_array_equal(y1d, y2d)


def test_poisoned_pool_only_listed_slots_change_and_conservation():
    cfg = configs.get_config("cfg1-gqa")
    wl = workload.build(cfg, n_dec=3, k=3)
    kv = make_kv(wl)
    # poison every slot that holds no history
    hist = np.zeros(kv.K.shape[:2] + (kv.page_size,), dtype=bool)
    for l, trow, uid, n in wl.history_items():
        p = np.arange(n)
        hist[l, trow[p // kv.page_size], p % kv.page_size] = True
    kv.K.transpose(0, 1, 3, 2, 4)[~hist] = np.nan     # pool is [L][page][head][slot][d_h]
    kv.V.transpose(0, 1, 3, 2, 4)[~hist] = np.nan
    before_K = kv.K.copy()
    y_pre, y_dec, kv = run(wl, kv)
    assert np.all(np.isfinite(y_pre)) and np.all(np.isfinite(y_dec))     # nothing read a poisoned slot
    written = set(kv.writes)
    n_tok = sum(q for q, _ in wl.pre_seqs) + wl.k * len(wl.dec_ctx)
    assert len(kv.writes) == len(written) == n_tok * wl.n_layers            # each token written once
    changed = np.argwhere(np.any(~(np.isclose(kv.K, before_K, equal_nan=True)), axis=(2, 4)))
    assert set(map(tuple, changed.tolist())) <= written
    for (l, page, s) in written:
        assert np.all(np.isfinite(kv.K[l, page, :, s]))
    # slot formula, closed form
    trow = wl.dec_tables[0]
    for p in (0, 15, 16, 33):
        assert kv.slot(trow, p) == (int(trow[p // 16]), p % 16)
    assert kv.flat_offset(3, 1, 5, 7) == ((3 * kv.h_kv + 1) * 16 + 5) * kv.d_h + 7


# ------------------------------------------------------------------ LM head + greedy decode (f1)

def test_lm_head_brute_force_and_ties():
    """logits by explicit loops; argmax takes the lowest index among equal maxima."""
    from oracle import layer as OL
    rng = np.random.default_rng(7)
    d, v = 16, 12
    m = OL.Model(d, 32, 2, 2, 8, 1e4, 1e-5)
    head = {"g_norm": rng.normal(size=d), "w_head": rng.normal(size=(v, d)), "embed": rng.normal(size=(v, d))}
    y = rng.normal(size=(3, d))
    logits, tok = OL.lm_head_greedy(m, head, y)
    for i in range(3):
        ms = sum(float(t) * float(t) for t in y[i]) / d
        h = [y[i][e] / math.sqrt(ms + 1e-5) * head["g_norm"][e] for e in range(d)]
        for t in range(v):
            ref = sum(h[e] * head["w_head"][t][e] for e in range(d))
            assert abs(ref - logits[i, t]) <= 1e-12 * max(1.0, abs(ref))
        best = max(range(v), key=lambda t: (logits[i, t], -t))
        assert tok[i] == best
    head["g_norm"] = np.ones(d)
    head["w_head"][5] = head["w_head"][9] = 10.0 * np.ones(d)   # two identical maxima rows
    _, tok = OL.lm_head_greedy(m, head, np.ones((1, d)))
    assert tok[0] == 5


def test_lm_head_tied_embedding_recovers_token():
    """With w_head = embed (tied) and y = embed[t], the greedy token is t: a row's dot product with
    itself dominates in high dimension (the invariant an autoregressive loop relies on)."""
    from oracle import layer as OL
    rng = np.random.default_rng(3)
    d, v = 256, 64
    m = OL.Model(d, 32, 2, 2, 128, 1e4, 1e-5)
    E = rng.normal(size=(v, d))
    head = {"g_norm": np.ones(d), "w_head": E, "embed": E}
    t = np.array([0, 17, 63, 5])
    _, tok = OL.lm_head_greedy(m, head, E[t])
    assert np.array_equal(tok, t)


def test_decode_window_with_head_feeds_embedding():
    """Step j+1's input is embed[token_j]: the window equals k single steps chained by hand."""
    from oracle import layer as OL
    from synth import configs, head_weights, workload
    from tests.oracle_run import make_kv
    cfg = configs.get_config("cfg1")
    wl = workload.build(cfg, k=2)
    m = OL.Model.from_cfg(cfg.model)
    head = head_weights(cfg.model, cfg.seed)
    toks = []
    y = OL.decode_window(m, wl.weights, wl.x_dec, wl.dec_ctx, wl.dec_tables, make_kv(wl), 2, head, toks)
    kv = make_kv(wl)
    y1 = OL.decode_window(m, wl.weights, wl.x_dec, wl.dec_ctx, wl.dec_tables, kv, 1)
    _, t1 = OL.lm_head_greedy(m, head, y1[0])
    x2 = np.asarray(head["embed"], dtype=np.float64)[t1]
    y2 = OL.decode_window(m, wl.weights, x2, [c + 1 for c in wl.dec_ctx], wl.dec_tables, kv, 1)
    assert np.array_equal(toks[0][1], t1)
    assert np.allclose(y[1], y2[0], rtol=0, atol=1e-12)


def test_decode_window_feedback_chains_outputs():
    """Reading #26 (head = None): step j+1's input is step j's final-layer OUTPUT (not the window's
    input x): a k = 2 window equals two single-step windows chained by hand, and differs from feeding x
    again."""
    from oracle import layer as OL
    from synth import configs, workload
    from tests.oracle_run import make_kv
    cfg = configs.get_config("cfg1")
    wl = workload.build(cfg, k=2)
    m = OL.Model.from_cfg(cfg.model)
    y = OL.decode_window(m, wl.weights, wl.x_dec, wl.dec_ctx, wl.dec_tables, make_kv(wl), 2)
    kv = make_kv(wl)
    y1 = OL.decode_window(m, wl.weights, wl.x_dec, wl.dec_ctx, wl.dec_tables, kv, 1)
    y2 = OL.decode_window(m, wl.weights, y1[0], [c + 1 for c in wl.dec_ctx], wl.dec_tables, kv, 1)
    assert np.allclose(y[0], y1[0], rtol=0, atol=1e-12)
    assert np.allclose(y[1], y2[0], rtol=0, atol=1e-12)
    kv_x = make_kv(wl)
    OL.decode_window(m, wl.weights, wl.x_dec, wl.dec_ctx, wl.dec_tables, kv_x, 1)
    y2_x = OL.decode_window(m, wl.weights, wl.x_dec, [c + 1 for c in wl.dec_ctx], wl.dec_tables, kv_x, 1)
    assert not np.allclose(y[1], y2_x[0], rtol=0, atol=1e-3)   # feeding x again is a different result


def test_row_parallel_allreduce_equals_unsharded_linear():
    """f3 reference (oracle.layer.row_parallel_allreduce): splitting the contraction dimension of one
    linear over N ranks and summing the partials is the unsharded linear — checked exactly on integer
    matrices (every product and sum exact in float64) for uneven shard widths."""
    rng = np.random.default_rng(11)
    n, k, dout = 37, 96, 40
    A = rng.integers(-8, 9, size=(n, k)).astype(np.float64)
    W = rng.integers(-8, 9, size=(dout, k)).astype(np.float64)
    R = rng.integers(-8, 9, size=(n, dout)).astype(np.float64)
    for cuts in ([48], [16, 64], [8, 40, 72]):   # N = 2, 3, 4 ranks, uneven widths
        edges = [0] + cuts + [k]
        a_sh = [A[:, edges[i]:edges[i + 1]] for i in range(len(edges) - 1)]
        w_sh = [W[:, edges[i]:edges[i + 1]] for i in range(len(edges) - 1)]
        got = OL.row_parallel_allreduce(a_sh, w_sh, R)
        want = R + np.einsum("ik,jk->ij", A, W)
        assert np.array_equal(got, want)
    # dropping a rank's partial is caught
    assert not np.array_equal(OL.row_parallel_allreduce(a_sh[:-1], w_sh[:-1], R), want)

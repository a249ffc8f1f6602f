"""Materialise a synth workload directly in device memory (torch plumbing, no method arithmetic).

Same values as ``synth.layer_weights`` / ``synth.kv_history`` / ``synth.x_rows`` (the counter
generator has identical numpy and torch implementations), generated on the GPU so that
BASELINE-size configurations (GBs of KV history) do not go through the host.
"""
from __future__ import annotations

import numpy as np
import torch

from . import (S_BQKV, S_EMBED, S_G1, S_G2, S_GFINAL, S_KHIST, S_VHIST, S_WDOWN, S_WGU, S_WHEAD, S_WO, S_WQKV,
               S_XDEC, S_XPRE, counter_values_torch, pow2_scale)


def head_weights_gpu(cfg_model, seed: int, device, dtype) -> dict:
    """Same values as synth.head_weights (LM head of the decode loop, f1), generated on the GPU."""
    d, v = cfg_model.d_model, cfg_model.vocab
    return {
        "g_norm": (1.0 + counter_values_torch(seed, S_GFINAL, (d,), 0, 3, device=device)).to(dtype),
        "w_head": counter_values_torch(seed, S_WHEAD, (v, d), 0, pow2_scale(d), device=device, dtype=dtype),
        "embed": counter_values_torch(seed, S_EMBED, (v, d), 0, 0, device=device, dtype=dtype),
    }


def layer_weights_gpu(cfg_model, layer: int, seed: int, device, dtype) -> dict:
    m = cfg_model
    d, f, hq, hkv, dh = m.d_model, m.ffn_dim, m.n_q_heads, m.n_kv_heads, m.head_dim
    nqkv = (hq + 2 * hkv) * dh
    base = layer * (1 << 36)
    cv = lambda s, shape, sc: counter_values_torch(seed, s, shape, base, sc, device=device, dtype=dtype)
    w = {
        "w_qkv": cv(S_WQKV, (nqkv, d), pow2_scale(d)),
        "w_o": cv(S_WO, (d, hq * dh), pow2_scale(hq * dh)),
        "w_gate_up": cv(S_WGU, (2 * f, d), pow2_scale(d)),
        "w_down": cv(S_WDOWN, (d, f), pow2_scale(f)),
        "g_norm1": (1.0 + counter_values_torch(seed, S_G1, (d,), base, 3, device=device)).to(dtype),
        "g_norm2": (1.0 + counter_values_torch(seed, S_G2, (d,), base, 3, device=device)).to(dtype),
    }
    if m.qkv_bias:
        w["b_qkv"] = cv(S_BQKV, (nqkv,), 6)
    return w


def kv_pools_gpu(wl, device, dtype, fill=0.0):
    """Per-layer K and V pools with every pre-existing history placed at its page slots."""
    m = wl.cfg.model
    P = wl.cfg.batch.page_size
    shape = (wl.n_pages, m.n_kv_heads, P, m.head_dim)
    K = [torch.full(shape, fill, dtype=dtype, device=device) for _ in range(wl.n_layers)]
    V = [torch.full(shape, fill, dtype=dtype, device=device) for _ in range(wl.n_layers)]
    per_req = 1 << 30
    for l, trow, uid, n in wl.history_items():
        base = (l * 4096 + uid) * per_req
        p = torch.arange(n, device=device)
        pages = torch.from_numpy(np.ascontiguousarray(trow).astype(np.int64)).to(device)[p // P]
        slots = p % P
        Kh = counter_values_torch(wl.cfg.seed, S_KHIST, (n, m.n_kv_heads, m.head_dim), base, device=device,
                                  dtype=dtype)
        K[l][pages, :, slots, :] = Kh
        del Kh
        Vh = counter_values_torch(wl.cfg.seed, S_VHIST, (n, m.n_kv_heads, m.head_dim), base, device=device,
                                  dtype=dtype)
        V[l][pages, :, slots, :] = Vh
        del Vh
    return K, V


def inputs_gpu(wl, device, dtype):
    m = wl.cfg.model
    n_p = sum(q for q, _ in wl.pre_seqs)
    x_pre = counter_values_torch(wl.cfg.seed, S_XPRE, (n_p, m.d_model), 0, device=device, dtype=dtype)
    x_dec = counter_values_torch(wl.cfg.seed, S_XDEC, (len(wl.dec_ctx), m.d_model), 0, device=device, dtype=dtype)
    return x_pre, x_dec

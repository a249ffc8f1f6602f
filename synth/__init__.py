"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and bench.py.

This module holds NO arithmetic of the method (no norm, projection, RoPE,
attention or roofline formula).  It only produces numbers:

* ``counter_values`` — a counter-based generator: the value of element ``i`` of
  stream ``s`` under ``seed`` is a pure function of ``(seed, s, i)``.  Values lie
  on the grid ``k/64`` with integer ``k`` in ``[-110, 110]`` (mean 0, variance
  ~0.99), every one of them exactly representable in bf16, fp32 and fp64, so the
  oracle (fp64) and the GPU path (bf16 or fp32) see bit-identical inputs with
  no rounding step.  A numpy and a torch implementation produce identical
  integers (checked in ``tests/test_synth.py``); the torch one runs on the GPU
  to fill tensors too large for the host (the 32-layer KV history).
* seeded page tables (a numpy ``PCG64`` permutation of the pool's pages),
* the configuration presets of SURVEY.md §8(d) (``synth.configs``).

Weight scaling uses a power of two near ``1/sqrt(d_in)`` so scaled values stay
exact in bf16 ("Input recipe").
"""
from __future__ import annotations

import math

import numpy as np

from .configs import ModelCfg, BatchCfg, CONFIGS, get_config  # noqa: F401

GRID_HALF = 110          # k in [-110, 110]
GRID_DEN = 64.0          # value = k / 64
_M32 = 0xFFFFFFFF

# stream ids (arbitrary, fixed): one per kind of tensor
S_WQKV, S_BQKV, S_WO, S_WGU, S_WDOWN, S_G1, S_G2 = 1, 2, 3, 4, 5, 6, 7
S_XPRE, S_XDEC, S_KHIST, S_VHIST = 11, 12, 13, 14
S_GFINAL, S_WHEAD, S_EMBED = 21, 22, 23


def _hash32_np(x: np.ndarray) -> np.ndarray:
    """lowbias32 finalizer on uint64 arrays holding 32-bit values."""
    x = x & _M32
    x = x ^ (x >> 16)
    x = (x * 0x7FEB352D) & _M32
    x = x ^ (x >> 15)
    x = (x * 0x846CA68B) & _M32
    x = x ^ (x >> 16)
    return x


def _key(seed: int, stream: int) -> int:
    k = np.array([(seed * 0x9E3779B1 + stream * 0x85EBCA77 + 0x165667B1) & _M32], dtype=np.uint64)
    return int(_hash32_np(_hash32_np(k))[0])


def counter_ints(seed: int, stream: int, idx: np.ndarray) -> np.ndarray:
    """Integer k in [-GRID_HALF, GRID_HALF] for each flat counter in ``idx`` (numpy)."""
    idx = np.asarray(idx, dtype=np.uint64)
    key = np.uint64(_key(seed, stream))
    lo = idx & np.uint64(_M32)
    hi = idx >> np.uint64(32)
    h = _hash32_np(lo ^ _hash32_np(hi ^ key))
    return (h % np.uint64(2 * GRID_HALF + 1)).astype(np.int64) - GRID_HALF


def counter_values(seed: int, stream: int, shape, offset: int = 0, scale_pow2: int = 0) -> np.ndarray:
    """float32 array of ``shape``; element i = counter_ints(offset+i) / 64 * 2**-scale_pow2."""
    n = int(np.prod(shape)) if len(shape) else 1
    idx = np.arange(offset, offset + n, dtype=np.uint64)
    k = counter_ints(seed, stream, idx).astype(np.float64)
    return (k / GRID_DEN * (2.0 ** -scale_pow2)).astype(np.float32).reshape(shape)


def counter_values_torch(seed: int, stream: int, shape, offset: int = 0, scale_pow2: int = 0,
                         device="cpu", dtype=None):
    """Same values as ``counter_values`` computed with torch int64 ops on ``device``."""
    import torch
    n = 1
    for s in shape:
        n *= int(s)
    M = _M32

    def h32(x):
        x = x & M
        x = x ^ (x >> 16)
        x = (x * 0x7FEB352D) & M
        x = x ^ (x >> 15)
        x = (x * 0x846CA68B) & M
        x = x ^ (x >> 16)
        return x

    key = _key(seed, stream)
    idx = torch.arange(offset, offset + n, dtype=torch.int64, device=device)
    lo = idx & M
    hi = idx >> 32
    h = h32(lo ^ h32(hi ^ key))
    k = (h % (2 * GRID_HALF + 1)) - GRID_HALF
    out = k.to(torch.float32) * (1.0 / GRID_DEN) * (2.0 ** -scale_pow2)
    if dtype is not None:
        out = out.to(dtype)
    return out.reshape(tuple(int(s) for s in shape))


def pow2_scale(d_in: int) -> int:
    """Exponent e so that 2**-e is the power of two nearest 1/sqrt(d_in)."""
    return int(round(math.log2(math.sqrt(d_in))))


# ---------------------------------------------------------------- model inputs

def layer_weights(cfg: ModelCfg, layer: int, seed: int) -> dict:
    """fp32 weights of one layer, nn.Linear layout [out, in]; gate_up rows = [gate(m); up(m)]."""
    d, m, hq, hkv, dh = cfg.d_model, cfg.ffn_dim, cfg.n_q_heads, cfg.n_kv_heads, cfg.head_dim
    nqkv = (hq + 2 * hkv) * dh
    base = layer * (1 << 36)
    w = {
        "w_qkv": counter_values(seed, S_WQKV, (nqkv, d), base, pow2_scale(d)),
        "w_o": counter_values(seed, S_WO, (d, hq * dh), base, pow2_scale(hq * dh)),
        "w_gate_up": counter_values(seed, S_WGU, (2 * m, d), base, pow2_scale(d)),
        "w_down": counter_values(seed, S_WDOWN, (d, m), base, pow2_scale(m)),
        # gamma = 1 + u/8  (values in [-0.72, 2.72], exact in bf16): non-trivial so a dropped gamma fails
        "g_norm1": (1.0 + counter_values(seed, S_G1, (d,), base, 3)).astype(np.float32),
        "g_norm2": (1.0 + counter_values(seed, S_G2, (d,), base, 3)).astype(np.float32),
        "b_qkv": None,
    }
    if cfg.qkv_bias:
        w["b_qkv"] = counter_values(seed, S_BQKV, (nqkv,), base, 6)
    return w


def head_weights(cfg: ModelCfg, seed: int) -> dict:
    """fp32 LM head of the decode loop: final norm gain [d], w_head [vocab][d]
    (scaled like a layer weight), embed [vocab][d] (unscaled grid values, like the x rows)."""
    d, v = cfg.d_model, cfg.vocab
    return {
        "g_norm": (1.0 + counter_values(seed, S_GFINAL, (d,), 0, 3)).astype(np.float32),
        "w_head": counter_values(seed, S_WHEAD, (v, d), 0, pow2_scale(d)),
        "embed": counter_values(seed, S_EMBED, (v, d), 0, 0),
    }


def x_rows(seed: int, stream: int, n_rows: int, d: int, row_offset: int = 0) -> np.ndarray:
    return counter_values(seed, stream, (n_rows, d), row_offset * d)


def kv_history(seed: int, layer: int, req_uid: int, n_pos: int, h_kv: int, d_h: int):
    """(K, V) history of one request in one layer, logical layout [n_pos, h_kv, d_h] (fp32, exact)."""
    per_req = 1 << 30            # counter space per (layer, request)
    base = (layer * 4096 + req_uid) * per_req
    K = counter_values(seed, S_KHIST, (n_pos, h_kv, d_h), base)
    V = counter_values(seed, S_VHIST, (n_pos, h_kv, d_h), base)
    return K, V


def kv_history_torch(seed: int, layer: int, req_uid: int, n_pos: int, h_kv: int, d_h: int, device, dtype):
    per_req = 1 << 30
    base = (layer * 4096 + req_uid) * per_req
    K = counter_values_torch(seed, S_KHIST, (n_pos, h_kv, d_h), base, device=device, dtype=dtype)
    V = counter_values_torch(seed, S_VHIST, (n_pos, h_kv, d_h), base, device=device, dtype=dtype)
    return K, V


def page_tables(seed: int, n_tokens_per_req, page_size: int, n_pages: int, max_pages: int | None = None):
    """Seeded fragmented page tables: a PCG64 permutation of the pool, handed out in request order.

    Returns (table int32 [n_req, max_pages] padded with -1, pages used)."""
    need = [(int(t) + page_size - 1) // page_size for t in n_tokens_per_req]
    total = sum(need)
    if total > n_pages:
        raise ValueError(f"pool of {n_pages} pages cannot hold {total}")
    perm = np.random.Generator(np.random.PCG64(seed)).permutation(n_pages).astype(np.int32)
    mp = max(need) if need else 0
    if max_pages is not None:
        mp = max(mp, max_pages)
    mp = max(mp, 1)
    table = np.full((len(need), mp), -1, dtype=np.int32)
    at = 0
    for r, n in enumerate(need):
        table[r, :n] = perm[at:at + n]
        at += n
    return table, total


def round_to_bf16(a: np.ndarray) -> np.ndarray:
    """RNE rounding of float32 values to the nearest bf16 (kept as float32). Identity on grid values."""
    a = np.ascontiguousarray(a, dtype=np.float32)
    u = a.view(np.uint32).astype(np.uint64)
    lsb = (u >> 16) & 1
    u = (u + 0x7FFF + lsb) & 0xFFFF0000
    return u.astype(np.uint32).view(np.float32)

"""Test helper: run the CPU oracle on a synth workload (test infrastructure)."""
from __future__ import annotations

import numpy as np

from oracle import layer as OL


def make_kv(wl) -> OL.PagedKV:
    m = wl.cfg.model
    kv = OL.PagedKV(wl.n_layers, wl.n_pages, m.n_kv_heads, wl.cfg.batch.page_size, m.head_dim)
    for l, trow, uid, n in wl.history_items():
        K, V = wl.history(l, uid, n)
        kv.load_history(l, trow, K, V)
    return kv


def run(wl, kv=None):
    m = OL.Model.from_cfg(wl.cfg.model)
    kv = make_kv(wl) if kv is None else kv
    y_pre, y_dec = OL.mixed_iteration(m, wl.weights, wl.x_pre, wl.pre_seqs, wl.pre_tables,
                                      wl.x_dec, wl.dec_ctx, wl.dec_tables, kv, wl.k)
    return y_pre, y_dec, kv


def rel_err(got, ref) -> float:
    """Normwise max relative error (C-6 / reading #27): max|g - o| / max|o|."""
    got = np.asarray(got, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    den = np.max(np.abs(ref)) if ref.size else 1.0
    if ref.size == 0:
        return 0.0
    return float(np.max(np.abs(got - ref)) / max(den, 1e-300))

"""A mixed-iteration workload: every seeded input of one configuration (numbers only).

Request uids: prefill sequence s has uid s, decode request r has uid n_prefill + r.
The page tables give each prefill sequence pages for c + q tokens and each decode
request pages for c + k tokens (look-ahead slots), from one seeded
permutation of the pool (fragmented placement).
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import (S_XDEC, S_XPRE, kv_history, layer_weights, page_tables, x_rows)
from .configs import Config


@dataclass
class Workload:
    cfg: Config
    weights: list            # per layer dict of fp32 arrays
    x_pre: np.ndarray        # [n_p, d] fp32
    x_dec: np.ndarray        # [n_d, d] fp32
    pre_seqs: list           # [(q, c)]
    dec_ctx: list            # [c_r]
    pre_tables: np.ndarray   # [n_seqs, max_pages] int32
    dec_tables: np.ndarray   # [n_d, max_pages] int32
    n_pages: int
    k: int

    @property
    def n_layers(self):
        return self.cfg.model.n_layers

    def history(self, layer: int, uid: int, n_pos: int):
        m = self.cfg.model
        return kv_history(self.cfg.seed, layer, uid, n_pos, m.n_kv_heads, m.head_dim)

    def history_items(self):
        """(layer, table_row, uid, n_pos) of every pre-existing KV history to place in the pool."""
        n_pre = len(self.pre_seqs)
        for l in range(self.n_layers):
            for s, (q, c) in enumerate(self.pre_seqs):
                if c > 0:
                    yield l, self.pre_tables[s], s, c
            for r, c in enumerate(self.dec_ctx):
                yield l, self.dec_tables[r], n_pre + r, c


def build(cfg: Config, k: int | None = None, n_dec: int | None = None, pre_seqs=None, dec_ctx=None,
          n_layers: int | None = None, with_weights: bool = True, spare_pages: int = 8) -> Workload:
    m = cfg.model
    k = cfg.batch.k if k is None else k
    pre = list(cfg.batch.prefill) if pre_seqs is None else list(pre_seqs)
    dec = list(cfg.batch.decode) if dec_ctx is None else list(dec_ctx)
    if n_dec is not None:
        dec = dec[:n_dec]
    L = m.n_layers if n_layers is None else n_layers
    P = cfg.batch.page_size
    need = [q + c for q, c in pre] + [c + k for c in dec]
    n_pages = sum((t + P - 1) // P for t in need) + spare_pages
    tables, _ = page_tables(cfg.seed, need, P, n_pages)
    n_pre = len(pre)
    weights = [layer_weights(m, l, cfg.seed) for l in range(L)] if with_weights else []
    n_p = sum(q for q, _ in pre)
    x_pre = x_rows(cfg.seed, S_XPRE, n_p, m.d_model)
    x_dec = x_rows(cfg.seed, S_XDEC, len(dec), m.d_model)
    from dataclasses import replace
    cfg2 = replace(cfg, model=replace(m, n_layers=L))
    return Workload(cfg2, weights, x_pre, x_dec, pre, dec, tables[:n_pre], tables[n_pre:], n_pages, k)

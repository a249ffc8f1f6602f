"""Oracle: one transformer layer (or stack) forward over a paged KV cache, float64.

TEST INFRASTRUCTURE ONLY (see ``oracle/__init__.py``).

Follows PAPER.md §2 "LLM Inference Process" under the readings of
DESIGN.md §Readings (numbered as in SURVEY.md §8(c) C-7):

  #1  pre-norm RMSNorm (Llama/Qwen, the models P:90 names) instead of the
      post-LayerNorm written at P:95-97;
  #2  softmax scale 1/sqrt(d_h), d_h = d/h_q;
  #3  SwiGLU FFN  y = x1 + (silu(h2 W_g^T) * (h2 W_u^T)) W_d^T  for sigma(vW1)W2;
  #4  GQA widths: W_qkv has (h_q + 2 h_kv) d_h rows (P:93 writes square W_k, W_v);
  #5  RoPE, NeoX half-split, theta from the model preset (not in the paper);
  #6  q-head j reads kv-head floor(j / (h_q/h_kv));
  #7  causal with a prefix: the token at absolute position p attends to every t <= p;
  #26 decode step j>1 of a look-ahead window takes the previous step's final-layer
      output as its input (synthetic feedback; P:335 samples tokens instead) — or, with an LM
      head, the embedding of the previous step's greedy token.

The KV cache is "concatenate then attend": every new token's (k, v)
is appended to its page slot before any attention of the same call reads it.
Paged layout (C-3): pool[page][h_kv][P][d_h]; slot(r, p) = (table[r][p // P], p % P).

Matmuls use numpy (a library primitive as one step, as allowed).  Attention is a
plain per-(row, head) softmax over the gathered keys — no blocking, no online
softmax, no reordering.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np


# ------------------------------------------------------------------ primitives

def rmsnorm(x: np.ndarray, gamma: np.ndarray, eps: float) -> np.ndarray:
    """h = x * (mean(x^2) + eps)^(-1/2) * gamma   (reading #1 of P:95; C-2 step 1)."""
    x = np.asarray(x, dtype=np.float64)
    ms = np.mean(x * x, axis=-1, keepdims=True)
    return x / np.sqrt(ms + eps) * np.asarray(gamma, dtype=np.float64)


def silu(g: np.ndarray) -> np.ndarray:
    """silu(g) = g / (1 + exp(-g))   (reading #3 of sigma at P:96)."""
    g = np.asarray(g, dtype=np.float64)
    return g / (1.0 + np.exp(-g))


def rope(t: np.ndarray, pos: np.ndarray, theta: float) -> np.ndarray:
    """NeoX half-split rotary embedding (reading #5).

    t: [..., n_heads, d_h] rows at absolute positions ``pos`` (shape [...]).
    For i < d_h/2, with theta_i = theta^(-2i/d_h) and phi = p * theta_i:
      t_i        <- a cos phi - b sin phi
      t_{i+d/2}  <- b cos phi + a sin phi,   (a, b) = (t_i, t_{i+d/2})
    """
    t = np.asarray(t, dtype=np.float64)
    d_h = t.shape[-1]
    half = d_h // 2
    i = np.arange(half, dtype=np.float64)
    inv = theta ** (-2.0 * i / d_h)
    phi = np.asarray(pos, dtype=np.float64)[..., None, None] * inv   # [..., 1, half]
    c, s = np.cos(phi), np.sin(phi)
    a, b = t[..., :half], t[..., half:]
    return np.concatenate([a * c - b * s, b * c + a * s], axis=-1)


def attend_row(q: np.ndarray, K: np.ndarray, V: np.ndarray, scale: float) -> np.ndarray:
    """softmax(q . K_t * scale) . V over all given keys t (reading #2), max-subtracted."""
    s = (K @ q) * scale
    s = s - np.max(s)
    e = np.exp(s)
    a = e / np.sum(e)
    return a @ V


# ------------------------------------------------------------------ paged KV

@dataclass
class PagedKV:
    """Paged KV pools, one K and one V pool per layer: [n_pages][h_kv][P][d_h] float64 (C-3)."""
    n_layers: int
    n_pages: int
    h_kv: int
    page_size: int
    d_h: int
    K: np.ndarray = field(init=False)
    V: np.ndarray = field(init=False)
    writes: list = field(init=False, default_factory=list)

    def __post_init__(self):
        shape = (self.n_layers, self.n_pages, self.h_kv, self.page_size, self.d_h)
        self.K = np.zeros(shape, dtype=np.float64)
        self.V = np.zeros(shape, dtype=np.float64)
        self.writes = []

    def slot(self, table_row: np.ndarray, p: int) -> tuple[int, int]:
        """slot(r, p) = (pt[r][p // P], p mod P)."""
        page = int(table_row[p // self.page_size])
        if page < 0 or page >= self.n_pages:
            raise IndexError(f"position {p} maps to page {page} outside the pool")
        return page, p % self.page_size

    def flat_offset(self, page: int, head: int, s: int, dim: int) -> int:
        """((page * h_kv + head) * P + s) * d_h + dim   (C-3)."""
        return ((page * self.h_kv + head) * self.page_size + s) * self.d_h + dim

    def write(self, layer: int, table_row: np.ndarray, p: int, k: np.ndarray, v: np.ndarray):
        page, s = self.slot(table_row, p)
        self.K[layer, page, :, s, :] = k
        self.V[layer, page, :, s, :] = v
        self.writes.append((layer, page, s))

    def read(self, layer: int, table_row: np.ndarray, n: int) -> tuple[np.ndarray, np.ndarray]:
        """Keys/values of positions 0..n-1 in order: [n, h_kv, d_h]."""
        pos = np.arange(n)
        pages = np.asarray(table_row)[pos // self.page_size]
        if np.any(pages < 0) or np.any(pages >= self.n_pages):
            raise IndexError("page table does not cover the requested positions")
        slots = pos % self.page_size
        return self.K[layer, pages, :, slots, :], self.V[layer, pages, :, slots, :]

    def load_history(self, layer: int, table_row: np.ndarray, K: np.ndarray, V: np.ndarray):
        """Place a logical history [n, h_kv, d_h] at positions 0..n-1 (input setup, not a counted write)."""
        n = K.shape[0]
        pos = np.arange(n)
        pages = np.asarray(table_row)[pos // self.page_size]
        slots = pos % self.page_size
        self.K[layer, pages, :, slots, :] = K
        self.V[layer, pages, :, slots, :] = V


def paged_causal_attention(q: np.ndarray, pos, tables: list, kv: PagedKV, layer: int, h_kv: int) -> np.ndarray:
    """o[i, j] = softmax(q[i, j] . K_t / sqrt(d_h)) . V over t = 0..pos[i] of row i's sequence,
    K, V of kv-head floor(j / (h_q / h_kv)) gathered from the pages (readings #2, #6, #7)."""
    n, hq, dh = q.shape
    g = hq // h_kv
    scale = 1.0 / np.sqrt(dh)
    o = np.empty((n, hq, dh), dtype=np.float64)
    for i in range(n):
        Kr, Vr = kv.read(layer, tables[i], int(pos[i]) + 1)
        for j in range(hq):
            jk = j // g
            o[i, j] = attend_row(q[i, j], Kr[:, jk, :], Vr[:, jk, :], scale)
    return o


# ------------------------------------------------------------------ layer

@dataclass
class Model:
    d_model: int
    ffn_dim: int
    n_q_heads: int
    n_kv_heads: int
    head_dim: int
    rope_theta: float
    norm_eps: float

    @staticmethod
    def from_cfg(cfg) -> "Model":
        return Model(cfg.d_model, cfg.ffn_dim, cfg.n_q_heads, cfg.n_kv_heads, cfg.head_dim,
                     cfg.rope_theta, cfg.norm_eps)


def layer_forward(m: Model, w: dict, layer: int, x: np.ndarray, pos: np.ndarray,
                  tables: list, kv: PagedKV, allreduce=None) -> np.ndarray:
    """One layer over rows ``x`` [n, d]; row i is at absolute position pos[i] of the sequence
    whose page-table row is tables[i].  Steps follow C-2 in order.

    Head-sharded tensor parallelism (reading #13): with ``m`` and ``w``
    the shard of one rank (h_q/N query heads, h_kv/N kv heads, m/N FFN columns; W_qkv / W_gate_up
    rows and W_o / W_down columns of those heads and columns) and ``allreduce`` the sum over the N
    ranks, the two row-parallel projections (O and down) produce partial sums that are all-reduced
    before the residual add.  ``allreduce=None`` is the unsharded layer."""
    x = np.asarray(x, dtype=np.float64)
    n = x.shape[0]
    hq, hkv, dh = m.n_q_heads, m.n_kv_heads, m.head_dim
    # 1. h = RMSNorm(x) * g1
    h = rmsnorm(x, w["g_norm1"], m.norm_eps)
    # 2. [q | k | v] = h W_qkv^T (+ b)
    qkv = h @ np.asarray(w["w_qkv"], dtype=np.float64).T
    if w.get("b_qkv") is not None:
        qkv = qkv + np.asarray(w["b_qkv"], dtype=np.float64)
    q = qkv[:, : hq * dh].reshape(n, hq, dh)
    k = qkv[:, hq * dh: (hq + hkv) * dh].reshape(n, hkv, dh)
    v = qkv[:, (hq + hkv) * dh:].reshape(n, hkv, dh)
    # 3. RoPE on q and k at each row's absolute position
    q = rope(q, pos, m.rope_theta)
    k = rope(k, pos, m.rope_theta)
    # 4. append (k, v) of every row before any attention reads
    for i in range(n):
        kv.write(layer, tables[i], int(pos[i]), k[i], v[i])
    # 5. causal attention over the paged cache
    o = paged_causal_attention(q, pos, tables, kv, layer, hkv)
    # 6. x1 = x + o W_o^T   (TP: x + allreduce(o_shard W_o,shard^T))
    part = o.reshape(n, hq * dh) @ np.asarray(w["w_o"], dtype=np.float64).T
    x1 = x + (part if allreduce is None else allreduce(part))
    # 7. h2 = RMSNorm(x1) * g2
    h2 = rmsnorm(x1, w["g_norm2"], m.norm_eps)
    # 8. y = x1 + (silu(h2 W_g^T) * h2 W_u^T) W_d^T     (gate_up rows = [gate; up])
    gu = h2 @ np.asarray(w["w_gate_up"], dtype=np.float64).T
    mm = m.ffn_dim
    a = silu(gu[:, :mm]) * gu[:, mm:]
    part = a @ np.asarray(w["w_down"], dtype=np.float64).T
    return x1 + (part if allreduce is None else allreduce(part))


def row_parallel_allreduce(a_shards, w_shards, residual) -> np.ndarray:
    """A row-parallel linear and its allreduce (§4.1 Communication Operators; steps 6 and 8 of
    ``layer_forward`` with the ``allreduce`` hook, reading #13): rank r holds the input columns
    a_r [n][k_r] and the matching weight columns w_r [d_out][k_r], computes its partial a_r w_r^T, the
    allreduce sums the N partials, and the residual is added once:  residual + sum_r a_r w_r^T.
    The reference for SURVEY §8(f) f3 (the fused GEMM + allreduce kernel)."""
    out = np.array(residual, dtype=np.float64, copy=True)
    for a, w in zip(a_shards, w_shards):
        out = out + np.asarray(a, dtype=np.float64) @ np.asarray(w, dtype=np.float64).T
    return out


def prefill_forward(m: Model, weights: list, x: np.ndarray, seqs: list, tables: np.ndarray,
                    kv: PagedKV) -> np.ndarray:
    """All layers over the prefill rows.  seqs = [(q_s, c_s)], rows grouped by sequence in order;
    sequence s occupies positions c_s .. c_s + q_s - 1 (C-2 step 9: y feeds the next layer)."""
    pos, trows = [], []
    for s, (q, c) in enumerate(seqs):
        pos.extend(range(c, c + q))
        trows.extend([tables[s]] * q)
    pos = np.asarray(pos, dtype=np.int64)
    h = np.asarray(x, dtype=np.float64)
    for l, w in enumerate(weights):
        h = layer_forward(m, w, l, h, pos, trows, kv)
    return h


def lm_head_greedy(m: Model, head: dict, y: np.ndarray):
    """Greedy next token of each row (P:250 t_cls, P:335 'sampled tokens'):
    h = RMSNorm(y) * g_final; logits = h W_head^T; token = argmax (the lowest index among equal
    maxima).  Returns (logits [n, vocab], tokens [n])."""
    h = rmsnorm(np.asarray(y, dtype=np.float64), head["g_norm"], m.norm_eps)
    logits = h @ np.asarray(head["w_head"], dtype=np.float64).T
    return logits, np.argmax(logits, axis=1)   # numpy returns the first maximum


def decode_window(m: Model, weights: list, x: np.ndarray, ctx: list, tables: np.ndarray,
                  kv: PagedKV, k: int, head: dict | None = None, tokens_out: list | None = None) -> np.ndarray:
    """k look-ahead decode steps.  Step j (1-based) of request r is at position c_r + j - 1;
    its input is x for j = 1; otherwise the previous step's final-layer output (synthetic feedback,
    reading #26) or, with an LM head, the embedding of the previous step's greedy token (f1).
    Returns y [k, n_req, d]; with a head, tokens_out receives (logits, tokens) of every step."""
    n = len(ctx)
    out = np.empty((k, n, m.d_model), dtype=np.float64)
    h_in = np.asarray(x, dtype=np.float64)
    trows = [tables[r] for r in range(n)]
    for j in range(1, k + 1):
        pos = np.asarray([c + j - 1 for c in ctx], dtype=np.int64)
        h = h_in
        for l, w in enumerate(weights):
            h = layer_forward(m, w, l, h, pos, trows, kv)
        out[j - 1] = h
        if head is None:
            h_in = h
        else:
            logits, tok = lm_head_greedy(m, head, h)
            if tokens_out is not None:
                tokens_out.append((logits, tok))
            h_in = np.asarray(head["embed"], dtype=np.float64)[tok]
    return out


def mixed_iteration(m: Model, weights: list, x_pre, pre_seqs, pre_tables, x_dec, dec_ctx, dec_tables,
                    kv: PagedKV, k: int):
    """One mixed iteration = prefill chunk + k decode steps.  SM partitioning changes when/where
    work runs, never what is computed (the two sides touch disjoint pages), so the oracle is the
    plain sequential definition.  Returns (y_prefill [n_p, d], y_decode [k, n_d, d])."""
    y_pre = prefill_forward(m, weights, x_pre, pre_seqs, pre_tables, kv) if len(pre_seqs) else \
        np.zeros((0, m.d_model))
    y_dec = decode_window(m, weights, x_dec, dec_ctx, dec_tables, kv, k) if len(dec_ctx) else \
        np.zeros((k, 0, m.d_model))
    return y_pre, y_dec

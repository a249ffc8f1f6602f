"""Test helper: place a synth workload on the GPU and run it through libduet.so's C ABI."""
from __future__ import annotations

import numpy as np
import torch

import paper_2511_04791_b200 as D


def torch_dtype(dtype: str):
    return torch.bfloat16 if dtype == "bf16" else torch.float32


def duet_dtype(dtype: str):
    return D.DUET_DTYPE_BF16 if dtype == "bf16" else D.DUET_DTYPE_FP32


def spec_of(model, dtype: str):
    return D.make_spec(model.n_layers, model.d_model, model.ffn_dim, model.n_q_heads, model.n_kv_heads,
                       model.head_dim, model.vocab, 2 if dtype == "bf16" else 4, int(model.ffn_gated),
                       int(model.qkv_bias), model.tp, model.rope_theta, model.norm_eps)


class GpuWorkload:
    def __init__(self, wl, dtype: str, device="cuda", poison=True):
        self.wl = wl
        self.dtype = dtype
        tdt = torch_dtype(dtype)
        m = wl.cfg.model
        self.W = [{k: torch.from_numpy(np.ascontiguousarray(v)).to(device=device, dtype=tdt)
                   for k, v in w.items() if v is not None} for w in wl.weights]
        fill = float("nan") if poison else 0.0
        shape = (wl.n_pages, m.n_kv_heads, wl.cfg.batch.page_size, m.head_dim)
        self.K = [torch.full(shape, fill, dtype=tdt, device=device) for _ in range(wl.n_layers)]
        self.V = [torch.full(shape, fill, dtype=tdt, device=device) for _ in range(wl.n_layers)]
        P = wl.cfg.batch.page_size
        for l, trow, uid, n in wl.history_items():
            Kh, Vh = wl.history(l, uid, n)
            p = np.arange(n)
            pages = torch.from_numpy(trow[p // P].astype(np.int64)).to(device)
            slots = torch.from_numpy((p % P).astype(np.int64)).to(device)
            self.K[l][pages, :, slots, :] = torch.from_numpy(Kh).to(device=device, dtype=tdt)
            self.V[l][pages, :, slots, :] = torch.from_numpy(Vh).to(device=device, dtype=tdt)
        self.x_pre = torch.from_numpy(wl.x_pre).to(device=device, dtype=tdt)
        self.x_dec = torch.from_numpy(wl.x_dec).to(device=device, dtype=tdt)
        self.y_pre = torch.zeros_like(self.x_pre)
        self.y_dec = torch.zeros((wl.k,) + tuple(self.x_dec.shape), dtype=tdt, device=device)

    def prefill_arg(self):
        if not self.wl.pre_seqs:
            return None
        return dict(q=[q for q, _ in self.wl.pre_seqs], c=[c for _, c in self.wl.pre_seqs],
                    table=self.wl.pre_tables, x=self.x_pre, y=self.y_pre)

    def add_head(self, head: dict, device="cuda"):
        """LM head (f1): synth.head_weights on the GPU + a tokens [k][n_dec] output."""
        tdt = torch_dtype(self.dtype)
        self.head = {k: torch.from_numpy(np.ascontiguousarray(v)).to(device=device, dtype=tdt) for k, v in head.items()}
        self.head["tokens"] = torch.full((self.wl.k, len(self.wl.dec_ctx)), -1, dtype=torch.int32, device=device)

    def decode_arg(self):
        if not self.wl.dec_ctx:
            return None
        return dict(c=self.wl.dec_ctx, table=self.wl.dec_tables, x=self.x_dec, y=self.y_dec,
                    head=getattr(self, "head", None))

    def step(self, ctx: D.Ctx, split, stream=None):
        ctx.step(self.W, self.prefill_arg(), self.decode_arg(), self.K, self.V, self.wl.n_pages, split, stream)


def make_ctx(wl, dtype: str, flags=0, extra_tokens=0):
    m = wl.cfg.model
    n_p = sum(q for q, _ in wl.pre_seqs)
    max_pages = max([wl.pre_tables.shape[1] if len(wl.pre_tables) else 1,
                     wl.dec_tables.shape[1] if len(wl.dec_tables) else 1])
    max_pos = max([c + q for q, c in wl.pre_seqs] + [c + wl.k for c in wl.dec_ctx] + [16])
    return D.Ctx(spec_of(m, dtype), max(n_p + extra_tokens, 1), max(len(wl.pre_seqs), 1), max(len(wl.dec_ctx), 1),
                 max(wl.k, 1), max_pages, max_pos + 16, duet_dtype(dtype), flags)

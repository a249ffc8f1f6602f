"""Configuration presets; dimensions only, no arithmetic of the method.

cfg1..cfg5 follow BASELINE.json ``configs`` in order.  Readings of values the
paper/baseline leave open are listed in DESIGN.md ("Readings", #29-#30).
"""
from __future__ import annotations

from dataclasses import dataclass, field, replace


@dataclass(frozen=True)
class ModelCfg:
    name: str
    n_layers: int
    d_model: int
    ffn_dim: int
    n_q_heads: int
    n_kv_heads: int
    head_dim: int
    vocab: int = 128256
    qkv_bias: bool = False
    rope_theta: float = 10000.0
    norm_eps: float = 1e-5
    ffn_gated: bool = True
    tp: int = 1


@dataclass(frozen=True)
class BatchCfg:
    # prefill sequences: list of (q, c) = (new tokens, cached prefix tokens)
    prefill: tuple = ()
    # decode requests: cached length c_r before step 1
    decode: tuple = ()
    k: int = 1
    page_size: int = 16
    tbt_slo_s: float = 0.1


@dataclass(frozen=True)
class Config:
    name: str
    model: ModelCfg
    batch: BatchCfg
    dtype: str = "bf16"
    seed: int = 4791
    note: str = ""


TINY = ModelCfg("tiny", n_layers=1, d_model=256, ffn_dim=1024, n_q_heads=4, n_kv_heads=4, head_dim=64,
                vocab=1024, rope_theta=1e4, norm_eps=1e-5)
TINY_GQA = replace(TINY, name="tiny-gqa", n_kv_heads=2)
LLAMA3_8B_LAYER = ModelCfg("llama-3-8b-layer", n_layers=1, d_model=4096, ffn_dim=14336, n_q_heads=32,
                           n_kv_heads=8, head_dim=128, vocab=128256, rope_theta=5e5, norm_eps=1e-5)
LLAMA3_8B = replace(LLAMA3_8B_LAYER, name="llama-3-8b", n_layers=32)
QWEN25_14B = ModelCfg("qwen2.5-14b", n_layers=48, d_model=5120, ffn_dim=13824, n_q_heads=40, n_kv_heads=8,
                      head_dim=128, vocab=152064, qkv_bias=True, rope_theta=1e6, norm_eps=1e-6)
LLAMA3_70B_SLICE = ModelCfg("llama-3-70b-8layer", n_layers=8, d_model=8192, ffn_dim=28672, n_q_heads=64,
                            n_kv_heads=8, head_dim=128, vocab=128256, rope_theta=5e5, norm_eps=1e-5)

CONFIGS = {
    "cfg1": Config("cfg1", TINY, BatchCfg(prefill=((128, 0),), decode=(256,) * 8, k=2), dtype="fp32",
                   seed=4791 + 1, note="tiny layer fp32; splits swept exhaustively"),
    "cfg1-bf16": Config("cfg1-bf16", TINY, BatchCfg(prefill=((128, 0),), decode=(256,) * 8, k=2), dtype="bf16",
                        seed=4791 + 1),
    "cfg1-gqa": Config("cfg1-gqa", TINY_GQA, BatchCfg(prefill=((128, 64),), decode=(256,) * 8, k=4), dtype="fp32",
                       seed=4791 + 1),
    "cfg2-mini": Config("cfg2-mini", LLAMA3_8B_LAYER,
                        BatchCfg(prefill=((200, 37), (77, 0), (520, 300)), decode=(300, 17, 1029), k=3),
                        dtype="bf16",
                        seed=4791 + 2, note="Llama-3-8B layer shapes, ragged small batch (parity only)"),
    "cfg4-mini": Config("cfg4-mini", replace(QWEN25_14B, name="qwen2.5-14b-layer", n_layers=1),
                        BatchCfg(prefill=((300, 0), (129, 45)), decode=(700, 33, 2049, 5), k=2), dtype="bf16",
                        seed=4791 + 4, note="Qwen2.5-14B layer shapes (GQA 5, QKV bias), ragged (parity only)"),
    "cfg2": Config("cfg2", LLAMA3_8B_LAYER, BatchCfg(prefill=((2048, 0),), decode=(4096,) * 64, k=1,
                                                     tbt_slo_s=50e-3 / 32), dtype="bf16", seed=4791 + 2,
                   note="Llama-3-8B single layer: prefill chunk 2048 + 64 decodes at ctx 4k"),
    "cfg3": Config("cfg3", LLAMA3_8B, BatchCfg(prefill=((8192, 0),),
                                               decode=tuple(2048 + (6144 * r) // 255 for r in range(256)), k=1,
                                               tbt_slo_s=50e-3), dtype="bf16", seed=4791 + 3,
                   note="Llama-3-8B 32 layers: 8k prompt into 256 decodes at ctx 2k-8k, TBT SLO 50 ms"),
    # cfg3 with the context ramp narrowed to 2k-6k so that 32 layers of KV (about 129 GiB) plus weights and
    # workspace fit one 180 GB B200 (SURVEY.md §8(d) fallback); used when the full ramp does not fit
    "cfg3-fit": Config("cfg3-fit", LLAMA3_8B, BatchCfg(prefill=((8192, 0),),
                                                       decode=tuple(2048 + (4096 * r) // 255 for r in range(256)),
                                                       k=1, tbt_slo_s=50e-3), dtype="bf16", seed=4791 + 3,
                       note="Llama-3-8B 32 layers: 8k prompt into 256 decodes at ctx 2k-6k (fits 180 GB), "
                            "TBT SLO 50 ms"),
    # cfg5: Llama-3-70B-shaped 8-layer slice, head-sharded TP = 2/4/8 (bench.py --tp N); the TBT SLO is
    # 50 ms scaled to the 8 of 80 layers
    "cfg5": Config("cfg5", LLAMA3_70B_SLICE, BatchCfg(prefill=((16384, 0),), decode=(4096,) * 512, k=1,
                                                      tbt_slo_s=50e-3 * 8 / 80), dtype="bf16", seed=4791 + 5,
                   note="Llama-3-70B shapes, 8 layers: 16k prefill chunk + 512 decodes at ctx 4k, TP over NVLink"),
}


def get_config(name: str) -> Config:
    return CONFIGS[name]

"""Head-sharded tensor-parallel slices of a layer's weights and KV pools.

Input preparation only (no arithmetic of the method): rank r of N holds query heads
[r h_q/N, (r+1) h_q/N), kv heads [r h_kv/N, (r+1) h_kv/N) and FFN columns [r m/N, (r+1) m/N):
  * W_qkv rows: its q-head rows, its k-head rows, its v-head rows (column-parallel), b_qkv likewise;
  * W_o columns: its q heads (row-parallel: the O projection yields a partial sum);
  * W_gate_up rows: its gate rows then its up rows (column-parallel; gate row j pairs with up row j);
  * W_down columns: its FFN columns (row-parallel);
  * norm gains are replicated; the KV pool holds its kv heads only.
Works on numpy arrays and torch tensors alike (plain slicing / concatenation).
"""
from __future__ import annotations


def _cat(parts):
    import numpy as np
    if isinstance(parts[0], np.ndarray):
        return np.concatenate(parts, axis=0)
    import torch
    return torch.cat(parts, dim=0)


def shard_dims(hq: int, hkv: int, m: int, rank: int, world: int):
    if hq % world or hkv % world or m % world:
        raise ValueError(f"h_q={hq}, h_kv={hkv}, m={m} not divisible by tp={world}")
    return hq // world, hkv // world, m // world


def shard_layer_weights(w: dict, hq: int, hkv: int, dh: int, m: int, rank: int, world: int) -> dict:
    """Rank `rank`'s shard of one layer's weights (keys as in oracle.layer / duet_layer_weights)."""
    if world == 1:
        return dict(w)
    lq, lkv, lm = shard_dims(hq, hkv, m, rank, world)
    q0, k0, v0 = rank * lq * dh, hq * dh + rank * lkv * dh, (hq + hkv) * dh + rank * lkv * dh
    out = dict(w)
    out["w_qkv"] = _cat([w["w_qkv"][q0:q0 + lq * dh], w["w_qkv"][k0:k0 + lkv * dh], w["w_qkv"][v0:v0 + lkv * dh]])
    if w.get("b_qkv") is not None:
        out["b_qkv"] = _cat([w["b_qkv"][q0:q0 + lq * dh], w["b_qkv"][k0:k0 + lkv * dh], w["b_qkv"][v0:v0 + lkv * dh]])
    out["w_o"] = w["w_o"][:, rank * lq * dh:(rank + 1) * lq * dh]
    out["w_gate_up"] = _cat([w["w_gate_up"][rank * lm:(rank + 1) * lm], w["w_gate_up"][m + rank * lm:m + (rank + 1) * lm]])
    out["w_down"] = w["w_down"][:, rank * lm:(rank + 1) * lm]
    for k in ("w_o", "w_down"):
        out[k] = out[k].copy() if hasattr(out[k], "copy") and not hasattr(out[k], "contiguous") else out[k].contiguous()
    return out


def shard_kv_pool(pool, hkv: int, rank: int, world: int):
    """pool [..., n_pages, h_kv, P, d_h] -> this rank's kv heads (contiguous)."""
    if world == 1:
        return pool
    l = hkv // world
    sl = pool[..., rank * l:(rank + 1) * l, :, :]
    return sl.copy() if hasattr(sl, "copy") and not hasattr(sl, "contiguous") else sl.contiguous()

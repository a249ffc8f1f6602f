"""Multi-process host logic of bench.py at world_size 2 over gloo (CPU): the max-over-ranks timing and the
whole-job aggregate of independent replicas ('replicas only')."""
import os
import socket

import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, ws, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(ws))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    import bench
    local_t = 1.0 + rank          # rank 1 is slower
    v, tmax = bench.whole_job_rate(1000.0, local_t, ws)
    bench.barrier(ws)
    q.put((rank, v, tmax))
    dist.destroy_process_group()


def test_replicas_max_over_ranks_gloo():
    ws = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, ws, port, q)) for r in range(ws)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(ws)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, v, tmax in res:
        assert tmax == 2.0                 # max over ranks
        assert v == pytest.approx(1000.0 * 2 / 2.0)


def _tp_worker(rank, ws, port, q):
    """Rank `rank` of a head-sharded TP group: its weight and KV shards (synth.tp), the
    oracle layer with the row-parallel partial sums all-reduced over gloo."""
    import numpy as np
    import torch
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(ws))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    from dataclasses import replace
    from oracle import layer as OL
    from synth import configs, tp, workload
    from tests.oracle_run import make_kv
    cfg = configs.get_config("cfg1-gqa")
    wl = workload.build(cfg, k=2)
    m = cfg.model
    full = OL.Model.from_cfg(m)
    lq, lkv, lm = tp.shard_dims(m.n_q_heads, m.n_kv_heads, m.ffn_dim, rank, ws)
    local = replace(full, n_q_heads=lq, n_kv_heads=lkv, ffn_dim=lm)
    weights = [tp.shard_layer_weights(w, m.n_q_heads, m.n_kv_heads, m.head_dim, m.ffn_dim, rank, ws)
               for w in wl.weights]
    kv_full = make_kv(wl)
    kv = OL.PagedKV(wl.n_layers, wl.n_pages, lkv, cfg.batch.page_size, m.head_dim)
    kv.K = tp.shard_kv_pool(kv_full.K, m.n_kv_heads, rank, ws)
    kv.V = tp.shard_kv_pool(kv_full.V, m.n_kv_heads, rank, ws)

    def allreduce(part):
        t = torch.from_numpy(np.ascontiguousarray(part))
        dist.all_reduce(t)
        return t.numpy()

    pos, trows = [], []
    for s, (qn, c) in enumerate(wl.pre_seqs):
        pos.extend(range(c, c + qn))
        trows.extend([wl.pre_tables[s]] * qn)
    y_tp = OL.layer_forward(local, weights[0], 0, wl.x_pre, np.asarray(pos), trows, kv, allreduce=allreduce)
    if rank == 0:
        y_ref = OL.layer_forward(full, wl.weights[0], 0, wl.x_pre, np.asarray(pos), trows, kv_full)
        q.put(float(np.max(np.abs(y_tp - y_ref)) / np.max(np.abs(y_ref))))
    dist.barrier()
    dist.destroy_process_group()


def test_tp_head_sharded_oracle_equals_unsharded_gloo():
    """The head-sharded TP recipe (synth.tp slices + allreduce after O and down) reproduces the
    unsharded layer: SURVEY §8(c) C-8 'TP shards summed equal unsharded', at world size 2 over gloo."""
    ws = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_tp_worker, args=(r, ws, port, q)) for r in range(ws)]
    for p in procs:
        p.start()
    err = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
    assert err < 1e-12, err


class _FakeArCtx:
    """Stands in for D.Ctx in the f3 handle exchange (no GPU): a rank-specific 64-byte handle."""

    def __init__(self, rank):
        self.rank = rank
        self.opened = None

    def ar_handle(self):
        return bytes([65 + self.rank]) * 64

    def ar_open(self, handles):
        self.opened = list(handles)


def _ar_worker(rank, ws, port, q):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(ws))
    dist.init_process_group("gloo", rank=rank, world_size=ws)
    from paper_2511_04791_b200._native import open_fused_allreduce
    c = _FakeArCtx(rank)
    open_fused_allreduce(c)
    q.put((rank, c.opened))
    dist.destroy_process_group()


def test_fused_allreduce_handle_exchange_gloo():
    """f3 plumbing (D.open_fused_allreduce): every rank opens the group with all ranks' arena handles in
    rank order — the layout duet_ctx_ar_open indexes its peer tables by (world size 2, gloo)."""
    ws = 2
    port = _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_ar_worker, args=(r, ws, port, q)) for r in range(ws)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in range(ws))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = [bytes([65 + r]) * 64 for r in range(ws)]
    assert res[0] == want and res[1] == want

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

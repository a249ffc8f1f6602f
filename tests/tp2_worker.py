"""Worker of tests/test_gpu_tp2.py (one process per GPU, launched by torch.distributed.run): rank r runs
its head shard of a cfg2-mini mixed iteration (synth.tp: h_q/2 query heads, h_kv/2 kv heads, ffn/2
columns) through libduet.so with real NCCL communicators, in temporal and spatial mode, with the NCCL
allreduce and with the fused GEMM + allreduce (f3, IPC-mapped peer arenas); the
all-reduced layer outputs must equal the UNSHARDED oracle on every rank (§8 a9)."""
import os
import sys
from dataclasses import replace

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    import torch.distributed as dist
    import paper_2511_04791_b200 as D
    from synth import configs, workload
    from synth import tp as TP
    from tests.gpu_helpers import GpuWorkload, make_ctx
    from tests.oracle_run import rel_err, run

    rank, ws = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
    cfg = configs.get_config("cfg2-mini")
    wl = workload.build(cfg, k=2)
    m = wl.cfg.model
    y_pre, y_dec, _ = run(wl)                       # the unsharded oracle
    wl1 = workload.build(cfg, k=1)
    y_pre1, y_dec1, _ = run(wl1)
    wl_tp = replace(wl, cfg=replace(wl.cfg, model=replace(m, tp=ws)))
    ids = [D.nccl_unique_id(), D.nccl_unique_id()] if rank == 0 else [None, None]
    dist.broadcast_object_list(ids, src=0)
    worst = 0.0
    for mode, fused in (("temporal", False), ("spatial", False), ("temporal", True), ("spatial", True)):
        src = wl1 if mode == "temporal" else wl
        g = GpuWorkload(src, "bf16")
        g.W = [TP.shard_layer_weights(w, m.n_q_heads, m.n_kv_heads, m.head_dim, m.ffn_dim, rank, ws) for w in g.W]
        g.K = [TP.shard_kv_pool(p, m.n_kv_heads, rank, ws) for p in g.K]
        g.V = [TP.shard_kv_pool(p, m.n_kv_heads, rank, ws) for p in g.V]
        ctx = make_ctx(replace(src, cfg=replace(src.cfg, model=replace(m, tp=ws))), "bf16")
        ctx.set_comms(rank, ids[0], ids[1])
        if fused:  # f3: O / down + allreduce fused over peer memory (IPC-mapped arenas)
            D.open_fused_allreduce(ctx)
        parts, total = ctx.partitions()
        split = D.split_struct(D.DUET_MODE_TEMPORAL, total, 0, 1) if mode == "temporal" else \
            D.split_struct(D.DUET_MODE_SPATIAL, total - parts[len(parts) // 2], parts[len(parts) // 2], 2)
        g.step(ctx, split)
        torch.cuda.synchronize()
        ctx.check_comms()
        yp, yd = (y_pre1, y_dec1) if mode == "temporal" else (y_pre, y_dec)
        e = rel_err(g.y_pre.float().cpu().numpy(), yp)
        for j in range(src.k):
            e = max(e, rel_err(g.y_dec[j].float().cpu().numpy(), yd[j]))
        print(f"rank {rank} {mode}{' fused' if fused else ''}: rel_err {e:.3e}", flush=True)
        worst = max(worst, e)
        ctx.close()
    dist.destroy_process_group()
    if worst > 2e-2:
        raise SystemExit(f"rank {rank}: rel_err {worst} > 2e-2")


if __name__ == "__main__":
    main()

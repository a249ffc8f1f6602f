#!/usr/bin/env python
"""DuetServe mixed-iteration hot path on B200 — benchmark (driver contract, one JSON line).

A step = one pass of the whole hot path over one mixed batch:
  a1/a2  duet_choose_split (roofline predictor + Alg. 1, host C++, against the tables measured by
         duet_calibrate at start-up),
  a3-a7  duet_step: metadata staging, partition binding, k decode steps (CUDA-graph replays on the
         S_d partition) concurrently with the prefill chunk (S_p partition), join.
Workload (N=1): cfg3 of BASELINE.json, the largest single-GPU configuration — Llama-3-8B, 32 layers,
bf16: an 8k-token prompt arriving into 256 in-flight decodes at ctx 2k-8k, TBT SLO 50 ms (cfg3-fit, the
2k-6k ramp, when the full ramp's KV does not fit next to the weights).  `--config cfg2` runs the
single-layer configuration (prefill 2048 + 64 decodes at 4k, tau = 50/32 ms).  Synthetic seeded inputs
(synth/), random weights of that architecture.

metric: tokens/s per mixed iteration = (k T_dec + T_pre) / window, summed over ranks (each rank
runs an independent replica: "replicas only" data parallelism, weak scaling).

--impl reference runs the CPU oracle (oracle/, numpy float64) on a bounded sample of the same
workload, rank 0 only.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "tokens/s per mixed iteration at TBT SLO vs SM split; % HBM/TC roofline"
FALLBACK_PEAKS = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}


_T0 = time.time()


def log(msg: str):
    """Progress on stderr (the JSON line is the only stdout output)."""
    sys.stderr.write(f"[bench {time.time() - _T0:7.1f}s] {msg}\n")
    sys.stderr.flush()


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return d, "measured (MEASURED_PEAKS.json)"
    return FALLBACK_PEAKS, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """SM clocks / clock-event (throttle) reasons sampled through NVML every ~2 ms during the timed
    region (nvidia-smi's 50 ms floor misses a region of a few tens of ms); stop() always takes one
    last sample before the caller's post-region synchronize returns control."""

    REASONS = (("hw_slowdown", "nvmlClocksEventReasonHwSlowdown"),
               ("hw_thermal_slowdown", "nvmlClocksEventReasonHwThermalSlowdown"),
               ("sw_thermal_slowdown", "nvmlClocksEventReasonSwThermalSlowdown"),
               ("sw_power_cap", "nvmlClocksEventReasonSwPowerCap"),
               ("hw_power_brake_slowdown", "nvmlClocksEventReasonHwPowerBrakeSlowdown"))

    def __init__(self, index=0):
        self.samples = []
        self.index = index
        self.nv = None
        self.run = False

    def _sample(self):
        nv = self.nv
        sm = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
        mask = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
        self.samples.append((sm, mask))

    def _loop(self):
        while self.run:
            try:
                self._sample()
            except Exception:
                return
            time.sleep(0.002)

    def start(self):
        try:
            import pynvml as nv
            nv.nvmlInit()
            self.nv = nv
            self.h = nv.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM)
            self.run = True
            self.th = threading.Thread(target=self._loop, daemon=True)
            self.th.start()
        except Exception:
            self.nv = None

    def stop(self):
        if self.nv is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        try:
            self._sample()
        except Exception:
            pass
        self.run = False
        self.th.join(timeout=1)
        sm = sorted(s[0] for s in self.samples)
        reasons = sorted({name for _, m in self.samples for name, attr in self.REASONS
                          if m & getattr(self.nv, attr, 0)})
        return {"sm_mhz": sm[len(sm) // 2] if sm else None, "sm_max_mhz": self.max_mhz, "reasons": reasons,
                "samples": len(self.samples), "source": "nvml"}


def dist_init():
    import torch
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    lrank = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1:
        import torch.distributed as dist
        torch.cuda.set_device(lrank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", lrank))
    else:
        if torch.cuda.is_available():
            torch.cuda.set_device(0)
    return ws, rank, lrank


def max_over_ranks(x: float, ws: int) -> float:
    if ws == 1:
        return x
    import torch
    import torch.distributed as dist
    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def whole_job_rate(units_local: float, seconds_local: float, ws: int) -> tuple:
    """value = units all ranks processed / max over ranks of the device-timed region (weak scaling:
    every rank runs the same replica workload, so units_all = units_local * ws)."""
    t_max = max_over_ranks(seconds_local, ws)
    return units_local * ws / t_max, t_max


def barrier(ws):
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()


# ----------------------------------------------------------------------------- oracle arm

class OracleSample:
    """The CPU oracle on a bounded sample of the workload, one layer: two prefill chunks of n_pre/2 rows
    each — the first rows of the prompt (c = 0) and its last rows (c = prompt - n_pre/2, the prefix given
    as KV history) — so the sample's mean attention cost per row is the prompt's (causal cost is linear
    in the position), plus n_dec decode requests spread evenly over the batch's context ramp.  Inputs
    are prepared once (not timed); run() times one oracle mixed iteration, returns (tokens, seconds)."""

    def __init__(self, cfg_name: str, n_pre: int, n_dec: int):
        import numpy as np
        from synth import configs, workload
        from tests.oracle_run import make_kv
        from oracle import layer as OL
        cfg = configs.get_config(cfg_name)
        # one layer of the configuration; deeper models are extrapolated per layer
        self.layers_total = cfg.model.n_layers
        n_full = sum(q for q, _ in cfg.batch.prefill)
        h = max(1, min(n_pre // 2, n_full // 2))
        dec_all = list(cfg.batch.decode)
        pick = [dec_all[int(i * (len(dec_all) - 1) / max(1, n_dec - 1))] for i in range(n_dec)] if n_dec else []
        wl = workload.build(cfg, pre_seqs=[(h, 0), (h, n_full - h)], dec_ctx=pick, k=1, n_layers=1)
        wl.weights = [{k_: (None if v is None else np.asarray(v, dtype=np.float64)) for k_, v in w.items()}
                      for w in wl.weights]
        self.wl, self.kv, self.OL = wl, make_kv(wl), OL
        self.mdl = OL.Model.from_cfg(wl.cfg.model)
        # tokens per second of the whole model = tokens / (time of one layer x layers)
        self.tokens = (2 * h + n_dec) / self.layers_total
        self.desc = (f"oracle (numpy float64) on {cfg_name}: prompt rows 0..{h - 1} and {n_full - h}..{n_full - 1} "
                     f"of the {n_full}-token chunk (the tail with its prefix as KV history) + {n_dec} of the "
                     f"{len(dec_all)} decodes spread over the context ramp, one layer"
                     + (f", extrapolated x{self.layers_total} layers" if self.layers_total > 1 else ""))

    def run(self):
        wl = self.wl
        t = time.perf_counter()
        self.OL.mixed_iteration(self.mdl, wl.weights, wl.x_pre, wl.pre_seqs, wl.pre_tables, wl.x_dec, wl.dec_ctx,
                                wl.dec_tables, self.kv, wl.k)
        return self.tokens, time.perf_counter() - t


def oracle_baseline(cfg_name: str, budget_s: float = 12.0):
    """cpu_baseline: repeat the (2 x 64 prompt rows + 4 decodes) sample for about budget_s seconds."""
    smp = OracleSample(cfg_name, 128, 4)
    tok = sec = 0.0
    n = 0
    while sec < budget_s or n < 2:
        a, b = smp.run()
        tok += a
        sec += b
        n += 1
    return tok / sec, f"{smp.desc}; {n} repetitions, {sec:.1f} s"


def oracle_cores():
    """Threads the oracle's BLAS actually uses (numpy matmuls are its only parallel part)."""
    try:
        from threadpoolctl import threadpool_info
        th = max((i.get("num_threads", 1) for i in threadpool_info()), default=1)
    except Exception:
        th = os.cpu_count()
    return int(th)


def host_cores():
    return {"nproc": os.cpu_count(), "blas_threads": oracle_cores()}


def run_reference(args, ws, rank):
    if rank != 0:
        return
    # per-step sample sized so that warmup + steps stay within ~2-3 minutes of CPU time
    n_steps = args.steps + args.warmup
    # (~2.9 s per 128-row + 4-decode cfg3 sample on 16 host threads)
    smp = OracleSample(args.config, 128, 4) if n_steps <= 30 else \
        OracleSample(args.config, 64, 2) if n_steps <= 120 else OracleSample(args.config, 32, 2)
    for _ in range(args.warmup):
        smp.run()
    tok = sec = 0.0
    for _ in range(args.steps):
        a, b = smp.run()
        tok += a
        sec += b
    v = tok / sec
    desc = smp.desc + ", per step"
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": "tokens/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": sec / args.steps * 1e3,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": args.config, "sample": desc},
            "cpu_baseline": {"value": v, "unit": "tokens/s", "cores": oracle_cores(), "kind": "oracle",
                             "sample": desc, "host": host_cores()},
            "e2e": {"value": v, "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------- duet arm

def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="duet", choices=["duet", "reference"])
    ap.add_argument("--config", default="cfg3",
                    help="cfg3 (the largest single-GPU config; cfg3-fit when the full ramp does not fit) or cfg2")
    ap.add_argument("--mode", default="auto", choices=["auto", "temporal", "spatial"])
    ap.add_argument("--tau", type=float, default=None, help="TBT SLO per iteration, seconds")
    ap.add_argument("--sweep", action="store_true",
                    help="also time every SM split at its Alg. 1 k, measured vs predicted (Fig. 7/8 table)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--calibration", default="corun", choices=["corun", "burst"],
                    help="predictor tables: co-run at sustained clocks (default) or standalone bursts")
    ap.add_argument("--profile-only", action="store_true", help="a few steps, no extras (for ncu)")
    ap.add_argument("--split", default=None, help="S_d,k: run this spatial split instead of Alg. 1's (profiling)")
    ap.add_argument("--fine-split", action="store_true",
                    help="2-SM (TPC) partition granularity (DUET_CTX_FINE_SPLIT) instead of the driver's 8-SM default")
    ap.add_argument("--lm-head", action="store_true",
                    help="close the decode window with the LM head + greedy tokens (f1; t_cls in the predictor)")
    ap.add_argument("--tp", type=int, default=1,
                    help="head-sharded tensor parallelism over the torchrun ranks (= WORLD_SIZE; default config "
                         "cfg5): one batch per step across all ranks, NCCL allreduce after O and down")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3 if not args.profile_only else args.warmup)

    ws, rank, lrank = dist_init()
    if args.impl == "reference":
        run_reference(args, ws, rank)
        return

    import numpy as np
    import torch
    import paper_2511_04791_b200 as D
    from synth import configs, workload
    from synth.gpu import inputs_gpu, kv_pools_gpu, layer_weights_gpu

    if args.config == "cfg3":   # full 2k-8k ramp needs ~187 GB with weights; fall back when it does not fit
        free, _ = torch.cuda.mem_get_info()
        if free < 190e9:
            args.config = "cfg3-fit"
    tp = args.tp
    if tp > 1 and tp != ws:
        raise SystemExit(f"--tp {tp} needs WORLD_SIZE = {tp} (torchrun --nproc-per-node {tp})")
    if tp > 1 and args.config in ("cfg2", "cfg3", "cfg3-fit"):
        args.config = "cfg5"
    cfg = configs.get_config(args.config)
    dev = torch.device("cuda", torch.cuda.current_device())
    tdt = torch.bfloat16 if cfg.dtype == "bf16" else torch.float32
    m = cfg.model
    k_max = 8                                            # look-ahead window cap (reading #17)
    nqkv = (m.n_q_heads + 2 * m.n_kv_heads) * m.head_dim
    step_bytes = m.n_layers * 2 * (nqkv * m.d_model + m.d_model * m.n_q_heads * m.head_dim + 3 * m.ffn_dim * m.d_model
                                   + sum(2 * m.n_kv_heads * m.head_dim * (c + 1) for c in cfg.batch.decode))
    wl = workload.build(cfg, k=k_max, with_weights=False)  # pages for up to k_max look-ahead steps
    log(f"config {args.config}: generating weights")
    if tp > 1:   # this rank's head shard (synth.tp; the full layer is generated, sliced, freed)
        from synth import tp as TP
        W = [TP.shard_layer_weights(layer_weights_gpu(m, l, cfg.seed, dev, tdt), m.n_q_heads, m.n_kv_heads,
                                    m.head_dim, m.ffn_dim, rank, tp) for l in range(m.n_layers)]
    else:
        W = [layer_weights_gpu(m, l, cfg.seed, dev, tdt) for l in range(m.n_layers)]
    x_pre, x_dec = inputs_gpu(wl, dev, tdt)
    head = None
    if args.lm_head:   # f1: LM head + embedding (vocab x d each) and a tokens [8][n_d] output
        from synth.gpu import head_weights_gpu
        head = head_weights_gpu(m, cfg.seed, dev, tdt)
        head["tokens"] = torch.zeros((8, len(wl.dec_ctx)), dtype=torch.int32, device=dev)
    torch.cuda.empty_cache()  # hand the generator's temporaries back: libduet allocates with cudaMalloc
    n_p, n_d = x_pre.shape[0], x_dec.shape[0]
    y_pre = torch.empty_like(x_pre)
    y_dec = torch.empty((8,) + tuple(x_dec.shape), dtype=tdt, device=dev)
    spec = D.make_spec(m.n_layers, m.d_model, m.ffn_dim, m.n_q_heads, m.n_kv_heads, m.head_dim, m.vocab,
                       2 if cfg.dtype == "bf16" else 4, 1, int(m.qkv_bias), tp, m.rope_theta, m.norm_eps)
    max_pages = max(wl.pre_tables.shape[1], wl.dec_tables.shape[1])
    max_pos = max([c + q for q, c in wl.pre_seqs] + [c + 8 for c in wl.dec_ctx]) + 16
    ctx = D.Ctx(spec, n_p, len(wl.pre_seqs), n_d, 8, max_pages, max_pos,
                D.DUET_DTYPE_BF16 if cfg.dtype == "bf16" else D.DUET_DTYPE_FP32,
                D.DUET_CTX_FINE_SPLIT if args.fine_split else 0)
    parts, total = ctx.partitions()
    nvl_bw, ar_alpha = 900e9, 3e-6
    if tp > 1:
        import torch.distributed as dist
        ids = [D.nccl_unique_id(), D.nccl_unique_id()] if rank == 0 else [None, None]
        dist.broadcast_object_list(ids, src=0)
        ctx.set_comms(rank, ids[0], ids[1])
        ar_alpha, nvl_bw = ctx.calibrate_allreduce()   # P:237 alpha and B_NVLink, measured

    # L0 calibration: Pi_SM(S), B_HBM(S) on this GPU with our kernels
    t0 = time.perf_counter()
    if args.profile_only:   # no calibration launches under a profiler: linear tables from the measured peaks
        pk0, _ = peaks()
        fl = [0.0] + [float(pk0["bf16_tflops"]) * 1e12 * s_ / total for s_ in range(1, total + 1)]
        bw = [0.0] + [float(pk0["hbm_gbs"]) * 1e9 * min(1.0, (s_ / total) ** 0.32) for s_ in range(1, total + 1)]
    elif args.calibration == "burst":
        fl, bw = ctx.calibrate(total)
    else:   # the rates each side achieves next to the other side's work, at sustained clocks (reading R-f)
        fl, bw = ctx.calibrate_corun(total, 0.2)
    t_cal = time.perf_counter() - t0
    # the hardware read-stream ceiling per partition size (decode-side roofline denominator), before the
    # KV pools take the memory
    stream_bw = ctx.calibrate_stream(total) if not args.profile_only else None
    hw = D.HwProfile(total, parts, fl, bw, nvlink_bw=nvl_bw, allreduce_alpha=ar_alpha)
    log(f"calibrated in {t_cal:.1f}s; generating the KV history")
    Kp, Vp = kv_pools_gpu(wl, dev, tdt)   # after calibration: the pools take most of HBM at cfg3
    if tp > 1:
        from synth import tp as TP
        for l in range(len(Kp)):
            Kp[l] = TP.shard_kv_pool(Kp[l], m.n_kv_heads, rank, tp)
            Vp[l] = TP.shard_kv_pool(Vp[l], m.n_kv_heads, rank, tp)
    log("KV ready; warm-up")
    torch.cuda.empty_cache()
    tau = args.tau if args.tau is not None else cfg.batch.tbt_slo_s
    # emits_logits: the decode rows when the LM head runs (P:250 t_cls over the entries that emit logits)
    batch = [(q, c, 0 if c == 0 else 1, 0) for q, c in wl.pre_seqs] + \
        [(1, c, 2, 1 if head is not None else 0) for c in wl.dec_ctx]
    opts = (D.DUET_OPT_FORCE_SPATIAL if args.mode == "spatial" else 0) | (D.DUET_OPT_INCLUDE_CLS if head is not None else 0)

    def decide():
        if args.mode == "temporal":
            return D.split_struct(D.DUET_MODE_TEMPORAL, total, 0, 1)
        if args.split:   # a fixed (S_d, k) — e.g. a profiler run reproducing a measured run's split
            sd_, k_ = (int(x) for x in args.split.split(","))
            return D.split_struct(D.DUET_MODE_SPATIAL, total - sd_, sd_, k_)
        return D.duet_choose_split(spec, hw, batch, tau, k_max, opts)

    def prefill_arg(bufs=None, chunk=None):
        xp, yp = (x_pre, y_pre) if bufs is None else (bufs[0], bufs[2])
        if chunk is not None:   # the first `chunk` tokens of the (single) prompt: a smaller chunked-prefill step
            return dict(q=[chunk], c=[0], table=wl.pre_tables[:1], x=xp[:chunk], y=yp[:chunk])
        return dict(q=[q for q, _ in wl.pre_seqs], c=[c for _, c in wl.pre_seqs], table=wl.pre_tables, x=xp, y=yp)

    def decode_arg(k, bufs=None):
        xd, yd = (x_dec, y_dec) if bufs is None else (bufs[1], bufs[3])
        return dict(c=wl.dec_ctx, table=wl.dec_tables, x=xd, y=yd[:k], head=head)

    def one_step(split=None, bufs=None, chunk=None):
        """bufs: optional (x_pre, x_dec, y_pre, y_dec) device buffers (the e2e double buffering)."""
        s = decide() if split is None else split
        k = s.k if s.mode == D.DUET_MODE_SPATIAL else 1
        if k > 8:
            s = D.split_struct(s.mode, s.s_p, s.s_d, 8, s.flags, s.t_mixed, s.t_p, s.t_d, s.rho)
            k = 8
        ctx.step(W, prefill_arg(bufs, chunk), decode_arg(k, bufs), Kp, Vp, wl.n_pages, s)
        return s, k

    # every step runs on a dedicated non-blocking stream: the legacy default stream would serialise
    # with the e2e leg's copy streams
    torch.cuda.synchronize()
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    s0 = decide()
    log(f"split: mode={s0.mode} s_p={s0.s_p} s_d={s0.s_d} k={s0.k} flags={s0.flags} t_mixed={s0.t_mixed * 1e3:.2f} ms "
        f"t_p={s0.t_p * 1e3:.2f} ms t_d={s0.t_d * 1e3:.2f} ms")
    for i in range(args.warmup):
        h = time.perf_counter()
        one_step()
        h = time.perf_counter() - h
        torch.cuda.synchronize()
        log(f"warm-up step {i} done ({ctx.last_step_times()['t_window'] * 1e3:.2f} ms on the device, "
            f"{h * 1e3:.3f} ms host enqueue)")

    # ------------------------------------------------ kernel-class breakdown (untimed pass, every class)
    # Event records cost ~1 us each on the GPU; the headline timed region below times only the
    # dominant class (for the roofline), this short pass gives the per-class shares.
    KCLASS = {"gemm": 0, "prefill_attn": 1, "decode_attn": 2, "other": 3, "gemm_decode": 4, "other_decode": 5}
    n_break = min(args.steps, 10)
    ctx.profile_enable(True)
    for _ in range(n_break):
        one_step()
    torch.cuda.synchronize()
    kstats_all = ctx.profile_read()
    ctx.profile_enable(False)
    dom = max(kstats_all, key=lambda kname: kstats_all[kname]["seconds"])

    log("timed region")
    # ------------------------------------------------ timed region
    barrier(ws)
    torch.cuda.synchronize()
    clocks = ClockSampler(lrank)
    clocks.start()
    ctx.profile_enable(0 if os.environ.get("DUET_BENCH_NOPROF") else 1 << KCLASS[dom])
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    tokens = 0
    kernels = 0
    torch.cuda.profiler.start()     # ncu --profile-from-start off captures exactly the timed steps
    e0.record(stream)
    h0 = time.perf_counter()
    for _ in range(args.steps):
        s, k = one_step()
        tokens += k * n_d + n_p
    e1.record(stream)
    host_ms = (time.perf_counter() - h0) * 1e3 / args.steps
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
    barrier(ws)
    clk = clocks.stop()
    t_ms = e0.elapsed_time(e1)
    kstats = ctx.profile_read()
    ctx.profile_enable(False)
    times = ctx.last_step_times()
    kernels = times["kernels"] * args.steps
    value, t_max_s = whole_job_rate(tokens, t_ms * 1e-3, ws)
    if tp > 1:   # the TP group processes ONE batch per step: units are not multiplied by the ranks
        value /= ws
    ms_per_step = t_max_s * 1e3 / args.steps
    split = s

    # ------------------------------------------------ per-side times & predictor error (synced steps)
    def side_times(split, n=3, **kw):
        """Median of n synced steps of each duet_last_step_times field (t_window, t_decode, t_prefill)."""
        rows = []
        for _ in range(n):
            one_step(split, **kw)
            torch.cuda.synchronize()
            rows.append(ctx.last_step_times())
        return {key: float(np.median([r[key] for r in rows])) for key in ("t_window", "t_decode", "t_prefill")}

    def pred_errors(sp_, st_):
        """|t_pred - t_meas| / t_meas per side and for the window (Alg. 1's t_d, t_p)."""
        k_ = sp_.k if sp_.mode == D.DUET_MODE_SPATIAL else 1
        if sp_.mode == D.DUET_MODE_SPATIAL:
            w_pred = max(k_ * sp_.t_d, sp_.t_p)
            td_meas = st_["t_decode"] / k_
            return {"window": abs(w_pred - st_["t_window"]) / st_["t_window"],
                    "decode": abs(sp_.t_d - td_meas) / td_meas if td_meas > 0 else None,
                    "prefill": abs(sp_.t_p - st_["t_prefill"]) / st_["t_prefill"] if st_["t_prefill"] > 0 else None,
                    "t_pred_window_ms": w_pred * 1e3, "t_pred_d_ms": sp_.t_d * 1e3, "t_pred_p_ms": sp_.t_p * 1e3}
        return {"window": abs(sp_.t_mixed - st_["t_window"]) / st_["t_window"], "t_pred_window_ms": sp_.t_mixed * 1e3}

    side = side_times(split)
    pe = pred_errors(split, side)
    t_pred = pe["t_pred_window_ms"] * 1e-3
    pred_err = pe["window"]

    # algorithmic work of one window per side (SURVEY §8(d) per-unit figures)
    es_b = 2 if cfg.dtype == "bf16" else 4
    d_, hq_, hkv_, dh_, f_ = m.d_model, m.n_q_heads, m.n_kv_heads, m.head_dim, m.ffn_dim
    w_elems = nqkv * d_ + d_ * hq_ * dh_ + 2 * f_ * d_ + f_ * d_          # per layer

    def prefill_flops(seqs):
        g = 2.0 * sum(q for q, _ in seqs) * w_elems
        a = sum(4.0 * hq_ * dh_ * (q * c + q * (q + 1) / 2) for q, c in seqs)
        return m.n_layers * (g + a)

    def decode_step_bytes(ctxs):
        n = len(ctxs)
        act = n * (d_ + nqkv + hq_ * dh_ + d_ + d_ + 2 * f_ + f_ + d_ + d_)   # GEMM inputs + outputs
        kv = sum(2 * hkv_ * dh_ * (c + 1) for c in ctxs)
        return m.n_layers * (w_elems + act + kv) * es_b

    F_pre = prefill_flops(wl.pre_seqs)
    B_dec = decode_step_bytes(wl.dec_ctx)
    pk, pk_src = peaks()

    def partition_roofline(sp_, st_):
        """Per-partition roofline (BASELINE north_star; SURVEY §8(d) 'which roofline bounds each side')."""
        if sp_.mode != D.DUET_MODE_SPATIAL:
            return None
        k_ = sp_.k
        ach_t = F_pre / st_["t_prefill"] / 1e12
        peak_p = float(pk["bf16_tflops_sustained"]) * sp_.s_p / total
        ach_b = k_ * B_dec / st_["t_decode"] / 1e9
        out = {"prefill": {"s_p": sp_.s_p, "achieved_tflops": ach_t, "peak_tflops": peak_p, "frac": ach_t / peak_p,
                           "peak_note": "sustained bf16 peak x S_p/148 (MEASURED_PEAKS.json)"},
               "decode": {"s_d": sp_.s_d, "achieved_gbs": ach_b, "frac_of_hbm_peak": ach_b / float(pk["hbm_gbs"]),
                          "hbm_peak_gbs": float(pk["hbm_gbs"])}}
        if stream_bw is not None and stream_bw[sp_.s_d] > 0:
            out["decode"]["stream_ceiling_gbs"] = stream_bw[sp_.s_d] / 1e9
            out["decode"]["frac_of_stream_ceiling"] = ach_b * 1e9 / stream_bw[sp_.s_d]
            # per-operator roofline at S_d with the stream ceiling as B(S): sum_op max(F/Pi(S_d), B/B_stream(S_d))
            hw_s = D.HwProfile(total, parts, fl, [b if b > 0 else bw[i] for i, b in enumerate(stream_bw)],
                               nvlink_bw=nvl_bw, allreduce_alpha=ar_alpha)
            t_op = D.duet_predict_latency(spec, hw_s, [e for e in batch if e[2] == 2], sp_.s_d,
                                          opts & D.DUET_OPT_INCLUDE_CLS)["t_total"]
            out["decode"]["per_operator_roofline_ms"] = t_op * 1e3
            out["decode"]["frac_of_per_operator_roofline"] = t_op / (st_["t_decode"] / k_)
        return out

    log(f"timed: {ms_per_step:.3f} ms/step; comparisons")
    # ------------------------------------------------ aggregated vs partitioned (same kernels, same batch)
    def tbt_stats(ts, k_):
        """Inter-token gaps (ms) from the device token-time ring: every gap, and the window-boundary ones."""
        g = np.diff(np.asarray(ts, dtype=np.float64)) * 1e-6
        if g.size == 0:
            return {}
        bnd = g[[j for j in range(g.size) if (j + 1) % k_ == 0]]
        return {"tbt_max_ms": float(g.max()), "tbt_median_ms": float(np.median(g)), "tbt_p90_ms": float(np.percentile(g, 90)),
                "boundary_gap_max_ms": float(bnd.max()) if bnd.size else None,
                "boundary_gap_median_ms": float(np.median(bnd)) if bnd.size else None, "gaps": int(g.size)}

    def timed(split_fn, n=max(5, min(args.steps, 20)), chunk=None):
        """tokens/s over n back-to-back windows (CUDA events), TBT from the token-time ring of the same
        windows, per-side times of synced steps."""
        for _ in range(2):
            one_step(split_fn(), chunk=chunk)
        torch.cuda.synchronize()
        ctx.token_times_reset()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        tok = 0
        n_p_ = chunk if chunk is not None else n_p
        clk_ = ClockSampler(lrank)   # each leg's own clocks: a power-capped leg is compared at its clock
        clk_.start()
        a.record(stream)
        h_ = time.perf_counter()
        for _ in range(n):
            s_, k_ = one_step(split_fn(), chunk=chunk)
            tok += k_ * n_d + n_p_
        h_ = (time.perf_counter() - h_) / n
        b.record(stream)
        torch.cuda.synchronize()
        pg_ = ctx.last_step_times()["prefill_graph"]
        c_ = clk_.stop()
        ts = ctx.token_times(reset=True)
        sp_ = split_fn()
        st_ = side_times(sp_, chunk=chunk)
        k_ = sp_.k if sp_.mode == D.DUET_MODE_SPATIAL else 1
        r = {"tok_s": tok / (a.elapsed_time(b) * 1e-3), "window_ms": st_["t_window"] * 1e3,
             "t_decode_ms": st_["t_decode"] * 1e3, "t_prefill_ms": st_["t_prefill"] * 1e3, "k": k_,
             "sm_mhz": c_.get("sm_mhz"), "clock_reasons": c_.get("reasons"),
             "host_enqueue_ms": h_ * 1e3, "prefill_graph": bool(pg_)}
        r.update(tbt_stats(ts, k_))
        return r, st_

    comp, part_roof = {}, None
    if not args.profile_only:
        temporal = lambda: D.split_struct(D.DUET_MODE_TEMPORAL, total, 0, 1)
        agg, _ = timed(temporal)
        agg["t_pred_ms"] = split.t_mixed * 1e3
        # aggregated at the SLO: conventional chunked prefill with the chunk cut to the largest
        # multiple of 256 tokens for which the predicted mixed iteration meets tau — what a temporal-only
        # server must do to hold the TBT SLO
        q_slo = 0
        for q_ in range(n_p // 256 * 256, 0, -256):
            b_ = [(q_, 0, 0, 0)] + [e for e in batch if e[2] == 2]
            if D.duet_predict_latency(spec, hw, b_, total, opts & D.DUET_OPT_INCLUDE_CLS)["t_total"] <= tau:
                q_slo = q_
                break
        agg_slo = None
        if 0 < q_slo < n_p:
            agg_slo, _ = timed(temporal, chunk=q_slo)
            agg_slo["prefill_chunk"] = q_slo
        forced = D.duet_choose_split(spec, hw, batch, tau, k_max, D.DUET_OPT_FORCE_SPATIAL | (opts & D.DUET_OPT_INCLUDE_CLS))
        if forced.k > 8:
            forced = D.split_struct(1, forced.s_p, forced.s_d, 8, forced.flags, forced.t_mixed, forced.t_p,
                                    forced.t_d, forced.rho)
        spa, spa_side = timed(lambda: forced)
        spa.update({"s_d": forced.s_d, "s_p": forced.s_p, "k": forced.k, "flags": forced.flags})
        spa["predictor_error"] = pred_errors(forced, spa_side)
        part_roof = partition_roofline(forced, spa_side)
        # the boundary-aware optimizer (reading #23, opt-in): the window-boundary gap also within tau
        fb = D.duet_choose_split(spec, hw, batch, tau, 8, D.DUET_OPT_FORCE_SPATIAL | D.DUET_OPT_BOUNDARY_TBT |
                                 (opts & D.DUET_OPT_INCLUDE_CLS))
        spb = None
        if fb.mode == D.DUET_MODE_SPATIAL and not (fb.flags & D.DUET_FLAG_INFEASIBLE):
            spb, spb_side = timed(lambda: fb)
            spb.update({"s_d": fb.s_d, "s_p": fb.s_p, "k": fb.k, "flags": fb.flags,
                        "t_pred_boundary_gap_ms": (fb.t_d + max(0.0, fb.t_p - fb.k * fb.t_d)) * 1e3})
            spb["predictor_error"] = pred_errors(fb, spb_side)
        comp = {"aggregated": agg, "aggregated_chunked_at_slo": agg_slo, "partitioned_optimizer": spa,
                "partitioned_boundary_aware": spb, "tau_ms": tau * 1e3,
                "north_star": {"partitioned_tbt_max_ms": spa.get("tbt_max_ms"),
                               "partitioned_step_tbt_ms": spa["t_decode_ms"] / spa["k"],
                               # the paper's constraint is the decode step t_d <= tau; the
                               # window-boundary gap is reported beside it (reading #23)
                               "partitioned_meets_slo_paper": spa["t_decode_ms"] / spa["k"] <= tau * 1e3,
                               "partitioned_meets_slo": (spa.get("tbt_max_ms") or 1e9) <= tau * 1e3,
                               "boundary_aware_tbt_max_ms": spb.get("tbt_max_ms") if spb else None,
                               "boundary_aware_over_aggregated_at_slo":
                                   spb["tok_s"] / agg_slo["tok_s"] if (spb and agg_slo) else None,
                               "partitioned_over_aggregated": spa["tok_s"] / agg["tok_s"],
                               "partitioned_over_aggregated_at_slo":
                                   spa["tok_s"] / agg_slo["tok_s"] if agg_slo else None}}
        if args.sweep:
            rows = []
            P_b = [e for e in batch if e[2] != 2]
            D_b = [e for e in batch if e[2] == 2]
            for sd in parts:
                td = D.duet_predict_latency(spec, hw, D_b, sd, opts & D.DUET_OPT_INCLUDE_CLS)["t_total"]
                tpp = D.duet_predict_latency(spec, hw, P_b, total - sd, opts & D.DUET_OPT_INCLUDE_CLS)["t_total"]
                r_ = int(np.floor(tpp / td))
                ks = [min(max(x, 1), 8) for x in (r_, r_ + 1)]
                rhos = [(kk * len(D_b) + sum(e[0] for e in P_b)) / max(kk * td, tpp) for kk in ks]
                kk = ks[int(np.argmax(rhos))]
                sp_ = D.split_struct(1, total - sd, sd, kk, 0, split.t_mixed, tpp, td, max(rhos))
                r, st_ = timed(lambda: sp_, n=4)
                r.update({"s_d": sd, "s_p": total - sd, "t_pred_d_ms": td * 1e3, "t_pred_p_ms": tpp * 1e3,
                          "t_pred_window_ms": max(kk * td, tpp) * 1e3, "predicted_tok_s": max(rhos),
                          "optimizer_pick": sd == forced.s_d, "meets_slo_pred": td <= tau,
                          "meets_slo_meas": (r.get("tbt_max_ms") or 1e9) <= tau * 1e3})
                rows.append(r)
                log(f"sweep S_d={sd}: k={kk} {r['tok_s']:.0f} tok/s window {r['window_ms']:.2f} ms "
                    f"(pred {max(kk * td, tpp) * 1e3:.2f}) TBT max {r.get('tbt_max_ms', 0):.2f} ms")
            comp["sweep"] = rows

    log("e2e")
    # ------------------------------------------------ e2e through the C ABI with host buffers
    e2e = None
    if not args.profile_only:
        hx_pre = torch.empty(x_pre.shape, dtype=tdt, pin_memory=True)
        hx_dec = torch.empty(x_dec.shape, dtype=tdt, pin_memory=True)
        hx_pre.copy_(x_pre)
        hx_dec.copy_(x_dec)
        hy_pre = torch.empty(y_pre.shape, dtype=tdt, pin_memory=True)
        hy_dec = torch.empty(y_dec.shape, dtype=tdt, pin_memory=True)
        # The step's result a server reads back is the rows it samples from: every decode row's output and
        # the last row of each prefill sequence (the other prompt rows' hidden states never leave the
        # GPU in serving).  all_rows=True reads back every output row instead (reported alongside).
        last_rows = [int(r) for r in np.cumsum([q for q, _ in wl.pre_seqs]) - 1]
        hy_last = torch.empty((max(len(last_rows), 1), m.d_model), dtype=tdt, pin_memory=True)

        def e2e_leg(all_rows):
            n_e2e = max(5, args.steps // 2)
            NSET = int(os.environ.get("DUET_E2E_SETS", "2"))   # device buffer sets in flight
            # The caller's view: every step's inputs come from pinned host memory and its outputs go back to
            # it.  Two device buffer sets and a copy stream overlap step i's compute with the H2D of step
            # i+1 and the D2H of step i-1 (PCIe is full duplex); every copy is inside the timed region.
            bufs = [(x_pre, x_dec, y_pre, y_dec)] + [
                (torch.empty_like(x_pre), torch.empty_like(x_dec), torch.empty_like(y_pre), torch.empty_like(y_dec))
                for _ in range(NSET - 1)]
            cs = torch.cuda.Stream()    # H2D
            cs2 = torch.cuda.Stream()   # D2H (the other PCIe direction, concurrently)
            ev_in = [torch.cuda.Event() for _ in range(NSET)]
            ev_out = [torch.cuda.Event() for _ in range(NSET)]
            ev_d2h = [torch.cuda.Event() for _ in range(NSET)]
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            tok = 0
            h2d = d2h = 0
            # diagnosis only (never set for a reported run): DUET_E2E_SKIP=h2d / d2h drops one direction
            skip = os.environ.get("DUET_E2E_SKIP", "")
            tl = ([[torch.cuda.Event(enable_timing=True) for _ in range(5)] for _ in range(n_e2e)]
                  if os.environ.get("DUET_E2E_TIMELINE") else None)
            hts = []
            torch.cuda.synchronize()
            a.record(cs)
            h1 = time.perf_counter()
            def d2h_of(j, kj):
                """D2H of step j's outputs, issued one iteration late (after step j+1's work): a copy
                queued ahead of the next step could hold that step's launches behind it."""
                sj = j % NSET
                yp_, yd_ = bufs[sj][2], bufs[sj][3]
                with torch.cuda.stream(cs2):
                    cs2.wait_event(ev_out[sj])
                    if "d2h" not in skip:
                        if all_rows:
                            hy_pre.copy_(yp_, non_blocking=True)
                        else:
                            for j_, r_ in enumerate(last_rows):
                                hy_last[j_].copy_(yp_[r_], non_blocking=True)
                        hy_dec[:kj].copy_(yd_[:kj], non_blocking=True)
                    ev_d2h[sj].record(cs2)
                    if tl is not None:
                        tl[j][4].record(cs2)

            k_prev = None
            for i in range(n_e2e):
                st_ = i % NSET
                xp, xd, yp, yd = bufs[st_]
                if tl is not None:
                    hts.append([time.perf_counter()])
                with torch.cuda.stream(cs):
                    if i >= NSET:
                        cs.wait_event(ev_out[st_])      # step i-NSET has finished reading x of this set
                    if tl is not None:
                        tl[i][0].record(cs)
                    if "h2d" not in skip:
                        xp.copy_(hx_pre, non_blocking=True)
                        xd.copy_(hx_dec, non_blocking=True)
                    ev_in[st_].record(cs)
                    if tl is not None:
                        tl[i][1].record(cs)
                stream.wait_event(ev_in[st_])
                if i >= NSET:
                    stream.wait_event(ev_d2h[st_])      # step i-NSET's outputs of this set are on the host
                if tl is not None:
                    tl[i][2].record(stream)
                    hts[-1].append(time.perf_counter())
                s_, k_ = one_step(bufs=bufs[st_])
                if tl is not None:
                    hts[-1].append(time.perf_counter())
                ev_out[st_].record(stream)
                if tl is not None:
                    tl[i][3].record(stream)
                if k_prev is not None:
                    d2h_of(i - 1, k_prev)
                k_prev = k_
                tok += k_ * n_d + n_p
                h2d = hx_pre.numel() * hx_pre.element_size() + hx_dec.numel() * hx_dec.element_size()
                d2h = ((hy_pre.numel() if all_rows else len(last_rows) * m.d_model) * hy_pre.element_size()
                       + k_ * n_d * m.d_model * hy_dec.element_size())
            d2h_of(n_e2e - 1, k_prev)
            cs.wait_stream(cs2)
            b.record(cs)
            host_e2e_ms = (time.perf_counter() - h1) * 1e3 / n_e2e
            torch.cuda.synchronize()
            log(f"host enqueue ms/step: timed loop {host_ms:.3f}, e2e loop {host_e2e_ms:.3f}")
            if tl is not None:   # per-step timeline (ms from the loop start): h2d start/end, step start/end, d2h end
                for i in range(min(n_e2e, 12)):
                    log(f"e2e step {i}: " + " ".join(f"{a.elapsed_time(ev):8.3f}" for ev in tl[i]) + " | host " +
                        " ".join(f"{(t - h1) * 1e3:8.3f}" for t in hts[i]))
            te = max_over_ranks(a.elapsed_time(b), ws)
            return {"value": tok * (1 if tp > 1 else ws) / (te * 1e-3), "unit": "tokens/s",
                    "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h)}

        def e2e_safe(all_rows):
            # --sweep leaves a decode graph per split resident: on cfg3 the e2e leg's extra buffers may not
            # fit after it; report that instead of losing the line
            try:
                return e2e_leg(all_rows)
            except torch.OutOfMemoryError as ex:
                torch.cuda.empty_cache()
                log(f"e2e ({'all rows' if all_rows else 'sampled rows'}) skipped: out of memory")
                return {"value": None, "unit": "tokens/s", "error": f"out of memory: {str(ex)[:120]}"}

        e2e = e2e_safe(False)
        e2e["all_rows"] = e2e_safe(True)

    # ------------------------------------------------ roofline of the dominant kernel class
    pk, pk_src = peaks()
    st_ = kstats[dom]
    tensor_bound = dom in ("gemm", "prefill_attn", "gemm_decode")
    # the SMs the dominant class ran on: a spatial step's decode side (decode attention, *_decode) on S_d,
    # its prefill side on S_p, a temporal step on the whole device
    if split.mode == D.DUET_MODE_SPATIAL:
        dom_sms = split.s_d if dom in ("decode_attn", "gemm_decode", "other_decode") else split.s_p
    else:
        dom_sms = total
    traffic = None
    tpath = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tpath):
        traffic = json.load(open(tpath)).get(f"{args.config}:{dom}")
    if st_["launches"] and st_["seconds"] > 0:
        if tensor_bound:
            ach = st_["flops"] / st_["seconds"] / 1e12
            # the burst figure for a short timed region, the sustained one for a region of seconds
            # (the GPU settles at its power cap, B200_PROFILING.md)
            sustained = t_ms > 1000.0
            peak = float(pk["bf16_tflops_sustained" if sustained else "bf16_tflops"])
            roof = {"bound": "tensor", "achieved": ach, "peak": peak, "unit": "TFLOP/s", "frac": ach / peak,
                    "traffic": traffic, "kernel": dom, "launches": st_["launches"],
                    "avg_launch_us": st_["seconds"] / st_["launches"] * 1e6,
                    "peak_source": pk_src + (" sustained bf16 (timed region %.1f s)" % (t_ms / 1e3) if sustained
                                             else " burst bf16")}
            roof["partition"] = {"sms": dom_sms, "peak": peak * dom_sms / total, "frac": ach / (peak * dom_sms / total),
                                 "note": "the measured peak scaled to the SMs the kernel ran on"}
        else:
            ach = st_["bytes"] / st_["seconds"] / 1e9
            peak = float(pk["hbm_gbs"])
            roof = {"bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s", "frac": ach / peak,
                    "traffic": traffic, "kernel": dom, "launches": st_["launches"],
                    "avg_launch_us": st_["seconds"] / st_["launches"] * 1e6, "peak_source": pk_src}
            if dom_sms < total and stream_bw is not None and stream_bw[dom_sms] > 0:
                roof["partition"] = {"sms": dom_sms, "peak": stream_bw[dom_sms] / 1e9,
                                     "frac": ach * 1e9 / stream_bw[dom_sms],
                                     "note": "LDG stream ceiling on the kernel's S_d-SM partition (duet_calibrate_stream)"}
    else:
        roof = {"bound": "tensor", "achieved": None, "peak": None, "unit": "TFLOP/s", "frac": None, "traffic": None,
                "kernel": dom}
    share = {kname: v["seconds"] / n_break for kname, v in kstats_all.items()}

    log("cpu baseline")
    # ------------------------------------------------ CPU baseline (oracle), rank 0, N=1 only
    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu_baseline and not args.profile_only:
        v_c, desc_c = oracle_baseline(args.config)
        cpu = {"value": v_c, "unit": "tokens/s", "cores": oracle_cores(), "kind": "oracle", "sample": desc_c,
               "host": host_cores()}
        # Alg. 1 on the host ("< 1 ms"): the library's C++ and the oracle's Python on this batch
        import oracle.roofline as R
        t0_ = time.perf_counter()
        for _ in range(20):
            D.duet_choose_split(spec, hw, batch, tau, k_max, opts)
        cpu["optimizer_ms"] = (time.perf_counter() - t0_) / 20 * 1e3
        prof_o = R.Profile(total, tuple(parts), tuple(fl), tuple(bw), nvl_bw, ar_alpha)
        spec_o = R.Spec(m.n_layers, m.d_model, m.ffn_dim, m.n_q_heads, m.n_kv_heads, m.head_dim, m.vocab,
                        2 if cfg.dtype == "bf16" else 4, True, tp)
        reqs_o = [R.Req(e[0], e[1], e[2], e[3]) for e in batch]
        t0_ = time.perf_counter()
        R.choose_split(spec_o, prof_o, reqs_o, tau, k_max, opts)
        cpu["oracle_optimizer_ms"] = (time.perf_counter() - t0_) * 1e3

    if rank == 0:
        # the partition sizes a split can use (each decode size and its complement) and the full device
        cal_sizes = sorted({S for p in parts for S in (p, total - p)} | {total})
        line = {
            "metric": METRIC, "value": value, "unit": "tokens/s", "n_gpus": ws, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True, "scaling": "strong" if tp > 1 else "weak",
            "vs_baseline": None, "dtype": cfg.dtype, "data": "synthetic (seeded counter generator, random weights)",
            "config": {"workload": f"{args.config}: {cfg.note}" + (" + LM head / greedy tokens (f1)" if head is not None
                                                                      else ""),
                       "mode": ["temporal", "spatial"][split.mode],
                       "s_p": split.s_p, "s_d": split.s_d, "k": split.k, "flags": split.flags,
                       "attention_corun_s_d": times["corun_s_d"],
                       "tau_ms": tau * 1e3, "prefill_tokens": n_p, "decode_reqs": n_d,
                       "l2": f"inputs > L2 ({step_bytes / 1e9:.1f} GB of weights + KV read per step), no flush",
                       "parallelism": f"tp{tp} (head-sharded, NCCL allreduce after O and down)" if tp > 1
                       else f"dp{ws} (independent replicas)", "calibration_s": round(t_cal, 2),
                       "calibration": args.calibration, "partition_granularity_sms": 2 if args.fine_split else 8},
            "predictor": {"t_pred_ms": t_pred * 1e3, "t_meas_ms": side["t_window"] * 1e3, "err": pred_err,
                          "t_meas_decode_ms": side["t_decode"] * 1e3, "t_meas_prefill_ms": side["t_prefill"] * 1e3,
                          "per_side": pe,
                          "partitioned_optimizer_split": comp.get("partitioned_optimizer", {}).get("predictor_error")},
            "comparison": comp,
            "partition_roofline": part_roof,
            "roofline": roof,
            "kernel_seconds_per_step": share,
            "kernel_timing": (f"the {dom} launches inside the timed region (roofline): "
                              + ("device-side %globaltimer span of every decode-attention launch inside the decode "
                                 "CUDA graphs (duet_profile: no events in graphs)"
                                 if dom == "decode_attn" and split.mode == D.DUET_MODE_SPATIAL else
                                 "CUDA events on the launching stream")
                              + f"; per-class seconds per step from an untimed {n_break}-step pass"),
            "gpu_launches": int(kernels),
            "clocks": clk,
            "e2e": e2e,
            "cpu_baseline": cpu,
            # the calibrated Pi_SM(S) / B_HBM(S) tables Alg. 1 ran on (every calibrated partition size;
            # SURVEY §8(d) calibration inputs)
            "profile_tables": {"sms": cal_sizes,
                               "tflops": [round(fl[S] / 1e12, 3) for S in cal_sizes],
                               "hbm_gbs": [round(bw[S] / 1e9, 2) for S in cal_sizes],
                               "source": f"duet_calibrate{'_corun' if args.calibration == 'corun' else ''} on this box"},
        }
        print(json.dumps(line), flush=True)
    ctx.close()
    if ws > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

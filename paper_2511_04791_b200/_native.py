"""ctypes marshalling for libduet.so — same names as include/duet.h, no computation here."""
from __future__ import annotations

import ctypes as C
import os

import torch  # noqa: F401  (loads libcudart before libduet.so so both share one CUDA runtime)

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libduet.so")

DUET_OK = 0
DUET_PHASE_PREFILL_FULL, DUET_PHASE_PREFILL_CHUNK, DUET_PHASE_DECODE = 0, 1, 2
DUET_OPT_FORCE_SPATIAL, DUET_OPT_INCLUDE_CLS, DUET_OPT_VERBATIM_INFEASIBLE, DUET_OPT_BOUNDARY_TBT = 1, 2, 4, 8
DUET_MODE_TEMPORAL, DUET_MODE_SPATIAL = 0, 1
DUET_FLAG_INFEASIBLE, DUET_FLAG_DEGENERATE = 1, 2
DUET_DTYPE_BF16, DUET_DTYPE_FP32 = 0, 1
DUET_CTX_FINE_SPLIT, DUET_CTX_NO_GRAPH, DUET_CTX_NO_CORUN, DUET_CTX_NO_PREFILL_GRAPH = 1, 2, 4, 8
DUET_EPI_STORE, DUET_EPI_RESIDUAL, DUET_EPI_SWIGLU = 0, 1, 2
STATUS_NAMES = {0: "OK", -1: "INVALID_ARG", -2: "OUT_OF_RANGE", -3: "CONFIG", -4: "UNSUPPORTED", -5: "CUDA",
                -6: "CAPACITY", -7: "NCCL"}


class DuetError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"duet status {status} ({STATUS_NAMES.get(status, '?')}): {msg}")
        self.status = status


class duet_model_spec(C.Structure):
    _fields_ = [(n, C.c_int32) for n in ("n_layers", "d_model", "ffn_dim", "n_q_heads", "n_kv_heads", "head_dim",
                                         "vocab", "elem_bytes", "ffn_gated", "qkv_bias", "tp")] + \
               [("rope_theta", C.c_double), ("norm_eps", C.c_double)]


class duet_hw_profile(C.Structure):
    _fields_ = [("total_sms", C.c_int32), ("n_cand", C.c_int32), ("cand_sd_sms", C.POINTER(C.c_int32)),
                ("flops_at_sms", C.POINTER(C.c_double)), ("bw_at_sms", C.POINTER(C.c_double)),
                ("nvlink_bw", C.c_double), ("allreduce_alpha", C.c_double)]


class duet_req(C.Structure):
    _fields_ = [("q", C.c_int32), ("c", C.c_int32), ("phase", C.c_int32), ("emits_logits", C.c_int32)]


class duet_latency(C.Structure):
    _fields_ = [(n, C.c_double) for n in ("t_linear", "t_norm_act", "t_attn", "t_allreduce", "t_block", "t_cls",
                                          "t_total")]


class duet_split(C.Structure):
    _fields_ = [(n, C.c_int32) for n in ("mode", "s_p", "s_d", "k", "flags")] + \
               [(n, C.c_double) for n in ("t_mixed", "t_p", "t_d", "rho")]


class duet_ctx_limits(C.Structure):
    _fields_ = [(n, C.c_int32) for n in ("max_prefill_tokens", "max_prefill_seqs", "max_decode_reqs", "max_k",
                                         "max_pages_per_seq", "max_pos", "dtype")] + [("flags", C.c_uint32)]


class duet_layer_weights(C.Structure):
    _fields_ = [(n, C.c_void_p) for n in ("w_qkv", "b_qkv", "w_o", "w_gate_up", "w_down", "g_norm1", "g_norm2")]


class duet_prefill(C.Structure):
    _fields_ = [("n_seqs", C.c_int32), ("q", C.POINTER(C.c_int32)), ("c", C.POINTER(C.c_int32)),
                ("page_table", C.POINTER(C.c_int32)), ("max_pages", C.c_int32), ("x", C.c_void_p), ("y", C.c_void_p)]


class duet_lm_head(C.Structure):
    _fields_ = [("g_norm", C.c_void_p), ("w_head", C.c_void_p), ("embed", C.c_void_p), ("tokens", C.c_void_p)]


class duet_decode(C.Structure):
    _fields_ = [("n_reqs", C.c_int32), ("c", C.POINTER(C.c_int32)), ("page_table", C.POINTER(C.c_int32)),
                ("max_pages", C.c_int32), ("x", C.c_void_p), ("y", C.c_void_p), ("head", C.POINTER(duet_lm_head))]


class duet_kv_pages(C.Structure):
    _fields_ = [("k_pool", C.POINTER(C.c_void_p)), ("v_pool", C.POINTER(C.c_void_p)), ("n_pages", C.c_int32),
                ("page_size", C.c_int32)]


(DUET_KCLASS_GEMM, DUET_KCLASS_PREFILL_ATTN, DUET_KCLASS_DECODE_ATTN, DUET_KCLASS_OTHER, DUET_KCLASS_GEMM_DECODE,
 DUET_KCLASS_OTHER_DECODE, DUET_KCLASS_N) = range(7)
DUET_PROFILE_ALL = 0x3F


class duet_corun_profile(C.Structure):
    _fields_ = [("total_sms", C.c_int32), ("n_cand", C.c_int32), ("cand_sd_sms", C.POINTER(C.c_int32)),
                ("fa_flops_at_sms", C.POINTER(C.c_double)), ("dec_bw_at_sms", C.POINTER(C.c_double)),
                ("min_sms", C.c_int32), ("overhead_s", C.c_double)]


class duet_kernel_stats(C.Structure):
    _fields_ = [("launches", C.c_int32), ("seconds", C.c_double), ("flops", C.c_double), ("bytes", C.c_double)]


class duet_step_times(C.Structure):
    _fields_ = [("t_window", C.c_double), ("t_decode", C.c_double), ("t_prefill", C.c_double),
                ("mode", C.c_int32), ("k", C.c_int32), ("kernels", C.c_int32),
                ("corun_s_d", C.c_int32), ("prefill_graph", C.c_int32)]


_lib = None

_SIGS = {
    "duet_last_error": (C.c_char_p, []),
    "duet_abi_version": (C.c_int32, []),
    "duet_predict_latency": (C.c_int, [C.POINTER(duet_model_spec), C.POINTER(duet_hw_profile), C.POINTER(duet_req),
                                       C.c_int32, C.c_int32, C.c_uint32, C.POINTER(duet_latency)]),
    "duet_choose_split": (C.c_int, [C.POINTER(duet_model_spec), C.POINTER(duet_hw_profile), C.POINTER(duet_req),
                                    C.c_int32, C.c_double, C.c_int32, C.c_uint32, C.POINTER(duet_split)]),
    "duet_ctx_create": (C.c_int, [C.c_int32, C.POINTER(duet_model_spec), C.POINTER(duet_ctx_limits),
                                  C.POINTER(C.c_void_p)]),
    "duet_ctx_destroy": (C.c_int, [C.c_void_p]),
    "duet_ctx_partitions": (C.c_int, [C.c_void_p, C.POINTER(C.c_int32), C.POINTER(C.c_int32),
                                      C.POINTER(C.c_int32)]),
    "duet_step": (C.c_int, [C.c_void_p, C.POINTER(duet_layer_weights), C.POINTER(duet_prefill),
                            C.POINTER(duet_decode), C.POINTER(duet_kv_pages), C.POINTER(duet_split), C.c_void_p]),
    "duet_last_step_times": (C.c_int, [C.c_void_p, C.POINTER(duet_step_times)]),
    "duet_calibrate": (C.c_int, [C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_int32]),
    "duet_profile_enable": (C.c_int, [C.c_void_p, C.c_int32]),
    "duet_profile_read": (C.c_int, [C.c_void_p, C.c_void_p]),
    "duet_op_gemm": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32,
                               C.c_int32, C.c_int32, C.c_int32, C.c_void_p]),
    "duet_op_rmsnorm": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p]),
    "duet_sched_create": (C.c_int, [C.c_void_p, C.POINTER(C.c_void_p)]),
    "duet_sched_destroy": (C.c_int, [C.c_void_p]),
    "duet_sched_add": (C.c_int, [C.c_void_p, C.c_int64, C.c_int32, C.c_int32, C.c_double]),
    "duet_sched_next": (C.c_int, [C.c_void_p, C.c_double, C.c_void_p]),
    "duet_sched_commit": (C.c_int, [C.c_void_p, C.c_int32, C.POINTER(C.c_int32), C.POINTER(C.c_int32)]),
    "duet_sched_free_pages": (C.c_int, [C.c_void_p, C.POINTER(C.c_int32)]),
    "duet_nccl_unique_id": (C.c_int, [C.c_void_p, C.c_int32]),
    "duet_ctx_set_comms": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p]),
    "duet_calibrate_allreduce": (C.c_int, [C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_double)]),
    "duet_ctx_check_comms": (C.c_int, [C.c_void_p]),
    "duet_ctx_last_pod": (C.c_int32, [C.c_void_p]),
    "duet_ctx_ar_handle": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32]),
    "duet_ctx_ar_open": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p]),
    "duet_op_gemm_ar_emul": (C.c_int, [C.c_void_p, C.c_int32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_void_p,
                                       C.c_int32, C.c_int32, C.c_int32, C.c_void_p]),
    "duet_op_decode_attn": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p, C.c_int32,
                                      C.POINTER(C.c_int32), C.POINTER(C.c_int32), C.c_int32, C.c_void_p, C.c_void_p,
                                      C.c_int32, C.c_int32, C.c_void_p]),
    "duet_op_prefill_attn": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int32, C.c_void_p, C.c_int32,
                                       C.POINTER(C.c_int32), C.POINTER(C.c_int32), C.POINTER(C.c_int32), C.c_int32,
                                       C.c_void_p, C.c_void_p, C.c_int32, C.c_int32, C.c_void_p]),
    "duet_profile_smooth": (C.c_int, [C.POINTER(C.c_int32), C.c_int32, C.POINTER(C.c_double), C.c_int32]),
    "duet_corun_choose": (C.c_int, [C.POINTER(duet_corun_profile), C.c_double, C.c_double, C.POINTER(C.c_int32),
                                    C.POINTER(C.c_double)]),
    "duet_calibrate_corun": (C.c_int, [C.c_void_p, C.POINTER(C.c_double), C.POINTER(C.c_double), C.c_int32,
                                       C.c_double]),
    "duet_calibrate_stream": (C.c_int, [C.c_void_p, C.POINTER(C.c_double), C.c_int32]),
    "duet_token_times": (C.c_int, [C.c_void_p, C.c_int32, C.POINTER(C.c_uint64), C.c_int32,
                                   C.POINTER(C.c_int32)]),
}

EXPORTED = tuple(_SIGS)


def lib():
    """Load libduet.so (built in-tree by ``__graft_entry__.build()``); raises if absent."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} is missing: run `python -m paper_2511_04791_b200.build` "
                              "(there is no CPU fallback)")
        h = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            f = getattr(h, name)
            f.restype = res
            f.argtypes = args
        _lib = h
    return _lib


def _check(status: int):
    if status != DUET_OK:
        raise DuetError(status, lib().duet_last_error().decode())


# ------------------------------------------------------------------ struct builders

def make_spec(n_layers, d_model, ffn_dim, n_q_heads, n_kv_heads, head_dim, vocab=128256, elem_bytes=2,
              ffn_gated=1, qkv_bias=0, tp=1, rope_theta=1e4, norm_eps=1e-5) -> duet_model_spec:
    return duet_model_spec(n_layers, d_model, ffn_dim, n_q_heads, n_kv_heads, head_dim, vocab, elem_bytes,
                           int(ffn_gated), int(qkv_bias), tp, float(rope_theta), float(norm_eps))


class HwProfile:
    """Owns the arrays a duet_hw_profile points to."""

    def __init__(self, total_sms, cand_sd_sms, flops_at_sms, bw_at_sms, nvlink_bw=900e9, allreduce_alpha=3e-6):
        self.total_sms = int(total_sms)
        self.cand = (C.c_int32 * max(1, len(cand_sd_sms)))(*[int(s) for s in cand_sd_sms])
        self.n_cand = len(cand_sd_sms)
        self.flops = (C.c_double * len(flops_at_sms))(*[float(v) for v in flops_at_sms])
        self.bw = (C.c_double * len(bw_at_sms))(*[float(v) for v in bw_at_sms])
        self.struct = duet_hw_profile(self.total_sms, self.n_cand, self.cand, self.flops, self.bw,
                                      float(nvlink_bw), float(allreduce_alpha))


def _reqs(batch):
    arr = (duet_req * max(1, len(batch)))()
    for i, r in enumerate(batch):
        arr[i] = duet_req(int(r[0]), int(r[1]), int(r[2]), int(r[3]) if len(r) > 3 else 0)
    return arr


# ------------------------------------------------------------------ host entry points

def duet_predict_latency(spec: duet_model_spec, hw: HwProfile, batch, sms: int, opts: int = 0) -> dict:
    """batch: sequence of (q, c, phase[, emits_logits])."""
    out = duet_latency()
    _check(lib().duet_predict_latency(C.byref(spec), C.byref(hw.struct), _reqs(batch), len(batch), int(sms),
                                      int(opts), C.byref(out)))
    return {n: getattr(out, n) for n, _ in duet_latency._fields_}


def duet_choose_split(spec: duet_model_spec, hw: HwProfile, batch, tbt_slo_s: float, k_max: int = 32,
                      opts: int = 0) -> duet_split:
    out = duet_split()
    _check(lib().duet_choose_split(C.byref(spec), C.byref(hw.struct), _reqs(batch), len(batch), float(tbt_slo_s),
                                   int(k_max), int(opts), C.byref(out)))
    return out


def duet_profile_smooth(sizes, table):
    """Median-of-three smoothing of per-SM rates over the measured sizes (duet_profile_smooth); returns
    a new list."""
    s = (C.c_int32 * max(1, len(sizes)))(*sizes)
    t = (C.c_double * len(table))(*table)
    _check(lib().duet_profile_smooth(s, len(sizes), t, len(table)))
    return list(t)


def duet_corun_choose(total_sms, cand_sd_sms, fa_flops_at_sms, dec_bw_at_sms, attn_flops_pre, attn_bytes_dec,
                      min_sms=16, overhead_s=15e-6):
    """(s_d, t): the f4 attention co-run split of a temporal step (0 = one after the other)."""
    cand = (C.c_int32 * max(1, len(cand_sd_sms)))(*cand_sd_sms)
    fa = (C.c_double * (total_sms + 1))(*fa_flops_at_sms)
    bw = (C.c_double * (total_sms + 1))(*dec_bw_at_sms)
    p = duet_corun_profile(total_sms, len(cand_sd_sms), cand, fa, bw, min_sms, overhead_s)
    sd, t = C.c_int32(), C.c_double()
    _check(lib().duet_corun_choose(C.byref(p), float(attn_flops_pre), float(attn_bytes_dec), C.byref(sd), C.byref(t)))
    return sd.value, t.value


def split_tuple(s: duet_split):
    return (s.mode, s.s_p, s.s_d, s.k, s.flags, s.t_mixed, s.t_p, s.t_d, s.rho)


# ------------------------------------------------------------------ execution context

def _i32(a):
    import numpy as np
    a = np.ascontiguousarray(a, dtype=np.int32)
    return a, a.ctypes.data_as(C.POINTER(C.c_int32))


def _ptr(t):
    return None if t is None else C.c_void_p(t.data_ptr())


class duet_sched_cfg(C.Structure):
    _fields_ = [(n, C.c_int32) for n in ("page_size", "n_pages", "token_budget", "max_batch", "max_prefill_seqs",
                                           "k_max", "max_pages_per_seq")]


class duet_iteration(C.Structure):
    _fields_ = [("n_prefill", C.c_int32), ("n_decode", C.c_int32), ("ids", C.POINTER(C.c_int64)),
                ("q", C.POINTER(C.c_int32)), ("c", C.POINTER(C.c_int32)), ("page_table", C.POINTER(C.c_int32)),
                ("max_pages", C.c_int32), ("next_arrival_s", C.c_double), ("n_unfinished", C.c_int32)]


class Sched:
    """Iteration stream (duet_sched_*): decode-first chunked-prefill batch former + KV page allocator."""

    def __init__(self, page_size=16, n_pages=1 << 16, token_budget=8192, max_batch=1024, max_prefill_seqs=16,
                 k_max=8, max_pages_per_seq=4096):
        cfg = duet_sched_cfg(page_size, n_pages, token_budget, max_batch, max_prefill_seqs, k_max, max_pages_per_seq)
        h = C.c_void_p()
        _check(lib().duet_sched_create(C.byref(cfg), C.byref(h)))
        self.h = h
        self.page_size = page_size

    def close(self):
        if self.h:
            lib().duet_sched_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def add(self, rid: int, prompt: int, output: int, arrival: float):
        _check(lib().duet_sched_add(self.h, int(rid), int(prompt), int(output), float(arrival)))

    def next(self, now: float) -> dict:
        """dict(prefill=[(id, q, c)], decode=[(id, c)], table=np.int32 [n, max_pages], next_arrival, unfinished)."""
        import numpy as np
        it = duet_iteration()
        _check(lib().duet_sched_next(self.h, float(now), C.byref(it)))
        n = it.n_prefill + it.n_decode
        ids = [it.ids[i] for i in range(n)]
        q = [it.q[i] for i in range(n)]
        c = [it.c[i] for i in range(n)]
        tab = np.ctypeslib.as_array(it.page_table, shape=(max(n, 1), max(it.max_pages, 1))).copy()[:n] if n else \
            np.zeros((0, 1), dtype=np.int32)
        return dict(prefill=[(ids[i], q[i], c[i]) for i in range(it.n_prefill)],
                    decode=[(ids[i], c[i]) for i in range(it.n_prefill, n)], table=tab,
                    next_arrival=it.next_arrival_s, unfinished=it.n_unfinished)

    def commit(self, k_done: int):
        t, f = C.c_int32(), C.c_int32()
        _check(lib().duet_sched_commit(self.h, int(k_done), C.byref(t), C.byref(f)))
        return t.value, f.value

    def free_pages(self) -> int:
        v = C.c_int32()
        _check(lib().duet_sched_free_pages(self.h, C.byref(v)))
        return v.value


def nccl_unique_id() -> bytes:
    """A fresh ncclUniqueId (128 bytes) for duet_ctx_set_comms (duet_nccl_unique_id)."""
    buf = C.create_string_buffer(128)
    _check(lib().duet_nccl_unique_id(buf, 128))
    return buf.raw


def open_fused_allreduce(ctx, group=None):
    """f3 plumbing over torch.distributed: all-gather every rank's fused-allreduce arena handle
    (duet_ctx_ar_handle, 64 bytes) in rank order and map the peers' arenas (duet_ctx_ar_open).
    Collective over the group; every rank's ctx must have its communicators set."""
    import torch.distributed as dist
    h = ctx.ar_handle()
    hs = [None] * dist.get_world_size(group)
    dist.all_gather_object(hs, h, group=group)
    ctx.ar_open(hs)
    return hs


class Ctx:
    """Owns a duet_ctx.  Device tensors are torch tensors (plumbing only)."""

    def __init__(self, spec: duet_model_spec, max_prefill_tokens, max_prefill_seqs, max_decode_reqs, max_k,
                 max_pages_per_seq, max_pos, dtype=DUET_DTYPE_BF16, flags=0, device=0):
        lim = duet_ctx_limits(max_prefill_tokens, max_prefill_seqs, max_decode_reqs, max_k, max_pages_per_seq,
                              max_pos, dtype, flags)
        h = C.c_void_p()
        _check(lib().duet_ctx_create(int(device), C.byref(spec), C.byref(lim), C.byref(h)))
        self.h = h
        self.spec = spec
        self.dtype = dtype

    def close(self):
        if self.h:
            _check(lib().duet_ctx_destroy(self.h))
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def partitions(self):
        n = C.c_int32(0)
        tot = C.c_int32(0)
        _check(lib().duet_ctx_partitions(self.h, None, C.byref(n), C.byref(tot)))
        arr = (C.c_int32 * max(1, n.value))()
        _check(lib().duet_ctx_partitions(self.h, arr, C.byref(n), C.byref(tot)))
        return list(arr[:n.value]), tot.value

    def step(self, layer_weights, prefill, decode, kv_k, kv_v, n_pages, split: duet_split, stream=None):
        """layer_weights: list of dicts of torch tensors; prefill: dict(q, c, table, x, y) or None;
        decode: dict(c, table, x, y) or None; kv_k/kv_v: lists of per-layer pools."""
        L = len(layer_weights)
        W = (duet_layer_weights * L)()
        for l, w in enumerate(layer_weights):
            W[l] = duet_layer_weights(*[w.get(n).data_ptr() if w.get(n) is not None else None
                                        for n in ("w_qkv", "b_qkv", "w_o", "w_gate_up", "w_down", "g_norm1",
                                                  "g_norm2")])
        keep = []
        pre_s = None
        if prefill is not None:
            q, qp = _i32(prefill["q"])
            c, cp = _i32(prefill["c"])
            t, tp = _i32(prefill["table"])
            keep += [q, c, t]
            pre_s = duet_prefill(len(q), qp, cp, tp, t.shape[1], _ptr(prefill["x"]), _ptr(prefill["y"]))
        dec_s = None
        if decode is not None:
            c, cp = _i32(decode["c"])
            t, tp = _i32(decode["table"])
            keep += [c, t]
            head_p = None
            if decode.get("head") is not None:   # dict(g_norm, w_head, embed, tokens) of device tensors (f1)
                hd = decode["head"]
                hs = duet_lm_head(_ptr(hd["g_norm"]), _ptr(hd["w_head"]), _ptr(hd["embed"]), _ptr(hd["tokens"]))
                keep.append(hs)
                head_p = C.pointer(hs)
            dec_s = duet_decode(len(c), cp, tp, t.shape[1], _ptr(decode["x"]), _ptr(decode["y"]), head_p)
        kp = (C.c_void_p * L)(*[p.data_ptr() for p in kv_k])
        vp = (C.c_void_p * L)(*[p.data_ptr() for p in kv_v])
        kv = duet_kv_pages(kp, vp, int(n_pages), 16)
        if stream is None:
            stream = torch.cuda.current_stream().cuda_stream
        _check(lib().duet_step(self.h, W, C.byref(pre_s) if pre_s is not None else None,
                               C.byref(dec_s) if dec_s is not None else None, C.byref(kv), C.byref(split),
                               C.c_void_p(stream)))

    def last_step_times(self) -> dict:
        out = duet_step_times()
        _check(lib().duet_last_step_times(self.h, C.byref(out)))
        return {n: getattr(out, n) for n, _ in duet_step_times._fields_}

    def profile_enable(self, on=True):
        """on: False/0 = off, True = every kernel class, or a bitmask of 1 << DUET_KCLASS_*."""
        mask = DUET_PROFILE_ALL if on is True else int(on)
        _check(lib().duet_profile_enable(self.h, mask))

    def profile_read(self) -> dict:
        arr = (duet_kernel_stats * DUET_KCLASS_N)()
        _check(lib().duet_profile_read(self.h, arr))
        names = ("gemm", "prefill_attn", "decode_attn", "other", "gemm_decode", "other_decode")
        return {names[i]: {n: getattr(arr[i], n) for n, _ in duet_kernel_stats._fields_} for i in range(DUET_KCLASS_N)}

    def set_comms(self, rank: int, id_decode: bytes, id_prefill: bytes):
        """Tensor parallelism: collective over the tp ranks (duet_ctx_set_comms)."""
        a = C.create_string_buffer(bytes(id_decode), 128)
        b = C.create_string_buffer(bytes(id_prefill), 128)
        _check(lib().duet_ctx_set_comms(self.h, int(rank), a, b))

    def last_pod(self) -> bool:
        """Did the last temporal step run its attentions as the fused POD launch (duet_ctx_last_pod)?"""
        return bool(lib().duet_ctx_last_pod(self.h))

    def check_comms(self):
        """Raises DuetError(NCCL) when a communicator reports an asynchronous error (duet_ctx_check_comms)."""
        _check(lib().duet_ctx_check_comms(self.h))

    def ar_handle(self) -> bytes:
        """This rank's fused-allreduce arena as a 64-byte cudaIpcMemHandle_t (duet_ctx_ar_handle)."""
        buf = C.create_string_buffer(64)
        _check(lib().duet_ctx_ar_handle(self.h, buf, 64))
        return buf.raw

    def ar_open(self, handles):
        """handles: every rank's ar_handle() in rank order (duet_ctx_ar_open)."""
        blob = b"".join(bytes(h) for h in handles)
        buf = C.create_string_buffer(blob, len(blob))
        _check(lib().duet_ctx_ar_open(self.h, len(handles), buf))

    def op_gemm_ar_emul(self, A, B, R, Cout, stream=None):
        """A [n][M][K], B [n][N][K], R [M][N], Cout [n][M][N] (duet_op_gemm_ar_emul)."""
        n, M, K = A.shape
        N = B.shape[1]
        if stream is None:
            stream = torch.cuda.current_stream().cuda_stream
        _check(lib().duet_op_gemm_ar_emul(self.h, n, _ptr(A), _ptr(B), _ptr(R), _ptr(Cout), M, N, K,
                                          C.c_void_p(stream)))

    def calibrate_allreduce(self):
        """(alpha seconds, B_NVLink bytes/s) of the P:237 allreduce model (duet_calibrate_allreduce)."""
        a, b = C.c_double(), C.c_double()
        _check(lib().duet_calibrate_allreduce(self.h, C.byref(a), C.byref(b)))
        return a.value, b.value

    def calibrate(self, total_sms: int):
        fl = (C.c_double * (total_sms + 1))()
        bw = (C.c_double * (total_sms + 1))()
        _check(lib().duet_calibrate(self.h, fl, bw, total_sms + 1))
        return list(fl), list(bw)

    def calibrate_corun(self, total_sms: int, pair_seconds: float = 0.12):
        """Pi_SM(S), B_HBM(S) measured under co-run at sustained clocks (duet_calibrate_corun)."""
        fl = (C.c_double * (total_sms + 1))()
        bw = (C.c_double * (total_sms + 1))()
        _check(lib().duet_calibrate_corun(self.h, fl, bw, total_sms + 1, float(pair_seconds)))
        return list(fl), list(bw)

    def calibrate_stream(self, total_sms: int):
        """LDG stream ceiling (B/s) per achievable partition size (duet_calibrate_stream); 0 elsewhere."""
        bw = (C.c_double * (total_sms + 1))()
        _check(lib().duet_calibrate_stream(self.h, bw, total_sms + 1))
        return list(bw)

    def op_gemm(self, A, B, Cout, R=None, bias=None, epi=DUET_EPI_STORE, stream=None):
        M, K = A.shape
        N = Cout.shape[1]
        if stream is None:
            stream = torch.cuda.current_stream().cuda_stream
        _check(lib().duet_op_gemm(self.h, _ptr(A), _ptr(B), _ptr(Cout), _ptr(R), _ptr(bias), M, N, K, epi,
                                  C.c_void_p(stream)))

    def op_rmsnorm(self, x, g, h, stream=None):
        if stream is None:
            stream = torch.cuda.current_stream().cuda_stream
        _check(lib().duet_op_rmsnorm(self.h, _ptr(x), _ptr(g), _ptr(h), x.shape[0], C.c_void_p(stream)))


    def op_decode_attn(self, q, o, pos, table, k_pool, v_pool, n_pages, s_d=0, stream=None):
        """q: [n][>= h_q d_h] device rows (stride q.stride(0)); pos: host [n]; table: host [n][max_pages]."""
        p, pp = _i32(pos)
        t, tp = _i32(table)
        if stream is None:
            stream = torch.cuda.current_stream().cuda_stream
        _check(lib().duet_op_decode_attn(self.h, _ptr(q), q.stride(0), _ptr(o), len(p), pp, tp, t.shape[1],
                                         _ptr(k_pool), _ptr(v_pool), int(n_pages), int(s_d), C.c_void_p(stream)))

    def op_prefill_attn(self, q, o, q_len, c, table, k_pool, v_pool, n_pages, s_p=0, stream=None):
        """q: [sum q_len][>= h_q d_h] device rows; q_len, c: host [n_seqs]; table: host [n_seqs][max_pages]."""
        ql, qlp = _i32(q_len)
        cc, cp = _i32(c)
        t, tp = _i32(table)
        if stream is None:
            stream = torch.cuda.current_stream().cuda_stream
        _check(lib().duet_op_prefill_attn(self.h, _ptr(q), q.stride(0), _ptr(o), len(ql), qlp, cp, tp, t.shape[1],
                                          _ptr(k_pool), _ptr(v_pool), int(n_pages), int(s_p), C.c_void_p(stream)))

    def token_times_reset(self):
        _check(lib().duet_token_times(self.h, 1, None, 0, None))

    def token_times(self, reset=True):
        """%globaltimer stamps (ns) of the decode steps since the last reset (duet_token_times)."""
        n = C.c_int32(0)
        _check(lib().duet_token_times(self.h, 0, None, 0, C.byref(n)))
        arr = (C.c_uint64 * max(1, n.value))()
        _check(lib().duet_token_times(self.h, int(bool(reset)), arr, n.value, C.byref(n)))
        return list(arr[:n.value])


def split_struct(mode, s_p, s_d, k, flags=0, t_mixed=0.0, t_p=0.0, t_d=0.0, rho=0.0) -> duet_split:
    return duet_split(mode, s_p, s_d, k, flags, t_mixed, t_p, t_d, rho)


__all__ = [n for n in dir() if n.startswith(("duet_", "DUET_"))] + [
    "Ctx", "HwProfile", "make_spec", "split_struct", "split_tuple", "lib", "DuetError", "EXPORTED", "LIB_PATH",
    "nccl_unique_id", "Sched"]

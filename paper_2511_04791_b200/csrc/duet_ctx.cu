// Execution context and the mixed-iteration step of DuetServe on one B200.
//
//  * SM partitions (§4.3): a pre-created pool of green-context pairs, one pair per
//    achievable decode size S_d (the CUDA driver provisions disjoint SM sets; probe evidence in
//    profiles/r01_probe_green_ctx.txt).  libsmctrl is prior art resting on driver
//    internals and is not used.
//  * Interruption-free dispatch: decode is launched first as k replays of one
//    captured CUDA graph per (partition, batch shape); the graph reads positions and the step
//    index from device memory, so the k steps need no host synchronization; prefill kernels
//    are launched one by one on the other partition's stream; both sides join on events.
//  * Temporal mode (Alg. 1 l.4): the same kernels on one full-device stream over the
//    concatenated rows [prefill ; decode].
#include <cuda.h>
#include <dlfcn.h>
#include <nccl.h>  // types only: libnccl is dlopen-ed (the one torch already loaded)
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <array>
#include <map>
#include <tuple>
#include <vector>

#include "duet_common.h"
#include "kernels.h"

using namespace duet;

#define CUDA_TRY(expr)                                                                              \
  do {                                                                                              \
    cudaError_t e_ = (expr);                                                                        \
    if (e_ != cudaSuccess)                                                                          \
      DUET_FAIL(DUET_ERR_CUDA, "%s failed: %s (%s:%d)", #expr, cudaGetErrorString(e_), __FILE__, __LINE__); \
  } while (0)
#define CU_TRY(expr)                                                                                \
  do {                                                                                              \
    CUresult r_ = (expr);                                                                           \
    if (r_ != CUDA_SUCCESS) {                                                                       \
      const char* s_ = nullptr;                                                                     \
      DRV.GetErrorString(r_, &s_);                                                                    \
      DUET_FAIL(DUET_ERR_CUDA, "%s failed: %s (%s:%d)", #expr, s_ ? s_ : "?", __FILE__, __LINE__); \
    }                                                                                               \
  } while (0)

namespace {

// Driver entry points, resolved through the runtime (no link-time dependency on libcuda, so
// the library also loads on a GPU-less host for the predictor / optimizer).
struct Driver {
  bool ok = false;
  CUresult (*Init)(unsigned) = nullptr;
  CUresult (*DeviceGet)(CUdevice*, int) = nullptr;
  CUresult (*DeviceGetDevResource)(CUdevice, CUdevResource*, CUdevResourceType) = nullptr;
  CUresult (*DevSmResourceSplitByCount)(CUdevResource*, unsigned*, const CUdevResource*, CUdevResource*, unsigned,
                                        unsigned) = nullptr;
  CUresult (*DevResourceGenerateDesc)(CUdevResourceDesc*, CUdevResource*, unsigned) = nullptr;
  CUresult (*GreenCtxCreate)(CUgreenCtx*, CUdevResourceDesc, CUdevice, unsigned) = nullptr;
  CUresult (*GreenCtxStreamCreate)(CUstream*, CUgreenCtx, unsigned, int) = nullptr;
  CUresult (*GreenCtxDestroy)(CUgreenCtx) = nullptr;
  CUresult (*StreamDestroy)(CUstream) = nullptr;
  CUresult (*GetErrorString)(CUresult, const char**) = nullptr;
};
Driver DRV;

duet_status load_driver() {
  if (DRV.ok) return DUET_OK;
  auto get = [](const char* name, void** fn) -> duet_status {
    cudaDriverEntryPointQueryResult q;
    cudaError_t e = cudaGetDriverEntryPointByVersion(name, fn, 12080, cudaEnableDefault, &q);
    if (e != cudaSuccess || q != cudaDriverEntryPointSuccess || !*fn)
      DUET_FAIL(DUET_ERR_CUDA, "driver entry point %s unavailable", name);
    return DUET_OK;
  };
  DUET_TRY(get("cuInit", (void**)&DRV.Init));
  DUET_TRY(get("cuDeviceGet", (void**)&DRV.DeviceGet));
  DUET_TRY(get("cuDeviceGetDevResource", (void**)&DRV.DeviceGetDevResource));
  DUET_TRY(get("cuDevSmResourceSplitByCount", (void**)&DRV.DevSmResourceSplitByCount));
  DUET_TRY(get("cuDevResourceGenerateDesc", (void**)&DRV.DevResourceGenerateDesc));
  DUET_TRY(get("cuGreenCtxCreate", (void**)&DRV.GreenCtxCreate));
  DUET_TRY(get("cuGreenCtxStreamCreate", (void**)&DRV.GreenCtxStreamCreate));
  DUET_TRY(get("cuGreenCtxDestroy", (void**)&DRV.GreenCtxDestroy));
  DUET_TRY(get("cuStreamDestroy", (void**)&DRV.StreamDestroy));
  DUET_TRY(get("cuGetErrorString", (void**)&DRV.GetErrorString));
  DRV.ok = true;
  return DUET_OK;
}

// NCCL (tensor parallelism), resolved at run time from the process's libnccl.so.2 (PyTorch
// loads one; no link-time dependency), only when a context is given communicators.
struct NcclApi {
  bool ok = false;
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommInitRankConfig)(ncclComm_t*, int, ncclUniqueId, int, ncclConfig_t*) = nullptr;
  ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t*) = nullptr;
  ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};
NcclApi NCCL;

duet_status load_nccl() {
  if (NCCL.ok) return DUET_OK;
  void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
  if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
  if (!h) DUET_FAIL(DUET_ERR_NCCL, "libnccl.so.2 not found: %s", dlerror());
  auto get = [&](const char* name, void** fn) -> duet_status {
    *fn = dlsym(h, name);
    if (!*fn) DUET_FAIL(DUET_ERR_NCCL, "NCCL symbol %s missing", name);
    return DUET_OK;
  };
  DUET_TRY(get("ncclGetUniqueId", (void**)&NCCL.GetUniqueId));
  DUET_TRY(get("ncclCommInitRank", (void**)&NCCL.CommInitRank));
  DUET_TRY(get("ncclCommInitRankConfig", (void**)&NCCL.CommInitRankConfig));
  DUET_TRY(get("ncclCommGetAsyncError", (void**)&NCCL.CommGetAsyncError));
  DUET_TRY(get("ncclAllReduce", (void**)&NCCL.AllReduce));
  DUET_TRY(get("ncclCommDestroy", (void**)&NCCL.CommDestroy));
  DUET_TRY(get("ncclGetErrorString", (void**)&NCCL.GetErrorString));
  NCCL.ok = true;
  return DUET_OK;
}

#define NCCL_TRY(expr)                                                                            \
  do {                                                                                            \
    ncclResult_t r_ = (expr);                                                                     \
    if (r_ != ncclSuccess) DUET_FAIL(DUET_ERR_NCCL, "%s failed: %s", #expr, NCCL.GetErrorString(r_)); \
  } while (0)

constexpr int kPageSize = 16;
constexpr int kStageSlots = 4;
constexpr int kMaxSplits = 32;

struct Partition {
  int s_d = 0, s_p = 0;  // actual SM counts of the decode group and the remainder
  bool created = false;
  CUgreenCtx g_dec = nullptr, g_pre = nullptr;
  cudaStream_t s_dec = nullptr, s_pre = nullptr;
};

// Device workspace of one side (decode or prefill/temporal).
struct Side {
  int cap_rows = 0, cap_seqs = 0, cap_table_rows = 0, pitch = 0;
  void *xa = nullptr, *xb = nullptr, *h = nullptr, *qkv = nullptr, *o = nullptr, *x1 = nullptr, *h2 = nullptr,
       *act = nullptr, *xin = nullptr, *ylast = nullptr;
  int* meta = nullptr;  // [pos | tok_row | row0 | qlen | cpre | seq_row | step | order | table]
  float *part_o = nullptr, *part_ml = nullptr;
  int part_rows = 0;
  void* logits = nullptr;    // LM head (f1): [decode rows][vocab]
  float* gemm_ws = nullptr;  // split-K partials of the weight-streaming GEMMs (kernels.h GemmArgs)
  size_t gemm_ws_floats = 0;
  // offsets into meta (ints)
  size_t o_pos = 0, o_tok = 0, o_row0 = 0, o_qlen = 0, o_cpre = 0, o_seqrow = 0, o_step = 0, o_order = 0, o_table = 0,
         n_meta = 0;
  int* pos() const { return meta + o_pos; }
  int* order() const { return meta + o_order; }  // decode rows, longest context first
  int* tok() const { return meta + o_tok; }
  int* row0() const { return meta + o_row0; }
  int* qlen() const { return meta + o_qlen; }
  int* cpre() const { return meta + o_cpre; }
  int* seqrow() const { return meta + o_seqrow; }
  int* step() const { return meta + o_step; }
  int* table() const { return meta + o_table; }
};

struct GraphEntry {
  cudaGraphExec_t exec = nullptr;
  int kernels = 0;
  uint64_t last_use = 0;
};
// decode graphs kept per ctx (key: partition, batch size, layers, pointer hash, context bucket); the
// least recently used one is destroyed beyond this many (a serving loop changes the batch size often)
constexpr size_t kGraphCap = 48;
// prefill-side graphs (f4): one per repeated prefill shape; captured on a shape's second
// occurrence (a serving loop's one-off chunk shapes would pay the capture for nothing)
constexpr size_t kPreGraphCap = 8;
using PreKey = std::array<uint64_t, 6>;

}  // namespace

struct duet_ctx {
  int device = 0;
  duet_model_spec spec{};   // this rank's shard: h_q/tp, h_kv/tp, ffn_dim/tp (d_model, head_dim global)
  duet_model_spec gspec{};  // the model as given (tp = tensor-parallel degree)
  int tp_rank = 0;
  ncclComm_t comm_dec = nullptr, comm_pre = nullptr;  // one communicator per side
  duet_ctx_limits lim{};
  DT dt = DT::BF16;
  int total_sms = 0;
  CUdevice cudev = 0;
  CUdevResource sm_all{};
  std::vector<Partition> parts;
  cudaStream_t s_full = nullptr;
  cudaEvent_t ev_in = nullptr, ev_dec0 = nullptr, ev_dec1 = nullptr, ev_pre0 = nullptr, ev_pre1 = nullptr;
  // temporal-mode attention co-run: prefill attention on the remainder, decode
  // attention on an S_d group, forked from and joined back into the full-device stream per layer
  Partition* corun = nullptr;
  cudaEvent_t ev_cf = nullptr, ev_ca = nullptr, ev_cb = nullptr;
  float2* rope = nullptr;
  Side dec, pre;
  int* stage = nullptr;  // pinned, mapped [kStageSlots][stage_ints]
  int* stage_dev = nullptr;  // its device address (read zero-copy by launch_copy_bytes)
  size_t stage_ints = 0;
  cudaEvent_t stage_ev[kStageSlots] = {};
  // metadata prefetch (§5.3): device copy of the ring, filled on s_up as soon as duet_step is called
  int* stage_d = nullptr;
  cudaStream_t s_up = nullptr;
  cudaEvent_t up_ev[kStageSlots] = {}, use_ev[kStageSlots] = {};
  int stage_next = 0;
  std::vector<uint32_t> page_mark;
  uint32_t page_gen = 0;
  std::map<std::tuple<int, int, int, uint64_t>, GraphEntry> graphs;
  std::map<PreKey, GraphEntry> pre_graphs;
  std::map<PreKey, int> pre_seen;
  uint64_t graph_clock = 0;
  // last step
  int last_mode = -1, last_k = 0, last_kernels = 0, last_corun = 0;
  bool last_pod = false;  // the last temporal step ran its attentions as the fused POD launch (f4)
  bool last_pre_graph = false;  // the last spatial step's prefill side replayed a graph
  bool last_has_dec = false, last_has_pre = false;
  // live kernel timing
  bool prof_on = false, capturing = false;
  bool prof_dec_side = false;  // launches being made belong to a spatial step's decode side
  // device-side timing of the decode attention inside the decode graph (DecodeAttnArgs::dev_timer) and
  // the algorithmic work of the launches it timed
  unsigned long long* dev_timer = nullptr;
  double dtimer_flops = 0, dtimer_bytes = 0;
  int dtimer_launches = 0;
  int prof_mask = 0;
  struct ProfRec {
    int cls, idx;
    double flops, bytes;
  };
  std::vector<ProfRec> prof_pending;
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> prof_pool;
  size_t prof_used = 0;
  duet_kernel_stats prof_acc[DUET_KCLASS_N] = {};
  // f4 co-run rates per partition size (duet_corun_choose): prefill-attention FLOP/s, decode-attention B/s
  std::vector<double> cal_fa, cal_bw;
  // token-time ring (SURVEY §8(d) TBT per decode step): %globaltimer when each step's tokens are done
  unsigned long long* tok_ts = nullptr;
  int* tok_cnt = nullptr;
  // fused GEMM + allreduce: one IPC-exported arena per rank holding, per side, the
  // receive slots, the counters and the two [rows][d] outputs (x1 and the layer output) the owners push
  // into; ar_grp[side] is the group as seen from this rank (peer-mapped pointers), ar_on once opened
  struct ArSide {
    size_t off_slots = 0, off_cnt = 0, off_out0 = 0, off_out1 = 0;
  } ar_lay[2];
  size_t ar_bytes = 0;
  char* ar_arena = nullptr;
  char* ar_peer[kMaxTp] = {};
  GemmAr ar_grp[2];
  bool ar_on = false;
  // duet_op_gemm_ar_emul workspace (every emulated rank's slots and counters)
  float* emu_slots = nullptr;
  unsigned* emu_cnt = nullptr;
  size_t emu_slot_floats = 0, emu_cnt_n = 0;
};

static duet_status comms_healthy(duet_ctx* c);

// decode-side launches of a spatial step are counted in the *_DECODE classes
static int side_class(duet_ctx* c, int cls) {
  if (!c->prof_dec_side) return cls;
  return cls == DUET_KCLASS_GEMM ? DUET_KCLASS_GEMM_DECODE : cls == DUET_KCLASS_OTHER ? DUET_KCLASS_OTHER_DECODE : cls;
}
static int prof_begin(duet_ctx* c, cudaStream_t st, int cls) {
  cls = side_class(c, cls);
  if (!c->prof_on || c->capturing || !(c->prof_mask & (1 << cls))) return -1;
  if (c->prof_used == c->prof_pool.size()) {
    cudaEvent_t a, b;
    if (cudaEventCreate(&a) != cudaSuccess || cudaEventCreate(&b) != cudaSuccess) return -1;
    c->prof_pool.emplace_back(a, b);
  }
  const int idx = (int)c->prof_used++;
  cudaEventRecord(c->prof_pool[idx].first, st);
  return idx;
}
static void prof_end(duet_ctx* c, cudaStream_t st, int idx, int cls, double flops, double bytes) {
  if (idx < 0) return;
  cls = side_class(c, cls);
  cudaEventRecord(c->prof_pool[idx].second, st);
  c->prof_pending.push_back({cls, idx, flops, bytes});
}

// ---------------------------------------------------------------------------------- helpers

static duet_status side_alloc(duet_ctx* c, Side& s, int cap_rows, int cap_seqs, int cap_table_rows, int part_rows) {
  const auto& sp = c->spec;
  const size_t es = dt_size(c->dt);
  const size_t d = sp.d_model, nqkv = (size_t)(sp.n_q_heads + 2 * sp.n_kv_heads) * sp.head_dim;
  const size_t nq = (size_t)sp.n_q_heads * sp.head_dim, m = sp.ffn_dim;
  s.cap_rows = cap_rows;
  s.cap_seqs = cap_seqs;
  s.cap_table_rows = cap_table_rows;
  s.pitch = c->lim.max_pages_per_seq;
  const size_t R = std::max(cap_rows, 1);
  CUDA_TRY(cudaMalloc(&s.xa, R * d * es));
  CUDA_TRY(cudaMalloc(&s.xb, R * d * es));
  CUDA_TRY(cudaMalloc(&s.h, R * d * es));
  CUDA_TRY(cudaMalloc(&s.x1, R * d * es));
  CUDA_TRY(cudaMalloc(&s.h2, R * d * es));
  CUDA_TRY(cudaMalloc(&s.xin, R * d * es));
  CUDA_TRY(cudaMalloc(&s.ylast, R * d * es));
  CUDA_TRY(cudaMalloc(&s.qkv, R * nqkv * es));
  CUDA_TRY(cudaMalloc(&s.o, R * nq * es));
  CUDA_TRY(cudaMalloc(&s.act, R * m * es));
  s.part_rows = std::max(part_rows, 1);
  CUDA_TRY(cudaMalloc(&s.part_o, (size_t)s.part_rows * sp.n_q_heads * kMaxSplits * sp.head_dim * sizeof(float)));
  CUDA_TRY(cudaMalloc(&s.part_ml, (size_t)s.part_rows * sp.n_q_heads * kMaxSplits * 2 * sizeof(float)));
  // split-K workspace: the largest need over the layer's four GEMMs at any M <= min(cap_rows, 128)
  for (int M : {std::min(cap_rows, 64), std::min(cap_rows, 128)}) {
    const int shapes[4][3] = {{(int)nqkv, (int)d, EPI_STORE}, {(int)d, (int)nq, EPI_RESIDUAL},
                              {(int)m, (int)d, EPI_SWIGLU}, {(int)d, (int)m, EPI_RESIDUAL}};
    for (auto& sh : shapes) s.gemm_ws_floats = std::max(s.gemm_ws_floats, gemm_tc_splitk_need(M, sh[0], sh[1], sh[2]));
  }
  // ... and of the CTA-pair GEMMs of under-filled grids (M > 128 in 256-row steps up to cap_rows)
  for (int M = 256; M - 256 < cap_rows && M <= 4096; M += 256) {
    const int Mc = std::min(M, cap_rows);
    const int shapes[2][3] = {{(int)d, (int)nq, EPI_RESIDUAL}, {(int)d, (int)m, EPI_RESIDUAL}};
    for (auto& sh : shapes) s.gemm_ws_floats = std::max(s.gemm_ws_floats, gemm2_splitk_need(Mc, sh[0], sh[1], sh[2]));
    s.gemm_ws_floats = std::max(s.gemm_ws_floats, gemm2_splitk_need(Mc, (int)nqkv, (int)d, EPI_STORE));
  }
  if (s.gemm_ws_floats > 0) CUDA_TRY(cudaMalloc(&s.gemm_ws, s.gemm_ws_floats * sizeof(float)));
  // LM head logits of the decode rows (f1), bf16 contexts with a vocabulary
  if (c->dt == DT::BF16 && sp.vocab > 0 && c->lim.max_decode_reqs > 0)
    CUDA_TRY(cudaMalloc(&s.logits, (size_t)c->lim.max_decode_reqs * sp.vocab * es));
  size_t off = 0;
  s.o_pos = off; off += R;
  s.o_tok = off; off += R;
  s.o_row0 = off; off += cap_seqs + 1;
  s.o_qlen = off; off += cap_seqs + 1;
  s.o_cpre = off; off += cap_seqs + 1;
  s.o_seqrow = off; off += cap_seqs + 1;
  s.o_step = off; off += 4;
  s.o_order = off; off += R;
  s.o_table = off; off += (size_t)std::max(cap_table_rows, 1) * s.pitch;
  s.n_meta = off;
  CUDA_TRY(cudaMalloc(&s.meta, s.n_meta * sizeof(int)));
  CUDA_TRY(cudaMemset(s.meta, 0, s.n_meta * sizeof(int)));
  return DUET_OK;
}

static void side_free(Side& s) {
  void* ptrs[] = {s.xa, s.xb, s.h, s.x1, s.h2, s.xin, s.ylast, s.qkv, s.o, s.act, s.part_o, s.part_ml, s.meta, s.gemm_ws, s.logits};
  for (void* p : ptrs)
    if (p) cudaFree(p);
  s = Side{};
}

static duet_status ensure_partition(duet_ctx* c, Partition& p) {
  if (p.created) return DUET_OK;
  const unsigned flags = (c->lim.flags & DUET_CTX_FINE_SPLIT) ? CU_DEV_SM_RESOURCE_SPLIT_IGNORE_SM_COSCHEDULING : 0;
  CUdevResource grp[1], rem;
  unsigned n = 1;
  CU_TRY(DRV.DevSmResourceSplitByCount(grp, &n, &c->sm_all, &rem, flags, (unsigned)p.s_d));
  if (n != 1 || (int)grp[0].sm.smCount != p.s_d)
    DUET_FAIL(DUET_ERR_CUDA, "green-context split for S_d = %d gave %u SMs", p.s_d, grp[0].sm.smCount);
  CUdevResourceDesc d1, d2;
  CU_TRY(DRV.DevResourceGenerateDesc(&d1, grp, 1));
  CU_TRY(DRV.DevResourceGenerateDesc(&d2, &rem, 1));
  CU_TRY(DRV.GreenCtxCreate(&p.g_dec, d1, c->cudev, CU_GREEN_CTX_DEFAULT_STREAM));
  CU_TRY(DRV.GreenCtxCreate(&p.g_pre, d2, c->cudev, CU_GREEN_CTX_DEFAULT_STREAM));
  CUstream s1, s2;
  CU_TRY(DRV.GreenCtxStreamCreate(&s1, p.g_dec, CU_STREAM_NON_BLOCKING, 0));
  CU_TRY(DRV.GreenCtxStreamCreate(&s2, p.g_pre, CU_STREAM_NON_BLOCKING, 0));
  p.s_dec = (cudaStream_t)s1;
  p.s_pre = (cudaStream_t)s2;
  p.s_p = (int)rem.sm.smCount;
  p.created = true;
  return DUET_OK;
}

static duet_status check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) DUET_FAIL(DUET_ERR_CUDA, "launch of %s failed: %s", what, cudaGetErrorString(e));
  return DUET_OK;
}

// Attention plan of one layer-stack run: prefill rows [0, n_pre), decode rows [n_pre, n_pre + n_dec).
struct AttnPlan {
  int n_pre = 0, n_seqs = 0, max_q = 0, max_len_pre = 0;
  int n_dec = 0, max_len_dec = 0;
  // algorithmic work of one attention launch: causal FLOPs 4 h_q d_h (pos + 1) per query row;
  // bytes = q + o + each KV head read once per sequence
  double attn_flops_pre = 0, attn_bytes_pre = 0, attn_flops_dec = 0, attn_bytes_dec = 0;
};

// f4 co-run partition choice for a temporal step with both phases: duet_corun_choose on
// the ctx's per-size attention rates — measured by duet_calibrate (prefill attention FLOP/s, decode
// attention B/s on every partition side), until then the prior fitted on B200 in round 1
// (tools/gpu/run_corun.sh): ~4.0 TFLOP/s per SM, B(S) = 5.9 TB/s (1 - e^(-S/28)), 6.1 TB/s full device.
static Partition* corun_pick(duet_ctx* c, const AttnPlan& ap) {
  constexpr double kOverhead = 15e-6;  // fork / join / lost launch overlap per layer
  std::vector<int32_t> cand;
  for (auto& p : c->parts) cand.push_back(p.s_d);
  duet_corun_profile prof{c->total_sms, (int32_t)cand.size(), cand.data(), c->cal_fa.data(), c->cal_bw.data(), 16,
                          kOverhead};
  int32_t sd = 0;
  if (duet_corun_choose(&prof, ap.attn_flops_pre, ap.attn_bytes_dec, &sd, nullptr) != DUET_OK || sd == 0)
    return nullptr;
  for (auto& p : c->parts)
    if (p.s_d == sd) return &p;
  return nullptr;
}

// Causal prefill attention (a6.4) of the prefill rows of plan ap (metadata in side S) — the launch of
// duet_step and of duet_op_prefill_attn.  Returns the kernels launched (<= 0: could not launch).
static int prefill_attn(duet_ctx* c, Side& S, const AttnPlan& ap, const void* q, int q_stride, void* o,
                        int total_rows, const void* k_pool, const void* v_pool, int n_pages, int num_sms,
                        cudaStream_t st, PrefillAttnArgs* args_only = nullptr, const int* shape_dev = nullptr) {
  const auto& sp = c->spec;
  PrefillAttnArgs pa{};
  pa.q = q;
  pa.q_stride = q_stride;
  pa.o = o;
  pa.n_seqs = ap.n_seqs;
  pa.hq = sp.n_q_heads;
  pa.hkv = sp.n_kv_heads;
  pa.dh = sp.head_dim;
  pa.row0 = S.row0();
  pa.qlen = S.qlen();
  pa.cpre = S.cpre();
  pa.seq_row = S.seqrow();
  pa.table = S.table();
  pa.max_pages = S.pitch;
  pa.page_size = kPageSize;
  pa.k_pool = k_pool;
  pa.v_pool = v_pool;
  pa.max_q = ap.max_q;
  pa.total_q = ap.n_pre;
  pa.num_sms = num_sms;
  pa.tok_pos = S.pos();
  pa.tok_row = S.tok();
  pa.max_len = ap.max_len_pre;
  pa.n_pages = n_pages;
  pa.total_rows = total_rows;
  pa.shape_dev = shape_dev;
  if (args_only) {  // the fused POD launch takes the arguments
    *args_only = pa;
    return 1;
  }
  return launch_prefill_attn(c->dt, pa, st);
}

// Paged decode attention (a5.4, split-K + LSE combine) of the decode rows of plan ap, which follow the
// ap.n_pre prefill rows in side S's metadata; q / o point at the first decode row.
static int decode_attn(duet_ctx* c, Side& S, const AttnPlan& ap, const void* q, int q_stride, void* o,
                       const void* k_pool, const void* v_pool, int n_pages, int num_sms, cudaStream_t st,
                       unsigned long long* dev_timer = nullptr, DecodeAttnArgs* args_only = nullptr) {
  const auto& sp = c->spec;
  DecodeAttnArgs da{};
  da.q = q;
  da.q_stride = q_stride;
  da.o = o;
  da.n = ap.n_dec;
  da.hq = sp.n_q_heads;
  da.hkv = sp.n_kv_heads;
  da.dh = sp.head_dim;
  da.pos = S.pos() + ap.n_pre;
  da.tok_row = S.tok() + ap.n_pre;
  da.table = S.table();
  da.max_pages = S.pitch;
  da.page_size = kPageSize;
  da.k_pool = k_pool;
  da.v_pool = v_pool;
  da.part_o = S.part_o;
  da.part_ml = S.part_ml;
  da.max_splits = kMaxSplits;
  da.num_sms = num_sms;
  da.max_len = ((ap.max_len_dec + 1023) / 1024) * 1024;  // same bucket in both modes
  da.n_pages = n_pages;
  da.dev_timer = dev_timer;
  static const bool ordered = !getenv("DUET_DECODE_ORDER") || atoi(getenv("DUET_DECODE_ORDER")) != 0;
  da.order = ordered ? S.order() : nullptr;  // DUET_DECODE_ORDER=0: request order as given (A/B)
  if (args_only) {
    *args_only = da;
    return 1;
  }
  return launch_decode_attn(c->dt, da, st);
}

// x_in2 / y_final2 / row_split: rows >= row_split of the layer input / final output live in a second
// buffer (the temporal batch [prefill ; decode] read and written in the caller's buffers, no copies)
static duet_status run_layers(duet_ctx* c, Side& S, cudaStream_t st, int num_sms, int n_rows, const void* x_in,
                              void* y_final, const duet_layer_weights* w, const duet_kv_pages* kv, const AttnPlan& ap,
                              int* kernels, const void* x_in2 = nullptr, void* y_final2 = nullptr,
                              int row_split = 1 << 30, const int* n_dev = nullptr) {
  // n_dev (nullable): the rows live on the device (meta) and n_rows is the side's capacity — the kernels
  // are launched for the capacity and read the row count themselves, so a captured graph of this stack
  // replays for any prefill shape (f4; the spatial prefill side's graphs)
  const auto& sp = c->spec;
  const DT dt = c->dt;
  const size_t es = dt_size(dt);
  const int d = sp.d_model, hq = sp.n_q_heads, hkv = sp.n_kv_heads, dh = sp.head_dim, m = sp.ffn_dim;
  const int nqkv = (hq + 2 * hkv) * dh;
  const float eps = (float)sp.norm_eps;
  int nk = 0;
  const double n = n_rows, e = (double)es;
  // algorithmic work per launch: FLOPs 2MNK; bytes = operands read once + output
  auto gemm_fl = [&](double N, double K) { return 2.0 * n * N * K; };
  auto gemm_by = [&](double N, double K, double Nout, bool resid) {
    return (n * K + N * K + n * Nout + (resid ? n * Nout : 0.0)) * e;
  };
  ncclComm_t comm = (&S == &c->dec) ? c->comm_dec : c->comm_pre;
  const bool lead = comm == nullptr || c->tp_rank == 0;
  const ncclDataType_t nccl_dt = dt == DT::BF16 ? ncclBfloat16 : ncclFloat32;
  // sum of the ranks' partial [rows][d] rows in place (2 allreduces per layer)
  auto allreduce = [&](void* buf, int rows) -> int {
    if (!comm || rows <= 0) return 1;
    const ncclResult_t r = NCCL.AllReduce(buf, buf, (size_t)rows * d, nccl_dt, ncclSum, comm, st);
    return r == ncclSuccess ? 1 : -1;
  };
  // f3: with the fused-allreduce group open, the O and down projections of a > 128-row batch run as
  // one GEMM + allreduce kernel each (outputs in this side's arena buffers out0 / out1, pushed there by
  // the tiles' owner ranks); the NCCL allreduce stays for batches the CTA-pair kernel does not take
  const int side_i = (&S == &c->dec) ? 0 : 1;
  const bool ar_side = c->ar_on && comm != nullptr && dt == DT::BF16;
  GemmAr ar_o, ar_d;
  char* ar_out0 = nullptr;
  char* ar_out1 = nullptr;
  if (ar_side) {
    const auto& L = c->ar_lay[side_i];
    ar_o = c->ar_grp[side_i];
    ar_d = ar_o;
    for (int r = 0; r < ar_o.n; ++r) ar_d.out[r] = (char*)ar_o.out[r] + (L.off_out1 - L.off_out0);
    ar_out0 = c->ar_arena + L.off_out0;
    ar_out1 = c->ar_arena + L.off_out1;
  }
  const void* x_carry = x_in;
  auto with_ws = [&](GemmArgs& g) {
    g.ws = S.gemm_ws;
    g.ws_floats = S.gemm_ws_floats;
  };
  // DUET_DEBUG_SYNC=1: synchronize after every launch and report it (hang / fault triage only)
  static const bool dbg_sync = getenv("DUET_DEBUG_SYNC") != nullptr;
  // every launch is checked where it is made: a launcher returns the number of kernels it queued
  // (> 0 here, n_rows > 0) or a negative value when it could not launch (e.g. a TMA map that cannot be
  // encoded), which fails the step naming the call
#define TIMED(cls, fl, by, call)                                                                  \
  do {                                                                                            \
    const int pi_ = prof_begin(c, st, cls);                                                       \
    const int r_ = (call);                                                                        \
    if (r_ <= 0) DUET_FAIL(DUET_ERR_CUDA, "layer %d: %s could not be launched (%d)", l, #call, r_); \
    nk += r_;                                                                                     \
    prof_end(c, st, pi_, cls, fl, by);                                                            \
    if (dbg_sync && !c->capturing) {                                                              \
      fprintf(stderr, "[duet] layer %d: %s ...", l, #call);                                       \
      cudaError_t e_ = cudaStreamSynchronize(st);                                                 \
      fprintf(stderr, " %s\n", cudaGetErrorString(e_));                                           \
    }                                                                                             \
  } while (0)
  for (int l = 0; l < sp.n_layers; ++l) {
    const void* X = x_carry;  // layer 0: x_in; then the previous layer's output (ping-pong or arena)
    void* Y = l == sp.n_layers - 1 ? y_final : ((l & 1) ? S.xb : S.xa);
    const duet_layer_weights& W = w[l];
    // 1. h = RMSNorm(x) g1
    TIMED(DUET_KCLASS_OTHER, 4.0 * n * d, 2.0 * n * d * e,
          launch_rmsnorm(dt, X, W.g_norm1, S.h, n_rows, d, eps, st, l == 0 ? x_in2 : nullptr,
                         l == 0 ? row_split : 1 << 30, n_dev));
    // 2. qkv = h W_qkv^T (+ b);  3. RoPE + paged KV append (before attention) — fused into the
    // CTA-pair GEMM's epilogue when it runs (k and v never round-trip through the qkv buffer)
    RopeKvArgs ra{S.qkv, nullptr, n_rows, hq, hkv, dh, S.pos(), S.tok(), S.table(), S.pitch, kPageSize,
                  kv->k_pool[l], kv->v_pool[l], c->rope};
    GemmArgs g{S.h, W.w_qkv, S.qkv, nullptr, W.b_qkv, n_rows, nqkv, d, d, d, nqkv, 0, EPI_STORE};
    with_ws(g);
    g.m_dev = n_dev;
    static const bool fuse_env = !getenv("DUET_FUSE_ROPE") || atoi(getenv("DUET_FUSE_ROPE")) != 0;
    const bool fuse_rope = fuse_env && dt == DT::BF16 && dh == 128 && kPageSize == 16 && gemm2_supported(g, num_sms);
    if (fuse_rope) {
      g.epi = EPI_QKV_ROPE;
      g.rope = &ra;
    }
    TIMED(DUET_KCLASS_GEMM, gemm_fl(nqkv, d), gemm_by(nqkv, d, nqkv, false), launch_gemm(dt, g, num_sms, st));
    if (!fuse_rope && n_dev) DUET_FAIL(DUET_ERR_UNSUPPORTED, "device-side row counts need the fused RoPE epilogue");
    if (!fuse_rope)
      TIMED(DUET_KCLASS_OTHER, 6.0 * n * (hq + hkv) * dh, n * (nqkv + (hq + 2.0 * hkv) * dh) * e,
            launch_rope_kv(dt, ra, st));
    // 4. attention; with a co-run partition the two attentions run side by side (compute-bound
    // prefill on the remainder, HBM-bound decode on S_d SMs) and the O GEMM waits for both
    Partition* cp = (c->corun && ap.n_pre > 0 && ap.n_dec > 0 && !c->capturing) ? c->corun : nullptr;
    // f4 POD-style fused attention (kernels_pod.cu): the co-run split as ONE launch on the full-device
    // stream — prefill-attention CTAs and S_d decode-attention CTAs in one grid, no fork / join.  Opt-in
    // (DUET_POD=1): measured 1-2 % slower per cfg2 step than the two launches on the green-context pair
    // (profiles/r02_pod_ab.txt), which stay the default
    static const bool pod_env = getenv("DUET_POD") && atoi(getenv("DUET_POD")) != 0;
    bool pod_done = false;
    if (cp && pod_env && dt == DT::BF16 && dh == 128) {
      PrefillAttnArgs pa{};
      DecodeAttnArgs da{};
      prefill_attn(c, S, ap, S.qkv, nqkv, S.o, n_rows, kv->k_pool[l], kv->v_pool[l], kv->n_pages, num_sms, st, &pa);
      decode_attn(c, S, ap, (const char*)S.qkv + (size_t)ap.n_pre * nqkv * es, nqkv,
                  (char*)S.o + (size_t)ap.n_pre * hq * dh * es, kv->k_pool[l], kv->v_pool[l], kv->n_pages, num_sms, st,
                  nullptr, &da);
      if (fa_tc_supported(pa) && decode_tc_supported(da)) {
        const int pi = prof_begin(c, st, DUET_KCLASS_PREFILL_ATTN);
        const int r = launch_pod_attn(dt, pa, da, cp->s_d, st);
        if (r <= 0) DUET_FAIL(DUET_ERR_UNSUPPORTED, "layer %d: fused prefill + decode attention could not be launched", l);
        prof_end(c, st, pi, DUET_KCLASS_PREFILL_ATTN, ap.attn_flops_pre, ap.attn_bytes_pre);
        nk += r;
        cp = nullptr;
        c->last_pod = true;
        pod_done = true;
      }
    }
    if (!pod_done) {  // the two attentions as two launches (sequential, or co-run on the green-context pair)
      cudaStream_t st_pa = st, st_da = st;
      int sms_pa = num_sms, sms_da = num_sms;
      if (cp) {
        CUDA_TRY(cudaEventRecord(c->ev_cf, st));
        CUDA_TRY(cudaStreamWaitEvent(cp->s_pre, c->ev_cf, 0));
        CUDA_TRY(cudaStreamWaitEvent(cp->s_dec, c->ev_cf, 0));
        st_pa = cp->s_pre;
        sms_pa = cp->s_p;
        st_da = cp->s_dec;
        sms_da = cp->s_d;
      }
      if (ap.n_pre > 0) {
        const int pi = prof_begin(c, st_pa, DUET_KCLASS_PREFILL_ATTN);
        const int r = prefill_attn(c, S, ap, S.qkv, nqkv, S.o, n_rows, kv->k_pool[l], kv->v_pool[l], kv->n_pages,
                                   sms_pa, st_pa, nullptr, n_dev);  // n_dev: the step's shape in the metadata
        if (r <= 0) DUET_FAIL(DUET_ERR_UNSUPPORTED, "layer %d: prefill attention could not be launched", l);
        prof_end(c, st_pa, pi, DUET_KCLASS_PREFILL_ATTN, ap.attn_flops_pre, ap.attn_bytes_pre);
        if (dbg_sync && !c->capturing) {
          fprintf(stderr, "[duet] layer %d: prefill attention ...", l);
          fprintf(stderr, " %s\n", cudaGetErrorString(cudaStreamSynchronize(st_pa)));
        }
        nk += r;
      }
      if (ap.n_dec > 0) {
        const int pi = prof_begin(c, st_da, DUET_KCLASS_DECODE_ATTN);
        // inside a graph capture the class is timed on the device (no events in graphs)
        unsigned long long* dt_ = c->capturing && c->prof_on && (c->prof_mask & (1 << DUET_KCLASS_DECODE_ATTN))
                                      ? c->dev_timer : nullptr;
        const int r = decode_attn(c, S, ap, (const char*)S.qkv + (size_t)ap.n_pre * nqkv * es, nqkv,
                                  (char*)S.o + (size_t)ap.n_pre * hq * dh * es, kv->k_pool[l], kv->v_pool[l],
                                  kv->n_pages, sms_da, st_da, dt_);
        if (r <= 0) DUET_FAIL(DUET_ERR_UNSUPPORTED, "layer %d: decode attention could not be launched", l);
        prof_end(c, st_da, pi, DUET_KCLASS_DECODE_ATTN, ap.attn_flops_dec, ap.attn_bytes_dec);
        nk += r;
      }
      if (cp) {
        CUDA_TRY(cudaEventRecord(c->ev_ca, cp->s_pre));
        CUDA_TRY(cudaEventRecord(c->ev_cb, cp->s_dec));
        CUDA_TRY(cudaStreamWaitEvent(st, c->ev_ca, 0));
        CUDA_TRY(cudaStreamWaitEvent(st, c->ev_cb, 0));
      }
    }
    // 5. x1 = x + o W_o^T
    // TP: the O projection of this rank's heads is a partial sum; rank 0 adds the
    // residual and the partials are all-reduced over the side's communicator
    GemmArgs go{S.o, W.w_o, S.x1, lead ? X : nullptr, nullptr, n_rows, d, hq * dh, hq * dh, hq * dh, d, d,
                lead ? EPI_RESIDUAL : EPI_STORE};
    with_ws(go);
    go.m_dev = n_dev;
    if (l == 0 && row_split < n_rows) {
      go.R2 = x_in2;
      go.row_split = row_split;
      go.C2 = (char*)S.x1 + (size_t)row_split * d * es;  // output stays in one buffer
    }
    const void* x1 = S.x1;
    bool fused_o = false;
    if (ar_side && !n_dev && !(l == 0 && row_split < n_rows)) {  // f3: O projection + allreduce in one kernel
      GemmArgs ga{S.o, W.w_o, nullptr, X, nullptr, n_rows, d, hq * dh, hq * dh, hq * dh, d, d, EPI_RESIDUAL_AR};
      ga.ar = &ar_o;
      if (gemm2_supported(ga, num_sms)) {
        go = ga;
        fused_o = true;
        x1 = ar_out0;
      }
    }
    TIMED(DUET_KCLASS_GEMM, gemm_fl(d, hq * dh), gemm_by(d, hq * dh, d, true), launch_gemm(dt, go, num_sms, st));
    if (comm && !fused_o) TIMED(DUET_KCLASS_OTHER, 0.0, 2.0 * n * d * e, allreduce(S.x1, n_rows));
    // 6. h2 = RMSNorm(x1) g2
    TIMED(DUET_KCLASS_OTHER, 4.0 * n * d, 2.0 * n * d * e,
          launch_rmsnorm(dt, x1, W.g_norm2, S.h2, n_rows, d, eps, st, nullptr, 1 << 30, n_dev));
    // 7. act = silu(h2 W_g^T) * (h2 W_u^T)
    GemmArgs gg{S.h2, W.w_gate_up, S.act, nullptr, nullptr, n_rows, m, d, d, d, m, 0, EPI_SWIGLU};
    with_ws(gg);
    gg.m_dev = n_dev;
    TIMED(DUET_KCLASS_GEMM, gemm_fl(2.0 * m, d), gemm_by(2.0 * m, d, m, false), launch_gemm(dt, gg, num_sms, st));
    // 8. y = x1 + act W_d^T
    GemmArgs gd{S.act, W.w_down, Y, lead ? x1 : nullptr, nullptr, n_rows, d, m, m, m, d, d,
                lead ? EPI_RESIDUAL : EPI_STORE};
    with_ws(gd);
    gd.m_dev = n_dev;
    if (l == sp.n_layers - 1 && row_split < n_rows) {
      gd.C2 = y_final2;
      gd.R2 = lead ? (const char*)x1 + (size_t)row_split * d * es : nullptr;
      gd.row_split = row_split;
    }
    bool fused_d = false;
    if (ar_side && !n_dev && !(l == sp.n_layers - 1 && row_split < n_rows)) {  // f3: down projection + allreduce
      GemmArgs ga{S.act, W.w_down, nullptr, x1, nullptr, n_rows, d, m, m, m, d, d, EPI_RESIDUAL_AR};
      ga.ar = &ar_d;
      if (gemm2_supported(ga, num_sms)) {
        gd = ga;
        fused_d = true;
      }
    }
    TIMED(DUET_KCLASS_GEMM, gemm_fl(d, m), gemm_by(d, m, d, true), launch_gemm(dt, gd, num_sms, st));
    x_carry = fused_d ? (const void*)ar_out1 : (const void*)Y;
    if (fused_d && l == sp.n_layers - 1)  // the caller's output buffer is not peer-mapped
      TIMED(DUET_KCLASS_OTHER, 0.0, 2.0 * n * d * e, launch_copy_bytes(Y, ar_out1, (size_t)n_rows * d * es, num_sms, st));
    if (comm && !fused_d) {
      // rows >= row_split of the last layer's output went to y_final2 (the temporal batch's decode
      // rows in the caller's decode buffer): each buffer is reduced over its own rows
      const bool split_out = l == sp.n_layers - 1 && row_split < n_rows;
      TIMED(DUET_KCLASS_OTHER, 0.0, 2.0 * n * d * e, allreduce(Y, split_out ? row_split : n_rows));
      if (split_out) TIMED(DUET_KCLASS_OTHER, 0.0, 0.0, allreduce(y_final2, n_rows - row_split));
    }
  }
#undef TIMED
  DUET_TRY(check_launch("layer stack"));
  *kernels += nk;
  return DUET_OK;
}

// Pinned staging slot (ring of kStageSlots; waits only if the host runs kStageSlots steps ahead).
// Side metadata <- staging slot, on stream st ahead of the step's kernels.  Default: the slot is
// uploaded right away on s_up (an early copy-engine H2D into a device ring, off the step's critical
// path) and copied device-to-device on st; DUET_META=0: st reads the mapped slot zero-copy.
static duet_status upload_meta(duet_ctx* c, Side& S, const int* img, int slot, size_t n_int, int num_sms,
                               cudaStream_t st, int* kernels) {
  static const bool prefetch = !getenv("DUET_META") || atoi(getenv("DUET_META")) != 0;
  const size_t bytes = n_int * sizeof(int);
  if (prefetch) {
    int* ring = c->stage_d + (size_t)slot * c->stage_ints;
    CUDA_TRY(cudaStreamWaitEvent(c->s_up, c->use_ev[slot], 0));  // the slot's previous reader is done
    CUDA_TRY(cudaMemcpyAsync(ring, img, bytes, cudaMemcpyHostToDevice, c->s_up));
    CUDA_TRY(cudaEventRecord(c->up_ev[slot], c->s_up));
    CUDA_TRY(cudaEventRecord(c->stage_ev[slot], c->s_up));  // host slot reusable once uploaded
    CUDA_TRY(cudaStreamWaitEvent(st, c->up_ev[slot], 0));
    *kernels += launch_copy_bytes(S.meta, ring, bytes, num_sms, st);
    CUDA_TRY(cudaEventRecord(c->use_ev[slot], st));
  } else {
    *kernels += launch_copy_bytes(S.meta, c->stage_dev + (img - c->stage), bytes, num_sms, st);
    CUDA_TRY(cudaEventRecord(c->stage_ev[slot], st));
  }
  return DUET_OK;
}

static duet_status stage_slot(duet_ctx* c, int** out, int* slot) {
  const int s = c->stage_next;
  c->stage_next = (s + 1) % kStageSlots;
  CUDA_TRY(cudaEventSynchronize(c->stage_ev[s]));
  *out = c->stage + (size_t)s * c->stage_ints;
  *slot = s;
  return DUET_OK;
}

// ---------------------------------------------------------------------------------- C ABI

extern "C" duet_status duet_ctx_create(int32_t device, const duet_model_spec* spec, const duet_ctx_limits* lim,
                                       duet_ctx** out) {
  clear_error();
  if (!spec || !lim || !out) DUET_FAIL(DUET_ERR_INVALID_ARG, "spec/limits/out is NULL");
  *out = nullptr;
  if (spec->n_layers <= 0 || spec->d_model <= 0 || spec->n_q_heads <= 0 || spec->n_kv_heads <= 0 ||
      spec->ffn_dim <= 0 || spec->head_dim <= 0 || spec->n_q_heads % spec->n_kv_heads ||
      spec->d_model != spec->n_q_heads * spec->head_dim)
    DUET_FAIL(DUET_ERR_CONFIG, "model spec is inconsistent (d_model = n_q_heads * head_dim, h_q %% h_kv == 0)");
  if (spec->head_dim != 64 && spec->head_dim != 128)
    DUET_FAIL(DUET_ERR_UNSUPPORTED, "head_dim = %d (kernels implement 64 and 128)", spec->head_dim);
  const int G = spec->n_q_heads / spec->n_kv_heads;
  if (G != 1 && G != 2 && G != 4 && G != 5 && G != 8)
    DUET_FAIL(DUET_ERR_UNSUPPORTED, "GQA group %d (kernels implement 1, 2, 4, 5, 8)", G);
  if (spec->d_model % 16 || spec->ffn_dim % 16)
    DUET_FAIL(DUET_ERR_UNSUPPORTED, "d_model and ffn_dim must be multiples of 16");
  const int tp = spec->tp < 1 ? 1 : spec->tp;
  if (spec->n_q_heads % tp || spec->n_kv_heads % tp || spec->ffn_dim % tp || (spec->ffn_dim / tp) % 16)
    DUET_FAIL(DUET_ERR_CONFIG, "tp = %d must divide h_q = %d, h_kv = %d and ffn_dim = %d (ffn_dim/tp %% 16 == 0)", tp,
              spec->n_q_heads, spec->n_kv_heads, spec->ffn_dim);
  if (lim->dtype != DUET_DTYPE_BF16 && lim->dtype != DUET_DTYPE_FP32)
    DUET_FAIL(DUET_ERR_INVALID_ARG, "dtype = %d", lim->dtype);
  if (lim->max_prefill_tokens < 0 || lim->max_decode_reqs < 0 || lim->max_k < 1 || lim->max_pages_per_seq < 1 ||
      lim->max_pos < 1 || lim->max_prefill_seqs < 0)
    DUET_FAIL(DUET_ERR_INVALID_ARG, "limits out of range");
  duet_ctx* c = new duet_ctx();
  c->device = device;
  c->gspec = *spec;
  c->spec = *spec;  // the shard this rank computes (head-sharded TP, reading #13)
  c->spec.n_q_heads /= tp;
  c->spec.n_kv_heads /= tp;
  c->spec.ffn_dim /= tp;
  c->spec.tp = tp;
  c->lim = *lim;
  c->dt = lim->dtype == DUET_DTYPE_BF16 ? DT::BF16 : DT::F32;
  auto fail = [&](duet_status s) {
    duet_ctx_destroy(c);
    return s;
  };
  if (cudaSetDevice(device) != cudaSuccess) {
    set_error("cudaSetDevice(%d) failed", device);
    return fail(DUET_ERR_CUDA);
  }
  cudaFree(nullptr);
  cudaDeviceGetAttribute(&c->total_sms, cudaDevAttrMultiProcessorCount, device);
  duet_status st;
#define STEP(expr)               \
  do {                           \
    st = (expr);                 \
    if (st != DUET_OK) return fail(st); \
  } while (0)
  auto init_cu = [&]() -> duet_status {
    DUET_TRY(load_driver());
    CU_TRY(DRV.Init(0));
    CU_TRY(DRV.DeviceGet(&c->cudev, device));
    CU_TRY(DRV.DeviceGetDevResource(c->cudev, &c->sm_all, CU_DEV_RESOURCE_TYPE_SM));
    // achievable decode sizes: simulate splits for every request count
    const unsigned flags = (lim->flags & DUET_CTX_FINE_SPLIT) ? CU_DEV_SM_RESOURCE_SPLIT_IGNORE_SM_COSCHEDULING : 0;
    std::vector<int> seen;
    for (int want = 1; want < c->total_sms; ++want) {
      CUdevResource grp[1], rem;
      unsigned n = 1;
      if (DRV.DevSmResourceSplitByCount(grp, &n, &c->sm_all, &rem, flags, (unsigned)want) != CUDA_SUCCESS) continue;
      if (n != 1) continue;
      const int got = (int)grp[0].sm.smCount;
      if (got >= c->total_sms || rem.sm.smCount == 0) continue;
      if (std::find(seen.begin(), seen.end(), got) == seen.end()) seen.push_back(got);
    }
    std::sort(seen.begin(), seen.end());
    for (int s : seen) {
      Partition p;
      p.s_d = s;
      c->parts.push_back(p);
    }
    CUDA_TRY(cudaStreamCreateWithFlags(&c->s_full, cudaStreamNonBlocking));
    cudaEvent_t* evs[] = {&c->ev_in, &c->ev_dec0, &c->ev_dec1, &c->ev_pre0, &c->ev_pre1};
    for (auto e : evs) CUDA_TRY(cudaEventCreate(e));
    cudaEvent_t* evc[] = {&c->ev_cf, &c->ev_ca, &c->ev_cb};
    for (auto e : evc) CUDA_TRY(cudaEventCreateWithFlags(e, cudaEventDisableTiming));
    CUDA_TRY(cudaStreamCreateWithFlags(&c->s_up, cudaStreamNonBlocking));
    for (int i = 0; i < kStageSlots; ++i) {
      CUDA_TRY(cudaEventCreateWithFlags(&c->stage_ev[i], cudaEventDisableTiming));
      CUDA_TRY(cudaEventRecord(c->stage_ev[i], c->s_full));
      CUDA_TRY(cudaEventCreateWithFlags(&c->up_ev[i], cudaEventDisableTiming));
      CUDA_TRY(cudaEventCreateWithFlags(&c->use_ev[i], cudaEventDisableTiming));
      CUDA_TRY(cudaEventRecord(c->use_ev[i], c->s_full));
    }
    // RoPE table (reading #5): theta_i = theta^(-2i/d_h), phi = p theta_i, computed in double
    const int half = spec->head_dim / 2;
    std::vector<float2> tab((size_t)lim->max_pos * half);
    for (int p = 0; p < lim->max_pos; ++p)
      for (int i = 0; i < half; ++i) {
        const double inv = std::pow(spec->rope_theta, -2.0 * i / spec->head_dim);
        const double phi = (double)p * inv;
        tab[(size_t)p * half + i] = make_float2((float)std::cos(phi), (float)std::sin(phi));
      }
    // co-run rates: the round-1 prior until duet_calibrate measures them
    c->cal_fa.assign(c->total_sms + 1, 0.0);
    c->cal_bw.assign(c->total_sms + 1, 0.0);
    for (int s = 1; s <= c->total_sms; ++s) {
      c->cal_fa[s] = 4.0e12 * s;
      c->cal_bw[s] = s == c->total_sms ? 6.1e12 : 5.9e12 * (1.0 - std::exp(-s / 28.0));
    }
    CUDA_TRY(cudaMalloc(&c->tok_ts, kTokTsSlots * sizeof(unsigned long long)));
    CUDA_TRY(cudaMalloc(&c->tok_cnt, sizeof(int)));
    CUDA_TRY(cudaMemset(c->tok_cnt, 0, sizeof(int)));
    CUDA_TRY(cudaMalloc(&c->rope, tab.size() * sizeof(float2)));
    CUDA_TRY(cudaMemcpy(c->rope, tab.data(), tab.size() * sizeof(float2), cudaMemcpyHostToDevice));
    return DUET_OK;
  };
  STEP(init_cu());
  const int nd = lim->max_decode_reqs, np = lim->max_prefill_tokens, ns = lim->max_prefill_seqs;
  STEP(side_alloc(c, c->dec, nd, 0, nd, nd));
  STEP(side_alloc(c, c->pre, np + nd, ns, ns + nd, nd));
  // pinned staging ring: large enough for the bigger side's metadata
  c->stage_ints = (std::max(c->dec.n_meta, c->pre.n_meta) * 2 + 3) / 4 * 4;  // 16-B aligned slots
  if (cudaHostAlloc(&c->stage, kStageSlots * c->stage_ints * sizeof(int), cudaHostAllocMapped) != cudaSuccess ||
      cudaHostGetDevicePointer(&c->stage_dev, c->stage, 0) != cudaSuccess ||
      cudaMalloc(&c->stage_d, kStageSlots * c->stage_ints * sizeof(int)) != cudaSuccess) {
    set_error("cudaHostAlloc of the staging ring failed");
    return fail(DUET_ERR_CUDA);
  }
  // decode rows use identity page-table rows (row r of the decode table)
  {
    std::vector<int> ident(std::max(nd, 1));
    for (int i = 0; i < nd; ++i) ident[i] = i;
    if (nd > 0 && cudaMemcpy(c->dec.tok(), ident.data(), nd * sizeof(int), cudaMemcpyHostToDevice) != cudaSuccess) {
      set_error("metadata init failed");
      return fail(DUET_ERR_CUDA);
    }
  }
  if (cudaDeviceSynchronize() != cudaSuccess) {
    set_error("ctx init failed: %s", cudaGetErrorString(cudaGetLastError()));
    return fail(DUET_ERR_CUDA);
  }
#undef STEP
  *out = c;
  return DUET_OK;
}

extern "C" duet_status duet_ctx_destroy(duet_ctx* c) {
  if (!c) return DUET_OK;
  cudaSetDevice(c->device);
  if (c->comm_dec) NCCL.CommDestroy(c->comm_dec);
  if (c->comm_pre) NCCL.CommDestroy(c->comm_pre);
  cudaDeviceSynchronize();
  for (auto& kv : c->graphs)
    if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
  for (auto& kv : c->pre_graphs)
    if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
  for (auto& p : c->parts) {
    if (!p.created) continue;
    DRV.StreamDestroy((CUstream)p.s_dec);
    DRV.StreamDestroy((CUstream)p.s_pre);
    DRV.GreenCtxDestroy(p.g_dec);
    DRV.GreenCtxDestroy(p.g_pre);
  }
  side_free(c->dec);
  side_free(c->pre);
  if (c->rope) cudaFree(c->rope);
  for (int r = 0; r < kMaxTp; ++r)
    if (c->ar_peer[r] && c->ar_peer[r] != c->ar_arena) cudaIpcCloseMemHandle(c->ar_peer[r]);
  if (c->ar_arena) cudaFree(c->ar_arena);
  if (c->emu_slots) cudaFree(c->emu_slots);
  if (c->emu_cnt) cudaFree(c->emu_cnt);
  if (c->tok_ts) cudaFree(c->tok_ts);
  if (c->tok_cnt) cudaFree(c->tok_cnt);
  if (c->dev_timer) cudaFree(c->dev_timer);
  if (c->stage) cudaFreeHost(c->stage);
  if (c->stage_d) cudaFree(c->stage_d);
  if (c->s_up) cudaStreamDestroy(c->s_up);
  for (int i = 0; i < kStageSlots; ++i) {
    if (c->up_ev[i]) cudaEventDestroy(c->up_ev[i]);
    if (c->use_ev[i]) cudaEventDestroy(c->use_ev[i]);
  }
  cudaEvent_t evs[] = {c->ev_in, c->ev_dec0, c->ev_dec1, c->ev_pre0, c->ev_pre1, c->ev_cf, c->ev_ca, c->ev_cb};
  for (auto e : evs)
    if (e) cudaEventDestroy(e);
  for (auto e : c->stage_ev)
    if (e) cudaEventDestroy(e);
  for (auto& pr : c->prof_pool) {
    cudaEventDestroy(pr.first);
    cudaEventDestroy(pr.second);
  }
  if (c->s_full) cudaStreamDestroy(c->s_full);
  delete c;
  return DUET_OK;
}

extern "C" duet_status duet_ctx_partitions(duet_ctx* c, int32_t* sd, int32_t* n, int32_t* total) {
  clear_error();
  if (!c || !n) DUET_FAIL(DUET_ERR_INVALID_ARG, "ctx/n is NULL");
  const int cnt = (int)c->parts.size();
  if (sd) {
    if (*n < cnt) DUET_FAIL(DUET_ERR_CAPACITY, "sd_sms capacity %d < %d partitions", *n, cnt);
    for (int i = 0; i < cnt; ++i) sd[i] = c->parts[i].s_d;
  }
  *n = cnt;
  if (total) *total = c->total_sms;
  return DUET_OK;
}

// ---------------------------------------------------------------------------------- validation

static duet_status check_pages(duet_ctx* c, const int32_t* table, int32_t max_pages, int row, int n_tokens,
                               int n_pages, const char* side) {
  const int need = (n_tokens + kPageSize - 1) / kPageSize;
  if (need > max_pages)
    DUET_FAIL(DUET_ERR_OUT_OF_RANGE, "%s request %d needs %d pages > max_pages %d", side, row, need, max_pages);
  if (need > c->lim.max_pages_per_seq)
    DUET_FAIL(DUET_ERR_CAPACITY, "%s request %d needs %d pages > ctx max_pages_per_seq %d", side, row, need,
              c->lim.max_pages_per_seq);
  for (int j = 0; j < need; ++j) {
    const int pg = table[(size_t)row * max_pages + j];
    if (pg < 0 || pg >= n_pages)
      DUET_FAIL(DUET_ERR_OUT_OF_RANGE, "%s request %d page %d = %d outside [0, %d)", side, row, j, pg, n_pages);
    if (c->page_mark[pg] == c->page_gen)
      DUET_FAIL(DUET_ERR_OUT_OF_RANGE, "%s request %d page %d = %d is used twice", side, row, j, pg);
    c->page_mark[pg] = c->page_gen;
  }
  return DUET_OK;
}

// a new generation of page marks: every page may be claimed once until the next call
static void begin_page_check(duet_ctx* c, int n_pages) {
  if ((int)c->page_mark.size() < n_pages) c->page_mark.assign(n_pages, 0);
  if (++c->page_gen == 0) {
    std::fill(c->page_mark.begin(), c->page_mark.end(), 0);
    c->page_gen = 1;
  }
}

static duet_status validate_step(duet_ctx* c, const duet_layer_weights* w, const duet_prefill* pre,
                                 const duet_decode* dec, const duet_kv_pages* kv, int k) {
  if (!w) DUET_FAIL(DUET_ERR_INVALID_ARG, "weights are NULL");
  for (int l = 0; l < c->spec.n_layers; ++l) {
    const auto& W = w[l];
    if (!W.w_qkv || !W.w_o || !W.w_gate_up || !W.w_down || !W.g_norm1 || !W.g_norm2)
      DUET_FAIL(DUET_ERR_INVALID_ARG, "layer %d: a weight pointer is NULL", l);
    if (c->spec.qkv_bias && !W.b_qkv) DUET_FAIL(DUET_ERR_INVALID_ARG, "layer %d: qkv_bias set but b_qkv NULL", l);
  }
  if (!kv || !kv->k_pool || !kv->v_pool) DUET_FAIL(DUET_ERR_INVALID_ARG, "kv pools are NULL");
  if (kv->page_size != kPageSize) DUET_FAIL(DUET_ERR_UNSUPPORTED, "page_size = %d (must be 16)", kv->page_size);
  for (int l = 0; l < c->spec.n_layers; ++l)
    if (!kv->k_pool[l] || !kv->v_pool[l]) DUET_FAIL(DUET_ERR_INVALID_ARG, "layer %d: kv pool NULL", l);
  if (kv->n_pages <= 0) DUET_FAIL(DUET_ERR_INVALID_ARG, "n_pages = %d", kv->n_pages);
  begin_page_check(c, kv->n_pages);
  if (pre && pre->n_seqs > 0) {
    if (pre->n_seqs > c->lim.max_prefill_seqs)
      DUET_FAIL(DUET_ERR_CAPACITY, "n_seqs = %d > max_prefill_seqs %d", pre->n_seqs, c->lim.max_prefill_seqs);
    if (!pre->q || !pre->c || !pre->page_table || !pre->x || !pre->y)
      DUET_FAIL(DUET_ERR_INVALID_ARG, "prefill: a pointer is NULL");
    long tot = 0;
    for (int s = 0; s < pre->n_seqs; ++s) {
      if (pre->q[s] < 1 || pre->c[s] < 0)
        DUET_FAIL(DUET_ERR_OUT_OF_RANGE, "prefill seq %d: q = %d, c = %d", s, pre->q[s], pre->c[s]);
      if ((long)pre->c[s] + pre->q[s] > c->lim.max_pos)
        DUET_FAIL(DUET_ERR_CAPACITY, "prefill seq %d: c + q = %ld > max_pos %d", s, (long)pre->c[s] + pre->q[s],
                  c->lim.max_pos);
      tot += pre->q[s];
      DUET_TRY(check_pages(c, pre->page_table, pre->max_pages, s, pre->c[s] + pre->q[s], kv->n_pages, "prefill"));
    }
    if (tot > c->lim.max_prefill_tokens)
      DUET_FAIL(DUET_ERR_CAPACITY, "prefill tokens %ld > max_prefill_tokens %d", tot, c->lim.max_prefill_tokens);
  }
  if (dec && dec->n_reqs > 0) {
    if (dec->n_reqs > c->lim.max_decode_reqs)
      DUET_FAIL(DUET_ERR_CAPACITY, "n_reqs = %d > max_decode_reqs %d", dec->n_reqs, c->lim.max_decode_reqs);
    if (!dec->c || !dec->page_table || !dec->x || !dec->y) DUET_FAIL(DUET_ERR_INVALID_ARG, "decode: a pointer is NULL");
    if (dec->head) {
      if (!dec->head->g_norm || !dec->head->w_head || !dec->head->embed || !dec->head->tokens)
        DUET_FAIL(DUET_ERR_INVALID_ARG, "decode: an LM-head pointer is NULL");
      if (c->dt != DT::BF16 || c->spec.vocab <= 0 || c->spec.vocab % 8 || !c->dec.logits)
        DUET_FAIL(DUET_ERR_UNSUPPORTED, "the LM head needs a bf16 context with vocab %% 8 == 0 (vocab = %d)",
                  c->spec.vocab);
    }
    if (k > c->lim.max_k) DUET_FAIL(DUET_ERR_CAPACITY, "k = %d > max_k %d", k, c->lim.max_k);
    for (int r = 0; r < dec->n_reqs; ++r) {
      if (dec->c[r] < 1) DUET_FAIL(DUET_ERR_OUT_OF_RANGE, "decode request %d: c = %d must be >= 1", r, dec->c[r]);
      if ((long)dec->c[r] + k > c->lim.max_pos)
        DUET_FAIL(DUET_ERR_CAPACITY, "decode request %d: c + k > max_pos %d", r, c->lim.max_pos);
      DUET_TRY(check_pages(c, dec->page_table, dec->max_pages, r, dec->c[r] + k, kv->n_pages, "decode"));
    }
  }
  return DUET_OK;
}

// ---------------------------------------------------------------------------------- metadata

// Fill a side's metadata image (host) for prefill rows followed by decode rows.
// Returns the number of ints to copy (prefix of the image up to the end of the used table rows).
static size_t build_meta(duet_ctx* c, const Side& S, int* img, const duet_prefill* pre, const duet_decode* dec,
                         AttnPlan* ap) {
  int n_pre = 0, n_seqs = 0;
  int max_q = 0, max_len_pre = 0;
  if (pre && pre->n_seqs > 0) {
    n_seqs = pre->n_seqs;
    for (int s = 0; s < n_seqs; ++s) {
      const int q = pre->q[s], cc = pre->c[s];
      img[S.o_row0 + s] = n_pre;
      img[S.o_qlen + s] = q;
      img[S.o_cpre + s] = cc;
      img[S.o_seqrow + s] = s;
      for (int i = 0; i < q; ++i) {
        img[S.o_pos + n_pre + i] = cc + i;
        img[S.o_tok + n_pre + i] = s;
      }
      for (int j = 0; j < S.pitch; ++j)
        img[S.o_table + (size_t)s * S.pitch + j] = j < pre->max_pages ? pre->page_table[(size_t)s * pre->max_pages + j] : 0;
      n_pre += q;
      max_q = std::max(max_q, q);
      max_len_pre = std::max(max_len_pre, cc + q);
    }
  }
  int n_dec = 0, max_len_dec = 0;
  if (dec && dec->n_reqs > 0) {
    n_dec = dec->n_reqs;
    for (int r = 0; r < n_dec; ++r) {
      img[S.o_pos + n_pre + r] = dec->c[r];
      img[S.o_tok + n_pre + r] = n_seqs + r;
      for (int j = 0; j < S.pitch; ++j)
        img[S.o_table + (size_t)(n_seqs + r) * S.pitch + j] =
            j < dec->max_pages ? dec->page_table[(size_t)r * dec->max_pages + j] : 0;
      max_len_dec = std::max(max_len_dec, dec->c[r] + 1);
    }
    // the decode attention's CTAs take the requests longest context first (a stable sort): the last
    // wave holds the shortest requests, not the longest (the cfg3 ramp put them last)
    std::vector<int> ord(n_dec);
    for (int r = 0; r < n_dec; ++r) ord[r] = r;
    std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) { return dec->c[a] > dec->c[b]; });
    for (int r = 0; r < n_dec; ++r) img[S.o_order + r] = ord[r];
  }
  img[S.o_step] = 0;
  img[S.o_step + 1] = n_pre + n_dec;  // the side's rows, sequences and longest chunk, read on the device by
  img[S.o_step + 2] = n_seqs;         // shape-agnostic prefill graphs (f4)
  img[S.o_step + 3] = max_q;
  for (int s = n_seqs; s < S.cap_seqs; ++s) img[S.o_qlen + s] = 0;  // no work items past the batch
  {
    const double hq = c->spec.n_q_heads, hkv = c->spec.n_kv_heads, dh = c->spec.head_dim, e = (double)dt_size(c->dt);
    double fl = 0, by = 0;
    if (pre)
      for (int s = 0; s < n_seqs; ++s) {
        const double q = pre->q[s], cc = pre->c[s];
        fl += 4.0 * hq * dh * (q * cc + q * (q + 1) / 2);
        by += 2.0 * q * hq * dh * e + 2.0 * hkv * dh * (cc + q) * e;
      }
    ap->attn_flops_pre = fl;
    ap->attn_bytes_pre = by;
    fl = by = 0;
    if (dec)
      for (int r = 0; r < n_dec; ++r) {
        fl += 4.0 * hq * dh * (dec->c[r] + 1.0);
        by += 2.0 * hq * dh * e + 2.0 * hkv * dh * (dec->c[r] + 1.0) * e;
      }
    ap->attn_flops_dec = fl;
    ap->attn_bytes_dec = by;
  }
  ap->n_pre = n_pre;
  ap->n_seqs = n_seqs;
  ap->max_q = max_q;
  ap->max_len_pre = max_len_pre;
  ap->n_dec = n_dec;
  ap->max_len_dec = max_len_dec;
  return S.o_table + (size_t)(n_seqs + n_dec) * S.pitch;
}

static uint64_t hash_ptrs(const duet_layer_weights* w, int L, const duet_kv_pages* kv, const void* y, int maxlen_bucket,
                          const duet_lm_head* head = nullptr) {
  uint64_t h = 1469598103934665603ull;
  auto mix = [&](const void* p) {
    h ^= (uint64_t)(uintptr_t)p;
    h *= 1099511628211ull;
  };
  for (int l = 0; l < L; ++l) {
    mix(w[l].w_qkv); mix(w[l].b_qkv); mix(w[l].w_o); mix(w[l].w_gate_up); mix(w[l].w_down);
    mix(w[l].g_norm1); mix(w[l].g_norm2); mix(kv->k_pool[l]); mix(kv->v_pool[l]);
  }
  mix(y);
  if (head) {
    mix(head->g_norm); mix(head->w_head); mix(head->embed); mix(head->tokens);
  }
  h ^= (uint64_t)maxlen_bucket * 0x9E3779B97F4A7C15ull;
  return h;
}

// LM head over n rows y (f1, P:250 t_cls): RMSNorm with the final gain, logits = h w_head^T (the
// weight-streaming GEMM), greedy token + embedding of the next input (x_next may be NULL).
static duet_status lm_head(duet_ctx* c, Side& S, cudaStream_t st, int num_sms, int n, const void* y,
                           const duet_lm_head* head, void* x_next, const int* step, int* kernels) {
  const int d = c->spec.d_model, V = c->spec.vocab;
  const size_t e = dt_size(c->dt);
  int nk = 0, r = 0;
  int pi = prof_begin(c, st, DUET_KCLASS_OTHER);
  if ((r = launch_rmsnorm(c->dt, y, head->g_norm, S.h, n, d, (float)c->spec.norm_eps, st)) <= 0)
    DUET_FAIL(DUET_ERR_CUDA, "LM head: final RMSNorm could not be launched");
  nk += r;
  prof_end(c, st, pi, DUET_KCLASS_OTHER, 4.0 * n * d, 2.0 * n * d * e);
  GemmArgs g{S.h, head->w_head, S.logits, nullptr, nullptr, n, V, d, d, d, V, 0, EPI_STORE};
  g.ws = S.gemm_ws;
  g.ws_floats = S.gemm_ws_floats;
  pi = prof_begin(c, st, DUET_KCLASS_GEMM);
  if ((r = launch_gemm(c->dt, g, num_sms, st)) <= 0) DUET_FAIL(DUET_ERR_CUDA, "LM head: GEMM could not be launched");
  nk += r;
  prof_end(c, st, pi, DUET_KCLASS_GEMM, 2.0 * n * (double)V * d, ((double)n * d + (double)V * d + (double)n * V) * e);
  pi = prof_begin(c, st, DUET_KCLASS_OTHER);
  if ((r = launch_argmax_embed(S.logits, V, head->embed, x_next, d, head->tokens, step, n, st)) <= 0)
    DUET_FAIL(DUET_ERR_CUDA, "LM head: argmax / embedding could not be launched");
  nk += r;
  prof_end(c, st, pi, DUET_KCLASS_OTHER, 0.0, ((double)n * V + (x_next ? 2.0 * n * d : 0.0)) * e);
  DUET_TRY(check_launch("lm head"));
  *kernels += nk;
  return DUET_OK;
}

// One decode step on the decode side (all layers + advance), launched on st.
static duet_status decode_step_kernels(duet_ctx* c, cudaStream_t st, int num_sms, const duet_layer_weights* w,
                                       const duet_kv_pages* kv, const AttnPlan& meta, int max_len, void* y_out,
                                       const duet_lm_head* head, int* kernels) {
  Side& S = c->dec;
  const int n = meta.n_dec;
  AttnPlan ap = meta;  // work counts of step 1 (timing statistics only)
  ap.max_len_dec = max_len;
  DUET_TRY(run_layers(c, S, st, num_sms, n, S.xin, S.ylast, w, kv, ap, kernels));
  // with an LM head the next input is the greedy token's embedding (f1), else the output (reading #26)
  if (head) DUET_TRY(lm_head(c, S, st, num_sms, n, S.ylast, head, S.xin, S.step(), kernels));
  *kernels += launch_decode_advance(c->dt, S.ylast, head ? nullptr : S.xin, y_out, n, c->spec.d_model, S.pos(),
                                    S.step(), st, c->tok_ts, c->tok_cnt);
  DUET_TRY(check_launch("decode advance"));
  return DUET_OK;
}

// ---------------------------------------------------------------------------------- step

extern "C" duet_status duet_step(duet_ctx* c, const duet_layer_weights* w, const duet_prefill* pre,
                                 const duet_decode* dec, const duet_kv_pages* kv, const duet_split* split,
                                 void* stream) {
  clear_error();
  if (!c || !split) DUET_FAIL(DUET_ERR_INVALID_ARG, "ctx/split is NULL");
  if (split->mode != DUET_MODE_TEMPORAL && split->mode != DUET_MODE_SPATIAL)
    DUET_FAIL(DUET_ERR_INVALID_ARG, "split mode = %d", split->mode);
  const bool spatial = split->mode == DUET_MODE_SPATIAL;
  const int k = spatial ? split->k : 1;
  if (k < 1) DUET_FAIL(DUET_ERR_OUT_OF_RANGE, "k = %d must be >= 1", k);
  DUET_TRY(validate_step(c, w, pre, dec, kv, k));
  if (c->comm_dec || c->comm_pre) DUET_TRY(comms_healthy(c));
  cudaStream_t ust = (cudaStream_t)stream;
  const bool has_pre = pre && pre->n_seqs > 0;
  const bool has_dec = dec && dec->n_reqs > 0;
  const size_t es = dt_size(c->dt);
  const int d = c->spec.d_model;
  int kernels = 0;
  CUDA_TRY(cudaSetDevice(c->device));
  c->last_has_dec = has_dec;
  c->last_has_pre = has_pre;
  c->last_mode = split->mode;
  c->last_k = k;
  c->last_pre_graph = false;

  if (!spatial) {
    // ---------------- temporal (aggregated) mode: one full-device stream, k = 1
    int* img;
    int slot;
    DUET_TRY(stage_slot(c, &img, &slot));
    AttnPlan ap;
    const size_t n_int = build_meta(c, c->pre, img, pre, dec, &ap);
    const int n_rows = ap.n_pre + ap.n_dec;
    cudaStream_t st = c->s_full;
    CUDA_TRY(cudaEventRecord(c->ev_in, ust));
    CUDA_TRY(cudaStreamWaitEvent(st, c->ev_in, 0));
    CUDA_TRY(cudaEventRecord(c->ev_pre0, st));
    DUET_TRY(upload_meta(c, c->pre, img, slot, n_int, c->total_sms, st, &kernels));
    // [prefill ; decode] rows straight from / into the caller's buffers when the CTA-pair GEMM runs
    // the O and down projections (it reads the residual and writes the output per row range)
    GemmArgs probe{};
    probe.M = n_rows;
    probe.N = d;
    probe.K = d;
    probe.lda = probe.ldb = probe.ldc = probe.ldr = d;
    probe.epi = EPI_RESIDUAL;
    if (has_pre && has_dec) {  // the caller's buffers must meet the kernel's alignment
      probe.R = pre->x;
      probe.C = pre->y;
      probe.R2 = dec->x;
      probe.C2 = dec->y;
    }
    const bool split_io = has_pre && has_dec && c->dt == DT::BF16 && gemm2_supported(probe, c->total_sms) &&
                          c->spec.ffn_dim % 64 == 0 && (c->spec.n_q_heads * c->spec.head_dim) % 64 == 0;
    // f4 co-run: the two attentions of each layer side by side, decode on an S_d group and prefill
    // on the remainder.  DUET_CORUN=<S_d> forces the partition whose decode group has
    // >= S_d SMs, 0 disables; unset, corun_pick's measured-rate model decides per step.
    c->corun = nullptr;
    if (has_pre && has_dec && !(c->lim.flags & DUET_CTX_NO_CORUN)) {
      static const int corun_sd = getenv("DUET_CORUN") ? atoi(getenv("DUET_CORUN")) : -1;
      Partition* cp = nullptr;
      if (corun_sd > 0) {
        for (auto& p : c->parts)
          if (p.s_d >= corun_sd) {
            cp = &p;
            break;
          }
      } else if (corun_sd < 0) {
        cp = corun_pick(c, ap);
      }
      if (cp) {
        DUET_TRY(ensure_partition(c, *cp));
        c->corun = cp;
      }
    }
    c->last_corun = c->corun ? c->corun->s_d : 0;
    c->last_pod = false;
    if (n_rows > 0 && !(has_pre && has_dec)) {  // one phase only: its own buffers, whatever the GEMM path
      DUET_TRY(run_layers(c, c->pre, st, c->total_sms, n_rows, has_pre ? pre->x : dec->x, has_pre ? pre->y : dec->y,
                          w, kv, ap, &kernels));
    } else if (n_rows > 0 && split_io) {
      DUET_TRY(run_layers(c, c->pre, st, c->total_sms, n_rows, pre->x, pre->y, w, kv, ap, &kernels, dec->x, dec->y,
                          ap.n_pre));
    } else if (n_rows > 0) {
      if (has_pre) kernels += launch_copy_bytes(c->pre.xin, pre->x, (size_t)ap.n_pre * d * es, c->total_sms, st);
      if (has_dec)
        kernels += launch_copy_bytes((char*)c->pre.xin + (size_t)ap.n_pre * d * es, dec->x, (size_t)ap.n_dec * d * es,
                                     c->total_sms, st);
      DUET_TRY(run_layers(c, c->pre, st, c->total_sms, n_rows, c->pre.xin, c->pre.ylast, w, kv, ap, &kernels));
      if (has_pre) kernels += launch_copy_bytes(pre->y, c->pre.ylast, (size_t)ap.n_pre * d * es, c->total_sms, st);
      if (has_dec)
        kernels += launch_copy_bytes(dec->y, (char*)c->pre.ylast + (size_t)ap.n_pre * d * es, (size_t)ap.n_dec * d * es,
                                     c->total_sms, st);
    }
    c->corun = nullptr;
    // the decode rows' greedy tokens (f1; k = 1 in temporal mode): from their outputs in dec->y
    if (has_dec && dec->head) DUET_TRY(lm_head(c, c->pre, st, c->total_sms, ap.n_dec, dec->y, dec->head, nullptr,
                                               nullptr, &kernels));
    if (has_dec) kernels += launch_stamp(c->tok_ts, c->tok_cnt, st);  // the decode rows' token time
    CUDA_TRY(cudaEventRecord(c->ev_pre1, st));
    CUDA_TRY(cudaStreamWaitEvent(ust, c->ev_pre1, 0));
    c->last_kernels = kernels;
    return DUET_OK;
  }

  // ---------------- spatial mode (Alg. 1 l.22; §4.3)
  Partition* P = nullptr;
  for (auto& p : c->parts)
    if (p.s_d == split->s_d) P = &p;
  if (!P) DUET_FAIL(DUET_ERR_OUT_OF_RANGE, "s_d = %d is not an achievable partition size", split->s_d);
  DUET_TRY(ensure_partition(c, *P));
  CUDA_TRY(cudaEventRecord(c->ev_in, ust));

  if (has_dec) {
    // decode FIRST: metadata, input copy, then k graph replays with no host sync
    int* img;
    int slot;
    DUET_TRY(stage_slot(c, &img, &slot));
    AttnPlan ap;
    const size_t n_int = build_meta(c, c->dec, img, nullptr, dec, &ap);
    cudaStream_t st = P->s_dec;
    CUDA_TRY(cudaStreamWaitEvent(st, c->ev_in, 0));
    CUDA_TRY(cudaEventRecord(c->ev_dec0, st));
    DUET_TRY(upload_meta(c, c->dec, img, slot, n_int, P->s_d, st, &kernels));
    const int n = ap.n_dec;
    kernels += launch_copy_bytes(c->dec.xin, dec->x, (size_t)n * d * es, P->s_d, st);
    int max_c = 0;
    for (int r = 0; r < n; ++r) max_c = std::max(max_c, dec->c[r]);
    const int max_len = ((max_c + k + 1023) / 1024) * 1024;  // bucket: graphs survive context growth
    // timing a decode-side GEMM / other class needs direct launches (events); the decode attention is
    // timed on the device inside the graph (a direct-launched decode side runs ~13 % slower at cfg3)
    constexpr int kDecClasses = (1 << DUET_KCLASS_GEMM_DECODE) | (1 << DUET_KCLASS_OTHER_DECODE);
    const bool timed_dec = c->prof_on && (c->prof_mask & kDecClasses);
    const bool dev_timed = c->prof_on && (c->prof_mask & (1 << DUET_KCLASS_DECODE_ATTN)) && !timed_dec &&
                           !(c->lim.flags & DUET_CTX_NO_GRAPH);
    if ((c->lim.flags & DUET_CTX_NO_GRAPH) || timed_dec) {
      c->prof_dec_side = true;
      for (int j = 0; j < k; ++j) {
        const duet_status sd = decode_step_kernels(c, st, P->s_d, w, kv, ap, max_len, dec->y, dec->head, &kernels);
        if (sd != DUET_OK) {
          c->prof_dec_side = false;
          return sd;
        }
      }
      c->prof_dec_side = false;
    } else {
      auto key = std::make_tuple(P->s_d, n, c->spec.n_layers + (dev_timed ? 1 << 20 : 0),
                                 hash_ptrs(w, c->spec.n_layers, kv, dec->y, max_len,
                                                                      dec->head));
      auto it = c->graphs.find(key);
      if (it == c->graphs.end()) {
        cudaStream_t cap = P->s_dec;
        cudaGraph_t graph;
        int nk = 0;
        CUDA_TRY(cudaStreamBeginCapture(cap, cudaStreamCaptureModeThreadLocal));
        c->capturing = true;
        duet_status s = decode_step_kernels(c, cap, P->s_d, w, kv, ap, max_len, dec->y, dec->head, &nk);
        c->capturing = false;
        cudaError_t e = cudaStreamEndCapture(cap, &graph);
        if (s != DUET_OK) return s;
        if (e != cudaSuccess) DUET_FAIL(DUET_ERR_CUDA, "graph capture failed: %s", cudaGetErrorString(e));
        GraphEntry ge;
        ge.kernels = nk;
        e = cudaGraphInstantiate(&ge.exec, graph, 0);
        cudaGraphDestroy(graph);
        if (e != cudaSuccess) DUET_FAIL(DUET_ERR_CUDA, "graph instantiate failed: %s", cudaGetErrorString(e));
        if (c->graphs.size() >= kGraphCap) {  // evict the least recently used graph
          auto lru = c->graphs.begin();
          for (auto g = c->graphs.begin(); g != c->graphs.end(); ++g)
            if (g->second.last_use < lru->second.last_use) lru = g;
          CUDA_TRY(cudaStreamSynchronize(P->s_dec));  // its last replay may still be queued
          cudaGraphExecDestroy(lru->second.exec);
          c->graphs.erase(lru);
        }
        it = c->graphs.emplace(key, ge).first;
      }
      it->second.last_use = ++c->graph_clock;
      for (int j = 0; j < k; ++j) CUDA_TRY(cudaGraphLaunch(it->second.exec, st));
      kernels += k * it->second.kernels;
      if (dev_timed) {  // the work of the decode-attention launches the device timer measures
        c->dtimer_launches += k * c->spec.n_layers;
        c->dtimer_bytes += (double)k * c->spec.n_layers * ap.attn_bytes_dec;
        c->dtimer_flops += (double)k * c->spec.n_layers * ap.attn_flops_dec;
      }
    }
    CUDA_TRY(cudaEventRecord(c->ev_dec1, st));
  }
  if (has_pre) {
    int* img;
    int slot;
    DUET_TRY(stage_slot(c, &img, &slot));
    AttnPlan ap;
    const size_t n_int = build_meta(c, c->pre, img, pre, nullptr, &ap);
    cudaStream_t st = P->s_pre;
    CUDA_TRY(cudaStreamWaitEvent(st, c->ev_in, 0));
    CUDA_TRY(cudaEventRecord(c->ev_pre0, st));
    DUET_TRY(upload_meta(c, c->pre, img, slot, n_int, P->s_p, st, &kernels));
    // the prefill side's L layers as one graph launch (f4): the kernels read the chunk's positions
    // and page tables from the metadata just uploaded, so a graph serves every batch of the same shape
    // (rows, sequences, longest chunk and context) and buffers; live kernel timing needs direct launches
    constexpr int kPreClasses = (1 << DUET_KCLASS_GEMM) | (1 << DUET_KCLASS_PREFILL_ATTN) | (1 << DUET_KCLASS_OTHER);
    const bool pre_graph = !(c->lim.flags & (DUET_CTX_NO_GRAPH | DUET_CTX_NO_PREFILL_GRAPH)) &&
                           !(c->prof_on && (c->prof_mask & kPreClasses));
    GraphEntry* ge = nullptr;
    // shape-agnostic capture (f4, "device-side shapes"): the kernels are launched for the side's capacity
    // and read the chunk's row count and per-sequence lengths from the metadata, so ONE graph per
    // partition and buffer set serves every prefill shape (bf16 CTA-pair path with the fused RoPE
    // epilogue, no TP; DUET_PREFILL_DEVSHAPE=0 keeps the per-shape graphs)
    static const bool devshape_env = !getenv("DUET_PREFILL_DEVSHAPE") || atoi(getenv("DUET_PREFILL_DEVSHAPE")) != 0;
    const bool dev_shape = pre_graph && devshape_env && c->dt == DT::BF16 && c->spec.head_dim == 128 &&
                           !c->comm_pre && !c->ar_on && c->pre.cap_rows > 128;
    AttnPlan ap_cap = ap;  // the plan the shape-agnostic graph is launched with
    if (dev_shape) {
      ap_cap.n_pre = c->pre.cap_rows;
      ap_cap.n_seqs = c->pre.cap_seqs;
      ap_cap.max_q = c->pre.cap_rows;
    }
    if (pre_graph) {
      const PreKey key{(uint64_t)P->s_d, dev_shape ? ~0ull : (uint64_t)ap.n_pre, dev_shape ? 0 : (uint64_t)ap.n_seqs,
                       dev_shape ? 0 : (uint64_t)ap.max_q, dev_shape ? 0 : (uint64_t)ap.max_len_pre,
                       hash_ptrs(w, c->spec.n_layers, kv, pre->y, 0) ^ ((uint64_t)(uintptr_t)pre->x * 0x9E3779B97F4A7C15ull)};
      auto it = c->pre_graphs.find(key);
      if (it == c->pre_graphs.end()) {
        if (c->pre_seen.size() > 4096) c->pre_seen.clear();
        if (++c->pre_seen[key] >= 2) {
          cudaGraph_t graph;
          int nk = 0;
          CUDA_TRY(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
          c->capturing = true;
          duet_status sc = dev_shape ? run_layers(c, c->pre, st, P->s_p, ap_cap.n_pre, pre->x, pre->y, w, kv, ap_cap,
                                                  &nk, nullptr, nullptr, 1 << 30, c->pre.step() + 1)
                                     : run_layers(c, c->pre, st, P->s_p, ap.n_pre, pre->x, pre->y, w, kv, ap, &nk);
          c->capturing = false;
          cudaError_t e = cudaStreamEndCapture(st, &graph);
          if (sc != DUET_OK) return sc;
          if (e != cudaSuccess) DUET_FAIL(DUET_ERR_CUDA, "prefill graph capture failed: %s", cudaGetErrorString(e));
          GraphEntry g;
          g.kernels = nk;
          e = cudaGraphInstantiate(&g.exec, graph, 0);
          cudaGraphDestroy(graph);
          if (e != cudaSuccess) DUET_FAIL(DUET_ERR_CUDA, "prefill graph instantiate failed: %s", cudaGetErrorString(e));
          if (c->pre_graphs.size() >= kPreGraphCap) {  // evict the least recently used one
            auto lru = c->pre_graphs.begin();
            for (auto q = c->pre_graphs.begin(); q != c->pre_graphs.end(); ++q)
              if (q->second.last_use < lru->second.last_use) lru = q;
            CUDA_TRY(cudaDeviceSynchronize());  // its last replay may still be queued on some partition
            cudaGraphExecDestroy(lru->second.exec);
            c->pre_graphs.erase(lru);
          }
          c->pre_seen.erase(key);
          it = c->pre_graphs.emplace(key, g).first;
        }
      }
      if (it != c->pre_graphs.end()) ge = &it->second;
    }
    if (ge) {
      ge->last_use = ++c->graph_clock;
      CUDA_TRY(cudaGraphLaunch(ge->exec, st));
      kernels += ge->kernels;
    } else if (dev_shape) {  // the same launches the graph holds (its first run is bitwise the replays)
      DUET_TRY(run_layers(c, c->pre, st, P->s_p, ap_cap.n_pre, pre->x, pre->y, w, kv, ap_cap, &kernels, nullptr,
                          nullptr, 1 << 30, c->pre.step() + 1));
    } else {
      DUET_TRY(run_layers(c, c->pre, st, P->s_p, ap.n_pre, pre->x, pre->y, w, kv, ap, &kernels));
    }
    c->last_pre_graph = ge != nullptr;
    CUDA_TRY(cudaEventRecord(c->ev_pre1, st));
  }
  // join (a7): the caller's stream waits for both sides; no host sync
  if (has_dec) CUDA_TRY(cudaStreamWaitEvent(ust, c->ev_dec1, 0));
  if (has_pre) CUDA_TRY(cudaStreamWaitEvent(ust, c->ev_pre1, 0));
  c->last_kernels = kernels;
  return DUET_OK;
}

extern "C" duet_status duet_last_step_times(duet_ctx* c, duet_step_times* out) {
  clear_error();
  if (!c || !out) DUET_FAIL(DUET_ERR_INVALID_ARG, "ctx/out is NULL");
  if (c->last_mode < 0) DUET_FAIL(DUET_ERR_INVALID_ARG, "no step has run");
  std::memset(out, 0, sizeof *out);
  out->mode = c->last_mode;
  out->k = c->last_k;
  out->kernels = c->last_kernels;
  out->corun_s_d = c->last_mode == DUET_MODE_TEMPORAL ? c->last_corun : 0;
  out->prefill_graph = c->last_mode == DUET_MODE_SPATIAL && c->last_pre_graph ? 1 : 0;
  float ms = 0;
  if (c->last_mode == DUET_MODE_TEMPORAL) {
    CUDA_TRY(cudaEventElapsedTime(&ms, c->ev_pre0, c->ev_pre1));
    out->t_window = out->t_decode = out->t_prefill = ms * 1e-3;
    return DUET_OK;
  }
  float td = 0, tp = 0, w = 0;
  if (c->last_has_dec) CUDA_TRY(cudaEventElapsedTime(&td, c->ev_dec0, c->ev_dec1));
  if (c->last_has_pre) CUDA_TRY(cudaEventElapsedTime(&tp, c->ev_pre0, c->ev_pre1));
  if (c->last_has_dec && c->last_has_pre) {
    // window: first start -> last end
    float a = 0, b = 0;
    CUDA_TRY(cudaEventElapsedTime(&a, c->ev_dec0, c->ev_pre1));  // pre end rel. dec start
    CUDA_TRY(cudaEventElapsedTime(&b, c->ev_dec0, c->ev_pre0));  // pre start rel. dec start
    const float start = std::min(0.f, b);
    const float end = std::max(td, a);
    w = end - start;
  } else {
    w = c->last_has_dec ? td : tp;
  }
  out->t_window = w * 1e-3;
  out->t_decode = td * 1e-3;
  out->t_prefill = tp * 1e-3;
  return DUET_OK;
}

// ---------------------------------------------------------------------------------- tensor parallelism

extern "C" duet_status duet_nccl_unique_id(void* out, int32_t len) {
  clear_error();
  if (!out || len < (int32_t)sizeof(ncclUniqueId))
    DUET_FAIL(DUET_ERR_INVALID_ARG, "out must hold %d bytes", (int)sizeof(ncclUniqueId));
  DUET_TRY(load_nccl());
  ncclUniqueId id;
  NCCL_TRY(NCCL.GetUniqueId(&id));
  memcpy(out, &id, sizeof(id));
  return DUET_OK;
}

extern "C" duet_status duet_ctx_set_comms(duet_ctx* c, int32_t rank, const void* id_decode, const void* id_prefill) {
  clear_error();
  if (!c || !id_decode || !id_prefill) DUET_FAIL(DUET_ERR_INVALID_ARG, "ctx / unique ids are NULL");
  if (rank < 0 || rank >= c->spec.tp) DUET_FAIL(DUET_ERR_OUT_OF_RANGE, "rank %d outside [0, tp = %d)", rank, c->spec.tp);
  if (c->comm_dec || c->comm_pre) DUET_FAIL(DUET_ERR_INVALID_ARG, "communicators already set");
  DUET_TRY(load_nccl());
  CUDA_TRY(cudaSetDevice(c->device));
  ncclUniqueId a, b;
  memcpy(&a, id_decode, sizeof(a));
  memcpy(&b, id_prefill, sizeof(b));
  // each side's collectives run inside its own green context next to that side's compute;
  // cap the CTAs NCCL may occupy so an allreduce never fills a small decode partition (env overrides:
  // DUET_NCCL_MAXCTAS_DEC / _PRE, DUET_NCCL_NVLSCTAS)
  auto env_int = [](const char* n, int dflt) { const char* v = getenv(n); return v ? atoi(v) : dflt; };
  ncclConfig_t cfg_dec = NCCL_CONFIG_INITIALIZER, cfg_pre = NCCL_CONFIG_INITIALIZER;
  cfg_dec.maxCTAs = env_int("DUET_NCCL_MAXCTAS_DEC", 4);
  cfg_pre.maxCTAs = env_int("DUET_NCCL_MAXCTAS_PRE", 16);
  cfg_dec.nvlsCTAs = std::min(cfg_dec.maxCTAs, env_int("DUET_NCCL_NVLSCTAS", 4));
  cfg_pre.nvlsCTAs = std::min(cfg_pre.maxCTAs, env_int("DUET_NCCL_NVLSCTAS", 16));
  cfg_dec.commName = "duet-decode";
  cfg_pre.commName = "duet-prefill";
  NCCL_TRY(NCCL.CommInitRankConfig(&c->comm_dec, c->spec.tp, a, rank, &cfg_dec));
  NCCL_TRY(NCCL.CommInitRankConfig(&c->comm_pre, c->spec.tp, b, rank, &cfg_pre));
  c->tp_rank = rank;
  cudaDeviceSynchronize();  // captured graphs predate the communicators: drop them
  for (auto& kv : c->graphs)
    if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
  for (auto& kv : c->pre_graphs)
    if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
  c->graphs.clear();
  c->pre_graphs.clear();
  return DUET_OK;
}

// Asynchronous NCCL errors (SURVEY §5 failure detection): a peer failure or a network error surfaces
// here, not as a CUDA error; duet_step polls it before enqueuing work on a TP ctx.
static duet_status comms_healthy(duet_ctx* c) {
  ncclComm_t cs[2] = {c->comm_dec, c->comm_pre};
  const char* names[2] = {"decode", "prefill"};
  for (int i = 0; i < 2; ++i) {
    if (!cs[i]) continue;
    ncclResult_t ae = ncclSuccess;
    NCCL_TRY(NCCL.CommGetAsyncError(cs[i], &ae));
    if (ae != ncclSuccess && ae != ncclInProgress)
      DUET_FAIL(DUET_ERR_NCCL, "%s-side communicator reports an asynchronous error: %s", names[i],
                NCCL.GetErrorString(ae));
  }
  return DUET_OK;
}

// ---------------------------------------------------------------- fused GEMM + allreduce (f3)
static size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

// ar_grp[side] from the ranks' arena bases (the layout is the same on every rank: same spec and limits)
static void ar_fill_groups(duet_ctx* c) {
  const int n = c->spec.tp, d = c->spec.d_model;
  Side* sides[2] = {&c->dec, &c->pre};
  for (int i = 0; i < 2; ++i) {
    const auto& L = c->ar_lay[i];
    GemmAr& g = c->ar_grp[i];
    g = GemmAr{};
    g.n = n;
    g.rank = c->tp_rank;
    g.emul = 0;
    g.slot_tiles = gemm_ar_slot_tiles(std::max(sides[i]->cap_rows, 1), d, n, c->total_sms);
    const size_t ncnt = gemm_ar_counters(std::max(sides[i]->cap_rows, 1), d, n, c->total_sms);
    for (int r = 0; r < n; ++r) {
      char* b = c->ar_peer[r];
      g.slots[r] = (float*)(b + L.off_slots);
      g.cnt[r] = (unsigned*)(b + L.off_cnt);
      g.done[r] = g.cnt[r] + ncnt;
      g.out[r] = b + L.off_out0;  // the O projection's; run_layers swaps in off_out1 for the down projection
    }
  }
}

extern "C" duet_status duet_ctx_ar_handle(duet_ctx* c, void* out, int32_t len) {
  clear_error();
  if (!c || !out || len < (int32_t)sizeof(cudaIpcMemHandle_t))
    DUET_FAIL(DUET_ERR_INVALID_ARG, "ctx / out is NULL or len < %d", (int)sizeof(cudaIpcMemHandle_t));
  if (!c->comm_pre) DUET_FAIL(DUET_ERR_INVALID_ARG, "duet_ctx_set_comms first (the rank and the group)");
  if (c->spec.tp > kMaxTp) DUET_FAIL(DUET_ERR_UNSUPPORTED, "tp = %d > %d", c->spec.tp, kMaxTp);
  if (c->dt != DT::BF16) DUET_FAIL(DUET_ERR_UNSUPPORTED, "the fused allreduce runs on the bf16 CTA-pair GEMM");
  CUDA_TRY(cudaSetDevice(c->device));
  if (!c->ar_arena) {
    const int n = c->spec.tp, d = c->spec.d_model;
    Side* sides[2] = {&c->dec, &c->pre};
    size_t off = 0;
    for (int i = 0; i < 2; ++i) {
      const int R = std::max(sides[i]->cap_rows, 1);
      auto& L = c->ar_lay[i];
      L.off_slots = off;
      off = align256(off + gemm_ar_slot_floats(R, d, n, c->total_sms) * sizeof(float));
      L.off_cnt = off;
      off = align256(off + (gemm_ar_counters(R, d, n, c->total_sms) + 1) * sizeof(unsigned));
      L.off_out0 = off;
      off = align256(off + (size_t)R * d * 2);
      L.off_out1 = off;
      off = align256(off + (size_t)R * d * 2);
    }
    char* a = nullptr;
    CUDA_TRY(cudaMalloc(&a, off));
    CUDA_TRY(cudaMemset(a, 0, off));  // counters start at zero (their waiters re-arm them)
    c->ar_arena = a;
    c->ar_bytes = off;
  }
  cudaIpcMemHandle_t h;
  CUDA_TRY(cudaIpcGetMemHandle(&h, c->ar_arena));
  memcpy(out, &h, sizeof(h));
  return DUET_OK;
}

extern "C" duet_status duet_ctx_ar_open(duet_ctx* c, int32_t n, const void* handles) {
  clear_error();
  if (!c || !handles) DUET_FAIL(DUET_ERR_INVALID_ARG, "ctx / handles is NULL");
  if (!c->ar_arena) DUET_FAIL(DUET_ERR_INVALID_ARG, "duet_ctx_ar_handle first");
  if (n != c->spec.tp) DUET_FAIL(DUET_ERR_INVALID_ARG, "%d handles for a tp = %d group", n, c->spec.tp);
  if (c->ar_on) DUET_FAIL(DUET_ERR_INVALID_ARG, "the fused allreduce is already open");
  CUDA_TRY(cudaSetDevice(c->device));
  for (int r = 0; r < n; ++r) {
    if (r == c->tp_rank) {
      c->ar_peer[r] = c->ar_arena;
      continue;
    }
    cudaIpcMemHandle_t h;
    memcpy(&h, (const char*)handles + (size_t)r * sizeof(h), sizeof(h));
    void* p = nullptr;
    CUDA_TRY(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
    c->ar_peer[r] = (char*)p;
  }
  ar_fill_groups(c);
  cudaDeviceSynchronize();  // captured graphs use the NCCL allreduce: drop them
  for (auto& kv : c->graphs)
    if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
  for (auto& kv : c->pre_graphs)
    if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
  c->graphs.clear();
  c->pre_graphs.clear();
  c->ar_on = true;
  return DUET_OK;
}

extern "C" duet_status duet_op_gemm_ar_emul(duet_ctx* c, int32_t n_ranks, const void* A, const void* B, const void* R,
                                           void* C, int32_t M, int32_t N, int32_t K, void* stream) {
  clear_error();
  if (!c || !A || !B || !R || !C) DUET_FAIL(DUET_ERR_INVALID_ARG, "NULL operand");
  if (n_ranks < 1 || n_ranks > kMaxTp) DUET_FAIL(DUET_ERR_OUT_OF_RANGE, "n_ranks = %d (1..%d)", n_ranks, kMaxTp);
  if (c->dt != DT::BF16) DUET_FAIL(DUET_ERR_UNSUPPORTED, "bf16 ctx only");
  if (M <= 128 || N <= 0 || N % 32 || K <= 0 || K % 64)
    DUET_FAIL(DUET_ERR_OUT_OF_RANGE, "shape M=%d N=%d K=%d (M > 128, N %% 32 == 0, K %% 64 == 0)", M, N, K);
  if (n_ranks > c->total_sms / 2) DUET_FAIL(DUET_ERR_UNSUPPORTED, "%d ranks need >= %d SMs", n_ranks, 2 * n_ranks);
  CUDA_TRY(cudaSetDevice(c->device));
  const size_t sf = gemm_ar_slot_floats(M, N, n_ranks, c->total_sms),
               cn = gemm_ar_counters(M, N, n_ranks, c->total_sms) + 1;
  if (sf * n_ranks > c->emu_slot_floats) {
    if (c->emu_slots) CUDA_TRY(cudaFree(c->emu_slots));
    c->emu_slots = nullptr;
    c->emu_slot_floats = 0;
    CUDA_TRY(cudaMalloc(&c->emu_slots, sf * n_ranks * sizeof(float)));
    c->emu_slot_floats = sf * n_ranks;
  }
  if (cn * n_ranks > c->emu_cnt_n) {
    if (c->emu_cnt) CUDA_TRY(cudaFree(c->emu_cnt));
    c->emu_cnt = nullptr;
    c->emu_cnt_n = 0;
    CUDA_TRY(cudaMalloc(&c->emu_cnt, cn * n_ranks * sizeof(unsigned)));
    CUDA_TRY(cudaMemset(c->emu_cnt, 0, cn * n_ranks * sizeof(unsigned)));
    c->emu_cnt_n = cn * n_ranks;
  }
  GemmAr ar;
  ar.n = n_ranks;
  ar.rank = 0;
  ar.emul = 1;
  ar.slot_tiles = gemm_ar_slot_tiles(M, N, n_ranks, c->total_sms);
  for (int r = 0; r < n_ranks; ++r) {
    ar.slots[r] = c->emu_slots + (size_t)r * sf;
    ar.cnt[r] = c->emu_cnt + (size_t)r * cn;
    ar.done[r] = ar.cnt[r] + cn - 1;
    ar.out[r] = (char*)C + (size_t)r * M * N * 2;
  }
  GemmArgs g{A, B, nullptr, R, nullptr, M, N, K, K, K, N, N, EPI_RESIDUAL_AR};
  g.ar = &ar;
  if (!gemm2_supported(g, c->total_sms)) DUET_FAIL(DUET_ERR_UNSUPPORTED, "operands misaligned for the CTA-pair GEMM");
  if (launch_gemm2(g, c->total_sms, (cudaStream_t)stream) <= 0)
    DUET_FAIL(DUET_ERR_UNSUPPORTED, "fused GEMM + allreduce M=%d N=%d K=%d could not be launched", M, N, K);
  DUET_TRY(check_launch("gemm_ar_emul"));
  return DUET_OK;
}

extern "C" int32_t duet_ctx_last_pod(duet_ctx* c) { return c && c->last_pod ? 1 : 0; }

extern "C" duet_status duet_ctx_check_comms(duet_ctx* c) {
  clear_error();
  if (!c) DUET_FAIL(DUET_ERR_INVALID_ARG, "ctx is NULL");
  return comms_healthy(c);
}

extern "C" duet_status duet_calibrate_allreduce(duet_ctx* c, double* alpha_s, double* bw_bytes_s) {
  clear_error();
  if (!c || !alpha_s || !bw_bytes_s) DUET_FAIL(DUET_ERR_INVALID_ARG, "NULL argument");
  if (!c->comm_pre) DUET_FAIL(DUET_ERR_INVALID_ARG, "no communicators (duet_ctx_set_comms)");
  const int N = c->spec.tp;
  *alpha_s = 0.0;
  *bw_bytes_s = 0.0;
  if (N < 2) return DUET_OK;
  const size_t big = (size_t)64 << 20;
  void* buf = nullptr;
  CUDA_TRY(cudaMalloc(&buf, big));
  CUDA_TRY(cudaMemset(buf, 0, big));
  cudaEvent_t e0, e1;
  CUDA_TRY(cudaEventCreate(&e0));
  CUDA_TRY(cudaEventCreate(&e1));
  auto time_ar = [&](size_t bytes, float* ms) -> duet_status {
    std::vector<float> t;
    for (int rep = 0; rep < 9; ++rep) {
      CUDA_TRY(cudaEventRecord(e0, c->s_full));
      NCCL_TRY(NCCL.AllReduce(buf, buf, bytes / 2, ncclBfloat16, ncclSum, c->comm_pre, c->s_full));
      CUDA_TRY(cudaEventRecord(e1, c->s_full));
      CUDA_TRY(cudaEventSynchronize(e1));
      float x;
      CUDA_TRY(cudaEventElapsedTime(&x, e0, e1));
      if (rep >= 2) t.push_back(x);
    }
    std::sort(t.begin(), t.end());
    *ms = t[t.size() / 2];
    return DUET_OK;
  };
  float t_small, t_big;
  DUET_TRY(time_ar(16, &t_small));
  DUET_TRY(time_ar(big, &t_big));
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(buf);
  // P:237 ring model: t(B) = 2(N-1) alpha + 2(N-1) B / (N B_NVL)  (+ the local-reduce term, negligible)
  *alpha_s = t_small * 1e-3 / (2.0 * (N - 1));
  const double t_bw = std::max(t_big * 1e-3 - 2.0 * (N - 1) * *alpha_s, 1e-9);
  *bw_bytes_s = 2.0 * (N - 1) * (double)big / (N * t_bw);
  return DUET_OK;
}

// ---------------------------------------------------------------------------------- single ops

extern "C" duet_status duet_op_gemm(duet_ctx* c, const void* A, const void* B, void* C, const void* R,
                                    const void* bias, int32_t M, int32_t N, int32_t K, int32_t epi, void* stream) {
  clear_error();
  if (!c || !A || !B || !C) DUET_FAIL(DUET_ERR_INVALID_ARG, "NULL operand");
  if (M < 0 || N <= 0 || K <= 0 || K % 16) DUET_FAIL(DUET_ERR_OUT_OF_RANGE, "shape M=%d N=%d K=%d (K %% 16 == 0)", M, N, K);
  if (epi < 0 || epi > 2) DUET_FAIL(DUET_ERR_INVALID_ARG, "epi = %d", epi);
  if (epi == DUET_EPI_RESIDUAL && !R) DUET_FAIL(DUET_ERR_INVALID_ARG, "residual epilogue needs R");
  GemmArgs g{A, B, C, R, bias, M, N, K, K, K, N, N, epi};
  g.ws = c->pre.gemm_ws;  // op calls are stream-ordered by the caller, never concurrent with a step
  g.ws_floats = c->pre.gemm_ws_floats;
  if (M > 0 && launch_gemm(c->dt, g, c->total_sms, (cudaStream_t)stream) <= 0)
    DUET_FAIL(DUET_ERR_UNSUPPORTED, "gemm M=%d N=%d K=%d could not be launched (operand alignment?)", M, N, K);
  DUET_TRY(check_launch("gemm"));
  return DUET_OK;
}

extern "C" duet_status duet_op_rmsnorm(duet_ctx* c, const void* x, const void* g, void* h, int32_t n, void* stream) {
  clear_error();
  if (!c || !x || !g || !h) DUET_FAIL(DUET_ERR_INVALID_ARG, "NULL operand");
  launch_rmsnorm(c->dt, x, g, h, n, c->spec.d_model, (float)c->spec.norm_eps, (cudaStream_t)stream);
  DUET_TRY(check_launch("rmsnorm"));
  return DUET_OK;
}

// Stream of an op: the caller's (s_sms == 0, full device) or one side of a green-context partition,
// ordered after the caller's stream; *join is the partition stream to join back (nullptr: none).
static duet_status op_stream(duet_ctx* c, int s_sms, bool decode_side, cudaStream_t ust, cudaStream_t* st, int* sms,
                             cudaStream_t* join) {
  *join = nullptr;
  if (s_sms == 0) {
    *st = ust;
    *sms = c->total_sms;
    return DUET_OK;
  }
  Partition* P = nullptr;
  for (auto& p : c->parts)
    if ((decode_side ? p.s_d : c->total_sms - p.s_d) == s_sms) P = &p;
  if (!P) DUET_FAIL(DUET_ERR_OUT_OF_RANGE, "%d SMs is not an achievable %s partition", s_sms,
                    decode_side ? "decode" : "prefill");
  DUET_TRY(ensure_partition(c, *P));
  *st = decode_side ? P->s_dec : P->s_pre;
  *sms = decode_side ? P->s_d : P->s_p;
  CUDA_TRY(cudaEventRecord(c->ev_in, ust));
  CUDA_TRY(cudaStreamWaitEvent(*st, c->ev_in, 0));
  *join = *st;
  return DUET_OK;
}

extern "C" duet_status duet_op_decode_attn(duet_ctx* c, const void* q, int32_t q_stride, void* o, int32_t n,
                                           const int32_t* pos, const int32_t* page_table, int32_t max_pages,
                                           const void* k_pool, const void* v_pool, int32_t n_pages, int32_t s_d,
                                           void* stream) {
  clear_error();
  if (!c || !q || !o || !pos || !page_table || !k_pool || !v_pool) DUET_FAIL(DUET_ERR_INVALID_ARG, "NULL operand");
  if (n < 1 || n > c->lim.max_decode_reqs) DUET_FAIL(DUET_ERR_CAPACITY, "n = %d outside [1, max_decode_reqs]", n);
  if (q_stride < c->spec.n_q_heads * c->spec.head_dim || n_pages <= 0 || max_pages < 1)
    DUET_FAIL(DUET_ERR_INVALID_ARG, "q_stride = %d, n_pages = %d, max_pages = %d", q_stride, n_pages, max_pages);
  begin_page_check(c, n_pages);
  for (int r = 0; r < n; ++r) {
    if (pos[r] < 0 || pos[r] + 1 > c->lim.max_pos)
      DUET_FAIL(DUET_ERR_OUT_OF_RANGE, "row %d: pos = %d outside [0, max_pos)", r, pos[r]);
    DUET_TRY(check_pages(c, page_table, max_pages, r, pos[r] + 1, n_pages, "decode"));
  }
  CUDA_TRY(cudaSetDevice(c->device));
  cudaStream_t st, join;
  int sms;
  DUET_TRY(op_stream(c, s_d, true, (cudaStream_t)stream, &st, &sms, &join));
  duet_decode dd{};
  dd.n_reqs = n;
  dd.c = pos;  // the row's own position: attends to 0..pos[r]
  dd.page_table = page_table;
  dd.max_pages = max_pages;
  int* img;
  int slot, nk = 0;
  DUET_TRY(stage_slot(c, &img, &slot));
  AttnPlan ap;
  const size_t n_int = build_meta(c, c->dec, img, nullptr, &dd, &ap);
  DUET_TRY(upload_meta(c, c->dec, img, slot, n_int, sms, st, &nk));
  if (decode_attn(c, c->dec, ap, q, q_stride, o, k_pool, v_pool, n_pages, sms, st) <= 0)
    DUET_FAIL(DUET_ERR_UNSUPPORTED, "decode attention could not be launched");
  DUET_TRY(check_launch("decode attention"));
  if (join) {
    CUDA_TRY(cudaEventRecord(c->ev_dec1, join));
    CUDA_TRY(cudaStreamWaitEvent((cudaStream_t)stream, c->ev_dec1, 0));
  }
  return DUET_OK;
}

extern "C" duet_status duet_op_prefill_attn(duet_ctx* c, const void* q, int32_t q_stride, void* o, int32_t n_seqs,
                                            const int32_t* q_len, const int32_t* cpre, const int32_t* page_table,
                                            int32_t max_pages, const void* k_pool, const void* v_pool,
                                            int32_t n_pages, int32_t s_p, void* stream) {
  clear_error();
  if (!c || !q || !o || !q_len || !cpre || !page_table || !k_pool || !v_pool)
    DUET_FAIL(DUET_ERR_INVALID_ARG, "NULL operand");
  if (n_seqs < 1 || n_seqs > c->lim.max_prefill_seqs)
    DUET_FAIL(DUET_ERR_CAPACITY, "n_seqs = %d outside [1, max_prefill_seqs]", n_seqs);
  if (q_stride < c->spec.n_q_heads * c->spec.head_dim || n_pages <= 0 || max_pages < 1)
    DUET_FAIL(DUET_ERR_INVALID_ARG, "q_stride = %d, n_pages = %d, max_pages = %d", q_stride, n_pages, max_pages);
  begin_page_check(c, n_pages);
  long tot = 0;
  for (int s = 0; s < n_seqs; ++s) {
    if (q_len[s] < 1 || cpre[s] < 0 || (long)cpre[s] + q_len[s] > c->lim.max_pos)
      DUET_FAIL(DUET_ERR_OUT_OF_RANGE, "seq %d: q = %d, c = %d", s, q_len[s], cpre[s]);
    tot += q_len[s];
    DUET_TRY(check_pages(c, page_table, max_pages, s, cpre[s] + q_len[s], n_pages, "prefill"));
  }
  if (tot > c->lim.max_prefill_tokens + c->lim.max_decode_reqs)
    DUET_FAIL(DUET_ERR_CAPACITY, "%ld query rows exceed the ctx capacity", tot);
  CUDA_TRY(cudaSetDevice(c->device));
  cudaStream_t st, join;
  int sms;
  DUET_TRY(op_stream(c, s_p, false, (cudaStream_t)stream, &st, &sms, &join));
  duet_prefill pp{};
  pp.n_seqs = n_seqs;
  pp.q = q_len;
  pp.c = cpre;
  pp.page_table = page_table;
  pp.max_pages = max_pages;
  int* img;
  int slot, nk = 0;
  DUET_TRY(stage_slot(c, &img, &slot));
  AttnPlan ap;
  const size_t n_int = build_meta(c, c->pre, img, &pp, nullptr, &ap);
  DUET_TRY(upload_meta(c, c->pre, img, slot, n_int, sms, st, &nk));
  if (prefill_attn(c, c->pre, ap, q, q_stride, o, ap.n_pre, k_pool, v_pool, n_pages, sms, st) <= 0)
    DUET_FAIL(DUET_ERR_UNSUPPORTED, "prefill attention could not be launched");
  DUET_TRY(check_launch("prefill attention"));
  if (join) {
    CUDA_TRY(cudaEventRecord(c->ev_pre1, join));
    CUDA_TRY(cudaStreamWaitEvent((cudaStream_t)stream, c->ev_pre1, 0));
  }
  return DUET_OK;
}

// ---------------------------------------------------------------------------------- token times

extern "C" duet_status duet_token_times(duet_ctx* c, int32_t reset, uint64_t* out_ns, int32_t cap, int32_t* n) {
  clear_error();
  if (!c) DUET_FAIL(DUET_ERR_INVALID_ARG, "ctx is NULL");
  CUDA_TRY(cudaSetDevice(c->device));
  int cnt = 0;
  if (n || out_ns) {
    CUDA_TRY(cudaDeviceSynchronize());
    CUDA_TRY(cudaMemcpy(&cnt, c->tok_cnt, sizeof(int), cudaMemcpyDeviceToHost));
    if (out_ns && cap > 0 && cnt > kTokTsSlots)
      DUET_FAIL(DUET_ERR_CAPACITY, "%d stamps since the last reset overran the %d-slot ring", cnt, kTokTsSlots);
    const int m = out_ns ? std::min(cnt, std::max(cap, 0)) : 0;
    if (m > 0) CUDA_TRY(cudaMemcpy(out_ns, c->tok_ts, m * sizeof(uint64_t), cudaMemcpyDeviceToHost));
    if (n) *n = cnt;
  }
  if (reset) {
    CUDA_TRY(cudaDeviceSynchronize());
    CUDA_TRY(cudaMemset(c->tok_cnt, 0, sizeof(int)));
  }
  return DUET_OK;
}

// ---------------------------------------------------------------------------------- calibration

static duet_status calibrate_impl(duet_ctx* c, double* flops, double* bw, int32_t len, double pair_s);

extern "C" duet_status duet_calibrate(duet_ctx* c, double* flops, double* bw, int32_t len) {
  return calibrate_impl(c, flops, bw, len, 0.0);
}

extern "C" duet_status duet_calibrate_corun(duet_ctx* c, double* flops, double* bw, int32_t len, double pair_seconds) {
  if (!(pair_seconds > 0)) {
    clear_error();
    DUET_FAIL(DUET_ERR_INVALID_ARG, "pair_seconds = %g must be > 0", pair_seconds);
  }
  return calibrate_impl(c, flops, bw, len, pair_seconds);
}

static duet_status calibrate_impl(duet_ctx* c, double* flops, double* bw, int32_t len, double pair_s) {
  clear_error();
  if (!c || !flops || !bw) DUET_FAIL(DUET_ERR_INVALID_ARG, "NULL argument");
  if (len < c->total_sms + 1) DUET_FAIL(DUET_ERR_CAPACITY, "tables need %d entries", c->total_sms + 1);
  for (auto& p : c->parts) DUET_TRY(ensure_partition(c, p));
  size_t free_b = 0, total_b = 0;
  CUDA_TRY(cudaMemGetInfo(&free_b, &total_b));
  size_t n_bytes = (size_t)2 << 30;  // >> L2 (126 MB)
  while (n_bytes > ((size_t)512 << 20) && n_bytes + ((size_t)1 << 30) > free_b) n_bytes >>= 1;
  void* buf = nullptr;
  unsigned long long* sink = nullptr;
  CUDA_TRY(cudaMalloc(&buf, n_bytes));
  CUDA_TRY(cudaMalloc(&sink, 4096 * sizeof(unsigned long long)));
  // Pi_SM(S): the achievable rate of the model's largest linear operator ("gemm
  // microbenchmark"): gate-up shape, M = the prefill chunk capacity (256..8192 rows), N = 2 m, K = d
  const int GM = std::max(256, std::min(8192, ((c->lim.max_prefill_tokens + 255) / 256) * 256));
  const int GN = ((2 * c->spec.ffn_dim + 255) / 256) * 256, GK = ((c->spec.d_model + 63) / 64) * 64;
  const size_t es = dt_size(c->dt);
  void *A = nullptr, *B = nullptr, *C = nullptr;
  CUDA_TRY(cudaMalloc(&A, (size_t)GM * GK * es));
  CUDA_TRY(cudaMalloc(&B, (size_t)GN * GK * es));
  CUDA_TRY(cudaMalloc(&C, (size_t)GM * GN * es));
  launch_fill_hash(c->dt, A, (size_t)GM * GK, 1u, c->s_full);
  launch_fill_hash(c->dt, B, (size_t)GN * GK, 2u, c->s_full);
  launch_fill_hash(DT::BF16, buf, n_bytes / 2, 3u, c->s_full);  // K/V pools of the bandwidth calibration
  CUDA_TRY(cudaStreamSynchronize(c->s_full));
  cudaEvent_t e0, e1;
  CUDA_TRY(cudaEventCreate(&e0));
  CUDA_TRY(cudaEventCreate(&e1));
  // B_HBM(S) is the bandwidth the library's memory-bound hot kernel achieves on S SMs: paged decode
  // attention (bf16) over a synthetic batch whose K/V pools fill the buffer (64 requests, identity page
  // tables), else (fp32 contexts) an 8 KiB-page cp.async streaming kernel.
  const auto& sp = c->spec;
  const int n_req = std::min(64, c->dec.part_rows);
  const size_t page_bytes = (size_t)sp.n_kv_heads * kPageSize * sp.head_dim * es;  // one page, all kv heads
  const int pages_per_req = (int)std::min<size_t>((n_bytes / 2) / page_bytes / std::max(n_req, 1), 4096);
  DecodeAttnArgs da{};
  int* d_meta = nullptr;
  void *dq = nullptr, *dout = nullptr;
  double attn_bytes = 0;
  bool use_attn = c->dt == DT::BF16 && n_req > 0 && pages_per_req >= 8;
  if (use_attn) {
    std::vector<int> meta((size_t)n_req * (pages_per_req + 2));
    int* h_pos = meta.data();
    int* h_tok = h_pos + n_req;
    int* h_tab = h_tok + n_req;
    const int len = pages_per_req * kPageSize;
    for (int r = 0; r < n_req; ++r) {
      h_pos[r] = len - 1;
      h_tok[r] = r;
      for (int j = 0; j < pages_per_req; ++j) h_tab[(size_t)r * pages_per_req + j] = r * pages_per_req + j;
    }
    CUDA_TRY(cudaMalloc(&d_meta, meta.size() * sizeof(int)));
    CUDA_TRY(cudaMemcpy(d_meta, meta.data(), meta.size() * sizeof(int), cudaMemcpyHostToDevice));
    CUDA_TRY(cudaMalloc(&dq, (size_t)n_req * sp.n_q_heads * sp.head_dim * es));
    CUDA_TRY(cudaMemset(dq, 0, (size_t)n_req * sp.n_q_heads * sp.head_dim * es));
    CUDA_TRY(cudaMalloc(&dout, (size_t)n_req * sp.n_q_heads * sp.head_dim * es));
    da.q = dq;
    da.q_stride = sp.n_q_heads * sp.head_dim;
    da.o = dout;
    da.n = n_req;
    da.hq = sp.n_q_heads;
    da.hkv = sp.n_kv_heads;
    da.dh = sp.head_dim;
    da.pos = d_meta;
    da.tok_row = d_meta + n_req;
    da.table = d_meta + 2 * n_req;
    da.max_pages = pages_per_req;
    da.page_size = kPageSize;
    da.k_pool = buf;
    da.v_pool = (const char*)buf + (size_t)n_req * pages_per_req * page_bytes;
    da.part_o = c->dec.part_o;
    da.part_ml = c->dec.part_ml;
    da.max_splits = kMaxSplits;
    da.max_len = len;
    da.n_pages = n_req * pages_per_req;
    attn_bytes = 2.0 * (double)n_req * pages_per_req * page_bytes;
  }
  // f4 co-run rates: the prefill-attention kernel on a causal chunk of QF rows over pages of the same
  // pool (bf16, d_h = 128 contexts whose tensor-core flash kernel runs)
  const int QF = std::min(2048, std::min(c->lim.max_pages_per_seq * kPageSize, c->lim.max_prefill_tokens)) / 128 * 128;
  void *dqf = nullptr, *dof = nullptr;
  AttnPlan apf;
  double fa_flops = 0;
  bool use_fa = use_attn && sp.head_dim == 128 && QF >= 128 && QF / kPageSize <= da.n_pages &&
                c->lim.max_prefill_seqs >= 1;
  if (use_fa) {
    const size_t qbytes = (size_t)QF * sp.n_q_heads * sp.head_dim * es;
    CUDA_TRY(cudaMalloc(&dqf, qbytes));
    CUDA_TRY(cudaMalloc(&dof, qbytes));
    launch_fill_hash(c->dt, dqf, qbytes / es, 7u, c->s_full);
    std::vector<int32_t> tab(QF / kPageSize);
    for (int j = 0; j < (int)tab.size(); ++j) tab[j] = j;
    const int32_t q1 = QF, c0 = 0;
    duet_prefill pp{1, &q1, &c0, tab.data(), (int32_t)tab.size(), nullptr, nullptr};
    int* img;
    int slot, nk = 0;
    DUET_TRY(stage_slot(c, &img, &slot));
    const size_t n_int = build_meta(c, c->pre, img, &pp, nullptr, &apf);
    DUET_TRY(upload_meta(c, c->pre, img, slot, n_int, c->total_sms, c->s_full, &nk));
    CUDA_TRY(cudaStreamSynchronize(c->s_full));
    fa_flops = apf.attn_flops_pre;
  }
  std::vector<double> mf(c->total_sms + 1, 0.0), mb(c->total_sms + 1, 0.0), mfa(c->total_sms + 1, 0.0);
  auto measure = [&](cudaStream_t st, int sms) -> duet_status {
    if (mf[sms] > 0) return DUET_OK;
    std::vector<float> tb, tf;
    for (int rep = 0; rep < 7; ++rep) {
      CUDA_TRY(cudaEventRecord(e0, st));
      if (use_attn) {
        da.num_sms = sms;
        launch_decode_attn(c->dt, da, st);
      } else {
        launch_stream_pages(buf, n_bytes, sink, sms, st);
      }
      CUDA_TRY(cudaEventRecord(e1, st));
      CUDA_TRY(cudaEventSynchronize(e1));
      float ms;
      CUDA_TRY(cudaEventElapsedTime(&ms, e0, e1));
      tb.push_back(ms);
    }
    GemmArgs g{A, B, C, nullptr, nullptr, GM, GN, GK, GK, GK, GN, 0, EPI_STORE};
    const int reps = c->dt == DT::BF16 ? 5 : 1;
    for (int rep = 0; rep < reps; ++rep) {
      CUDA_TRY(cudaEventRecord(e0, st));
      launch_gemm(c->dt, g, sms, st);
      CUDA_TRY(cudaEventRecord(e1, st));
      CUDA_TRY(cudaEventSynchronize(e1));
      float ms;
      CUDA_TRY(cudaEventElapsedTime(&ms, e0, e1));
      tf.push_back(ms);
    }
    if (use_fa) {
      std::vector<float> ta;
      for (int rep = 0; rep < 5; ++rep) {
        CUDA_TRY(cudaEventRecord(e0, st));
        if (prefill_attn(c, c->pre, apf, dqf, sp.n_q_heads * sp.head_dim, dof, QF, da.k_pool, da.v_pool, da.n_pages,
                         sms, st) <= 0)
          DUET_FAIL(DUET_ERR_CUDA, "calibration: prefill attention could not be launched");
        CUDA_TRY(cudaEventRecord(e1, st));
        CUDA_TRY(cudaEventSynchronize(e1));
        float ms;
        CUDA_TRY(cudaEventElapsedTime(&ms, e0, e1));
        ta.push_back(ms);
      }
      std::sort(ta.begin(), ta.end());
      mfa[sms] = fa_flops / (ta[ta.size() / 2] * 1e-3);
    }
    DUET_TRY(check_launch("calibration"));
    std::sort(tb.begin(), tb.end());
    std::sort(tf.begin(), tf.end());
    mb[sms] = (use_attn ? attn_bytes : (double)n_bytes) / (tb[tb.size() / 2] * 1e-3);
    mf[sms] = 2.0 * GM * (double)GN * GK / (tf[tf.size() / 2] * 1e-3);
    return DUET_OK;
  };
  DUET_TRY(measure(c->s_full, c->total_sms));
  for (auto& p : c->parts) {
    DUET_TRY(measure(p.s_dec, p.s_d));
    DUET_TRY(measure(p.s_pre, p.s_p));
  }
  // Co-run, sustained refinement (reading R-f, "achievable"): the tables the predictor needs are
  // the rates each partition side achieves while the other side runs the OTHER phase's hot kernel and
  // the GPU sits at its sustained (power-capped) clocks — not a short burst on an idle GPU.  After a
  // heat-up, every split (S_d, S_p) runs two phases of ~pair_s seconds: the GEMM on S_p while the
  // decode attention streams on S_d (-> Pi(S_p), B(S_d)), then the roles swapped (-> Pi(S_d), B(S_p));
  // the full device runs each kernel alone, sustained.  Each rate is taken over the middle 60 % of
  // its side's launches, where the two loops overlap.
  std::vector<double> mf_c(c->total_sms + 1, 0.0), mb_c(c->total_sms + 1, 0.0);
  if (pair_s > 0 && use_attn) {
    const double g_flops = 2.0 * GM * (double)GN * GK;
    GemmArgs g{A, B, C, nullptr, nullptr, GM, GN, GK, GK, GK, GN, 0, EPI_STORE};
    cudaEvent_t ev[4];
    for (auto& e : ev) CUDA_TRY(cudaEventCreate(&e));
    // n launches of one kernel on st; events after launch 2n/5 and before launch n - n/10: the first
    // 40 % let the clocks settle to the pair's power state (the previous phase ran another mix), the
    // last 10 % may run after the other side's loop has ended
    auto lo_of = [](int n) { return 2 * n / 5; };
    auto hi_of = [](int n) { return n - n / 10; };
    auto loop = [&](cudaStream_t st, int sms, bool gemm, int n, cudaEvent_t ea, cudaEvent_t eb) -> duet_status {
      const int lo = lo_of(n), hi = hi_of(n);
      for (int i = 0; i < n; ++i) {
        if (i == lo) CUDA_TRY(cudaEventRecord(ea, st));
        if (i == hi) CUDA_TRY(cudaEventRecord(eb, st));
        if (gemm) {
          if (launch_gemm(c->dt, g, sms, st) <= 0) DUET_FAIL(DUET_ERR_CUDA, "calibration GEMM could not be launched");
        } else {
          da.num_sms = sms;
          if (launch_decode_attn(c->dt, da, st) <= 0)
            DUET_FAIL(DUET_ERR_CUDA, "calibration decode attention could not be launched");
        }
      }
      return DUET_OK;
    };
    auto n_for = [&](double t_one, double secs) { return std::max(5, (int)std::ceil(secs / std::max(t_one, 1e-7))); };
    auto elapsed = [&](cudaEvent_t a0, cudaEvent_t a1) -> double {
      float ms = 0;
      cudaEventElapsedTime(&ms, a0, a1);
      return ms * 1e-3;
    };
    const int S = c->total_sms;
    // heat-up: about a second of the full-device GEMM (the clocks settle at the power cap)
    DUET_TRY(loop(c->s_full, S, true, n_for(g_flops / mf[S], 1.0), ev[0], ev[1]));
    CUDA_TRY(cudaStreamSynchronize(c->s_full));
    for (auto& p : c->parts) {
      for (int phase = 0; phase < 2; ++phase) {
        const int sg = phase == 0 ? p.s_p : p.s_d, sa = phase == 0 ? p.s_d : p.s_p;
        cudaStream_t stg = phase == 0 ? p.s_pre : p.s_dec, sta = phase == 0 ? p.s_dec : p.s_pre;
        const int ng = n_for(g_flops / mf[sg], pair_s), na = n_for(attn_bytes / mb[sa], pair_s);
        DUET_TRY(loop(stg, sg, true, ng, ev[0], ev[1]));
        DUET_TRY(loop(sta, sa, false, na, ev[2], ev[3]));
        CUDA_TRY(cudaStreamSynchronize(stg));
        CUDA_TRY(cudaStreamSynchronize(sta));
        mf_c[sg] = g_flops * (hi_of(ng) - lo_of(ng)) / elapsed(ev[0], ev[1]);
        mb_c[sa] = attn_bytes * (hi_of(na) - lo_of(na)) / elapsed(ev[2], ev[3]);
      }
    }
    {  // the full device, each kernel alone, sustained
      const int ng = n_for(g_flops / mf[S], 4 * pair_s), na = n_for(attn_bytes / mb[S], 2 * pair_s);
      DUET_TRY(loop(c->s_full, S, true, ng, ev[0], ev[1]));
      DUET_TRY(loop(c->s_full, S, false, na, ev[2], ev[3]));
      CUDA_TRY(cudaStreamSynchronize(c->s_full));
      mf_c[S] = g_flops * (hi_of(ng) - lo_of(ng)) / elapsed(ev[0], ev[1]);
      mb_c[S] = attn_bytes * (hi_of(na) - lo_of(na)) / elapsed(ev[2], ev[3]);
    }
    DUET_TRY(check_launch("co-run calibration"));
    for (auto e : ev) cudaEventDestroy(e);
    // reading R-g: one 0.1-s phase on a power-capped GPU varies by +-10 %; a median of three over the
    // per-SM rates of neighbouring sizes removes a lone outlier (which would mislead Alg. 1's k)
    std::vector<int32_t> sizes;
    for (int s = 1; s <= S; ++s)
      if (mf_c[s] > 0 && mb_c[s] > 0) sizes.push_back(s);
    DUET_TRY(duet_profile_smooth(sizes.data(), (int32_t)sizes.size(), mf_c.data(), S + 1));
    DUET_TRY(duet_profile_smooth(sizes.data(), (int32_t)sizes.size(), mb_c.data(), S + 1));
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(buf);
  if (dqf) cudaFree(dqf);
  if (dof) cudaFree(dof);
  // the f4 co-run decision of later temporal steps uses the measured attention rates
  if (use_attn && use_fa)
    for (int s = 1; s <= c->total_sms; ++s) {
      c->cal_bw[s] = mb[s];
      c->cal_fa[s] = mfa[s];
    }
  if (d_meta) cudaFree(d_meta);
  if (dq) cudaFree(dq);
  if (dout) cudaFree(dout);
  cudaFree(sink);
  cudaFree(A);
  cudaFree(B);
  cudaFree(C);
  for (int s2 = 1; s2 <= c->total_sms; ++s2) {
    if (mf_c[s2] > 0) mf[s2] = mf_c[s2];
    if (mb_c[s2] > 0) mb[s2] = mb_c[s2];
  }
  // fill unmeasured sizes by linear interpolation (from 0 at S = 0)
  std::vector<int> known;
  for (int s = 1; s <= c->total_sms; ++s)
    if (mf[s] > 0) known.push_back(s);
  for (int s = 0; s <= c->total_sms; ++s) {
    if (s == 0) {
      flops[0] = bw[0] = 0.0;
      continue;
    }
    if (mf[s] > 0) {
      flops[s] = mf[s];
      bw[s] = mb[s];
      continue;
    }
    int lo = 0, hi = -1;
    for (int kx : known) {
      if (kx < s) lo = kx;
      if (kx > s && hi < 0) hi = kx;
    }
    if (hi < 0) hi = known.back();
    const double f_lo = lo ? mf[lo] : 0.0, b_lo = lo ? mb[lo] : 0.0;
    const double t = (double)(s - lo) / (double)(hi - lo);
    flops[s] = f_lo + t * (mf[hi] - f_lo);
    bw[s] = b_lo + t * (mb[hi] - b_lo);
  }
  for (int s = c->total_sms + 1; s < len; ++s) flops[s] = bw[s] = 0.0;
  return DUET_OK;
}

// The hardware stream ceiling per partition size (roofline denominators of the decode side, SURVEY
// §8(d)): plain 16-B LDG streaming of a >= 1 GiB buffer from 2048 threads per SM, median of 5.
extern "C" duet_status duet_calibrate_stream(duet_ctx* c, double* bw, int32_t len) {
  clear_error();
  if (!c || !bw) DUET_FAIL(DUET_ERR_INVALID_ARG, "NULL argument");
  if (len < c->total_sms + 1) DUET_FAIL(DUET_ERR_CAPACITY, "table needs %d entries", c->total_sms + 1);
  CUDA_TRY(cudaSetDevice(c->device));
  for (auto& p : c->parts) DUET_TRY(ensure_partition(c, p));
  size_t free_b = 0, total_b = 0;
  CUDA_TRY(cudaMemGetInfo(&free_b, &total_b));
  size_t n_bytes = (size_t)2 << 30;
  while (n_bytes > ((size_t)256 << 20) && n_bytes + ((size_t)1 << 30) > free_b) n_bytes >>= 1;
  void* buf = nullptr;
  unsigned long long* sink = nullptr;
  CUDA_TRY(cudaMalloc(&buf, n_bytes));
  CUDA_TRY(cudaMalloc(&sink, 4 * 160 * sizeof(unsigned long long)));
  launch_fill_hash(DT::BF16, buf, n_bytes / 2, 5u, c->s_full);
  CUDA_TRY(cudaStreamSynchronize(c->s_full));
  cudaEvent_t e0, e1;
  CUDA_TRY(cudaEventCreate(&e0));
  CUDA_TRY(cudaEventCreate(&e1));
  for (int s = 0; s < len; ++s) bw[s] = 0.0;
  auto measure = [&](cudaStream_t st, int sms) -> duet_status {
    if (bw[sms] > 0) return DUET_OK;
    std::vector<float> t;
    for (int rep = 0; rep < 5; ++rep) {
      CUDA_TRY(cudaEventRecord(e0, st));
      launch_stream_read(buf, n_bytes, sink, sms, st);
      CUDA_TRY(cudaEventRecord(e1, st));
      CUDA_TRY(cudaEventSynchronize(e1));
      float ms;
      CUDA_TRY(cudaEventElapsedTime(&ms, e0, e1));
      t.push_back(ms);
    }
    std::sort(t.begin(), t.end());
    bw[sms] = (double)n_bytes / (t[t.size() / 2] * 1e-3);
    return DUET_OK;
  };
  duet_status st = measure(c->s_full, c->total_sms);
  for (auto& p : c->parts) {
    if (st == DUET_OK) st = measure(p.s_dec, p.s_d);
    if (st == DUET_OK) st = measure(p.s_pre, p.s_p);
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(buf);
  cudaFree(sink);
  return st;
}

// ---------------------------------------------------------------------------------- live timing

extern "C" duet_status duet_profile_enable(duet_ctx* c, int32_t class_mask) {
  clear_error();
  if (!c) DUET_FAIL(DUET_ERR_INVALID_ARG, "ctx is NULL");
  c->prof_on = (class_mask & DUET_PROFILE_ALL) != 0;
  c->prof_mask = class_mask & DUET_PROFILE_ALL;
  c->prof_pending.clear();
  c->prof_used = 0;
  for (auto& s : c->prof_acc) s = duet_kernel_stats{};
  CUDA_TRY(cudaSetDevice(c->device));
  if (!c->dev_timer) CUDA_TRY(cudaMalloc(&c->dev_timer, 8 * sizeof(unsigned long long)));
  CUDA_TRY(cudaDeviceSynchronize());
  const unsigned long long init[8] = {~0ull, 0, 0, 0, 0, 0, 0, 0};
  CUDA_TRY(cudaMemcpy(c->dev_timer, init, sizeof init, cudaMemcpyHostToDevice));
  c->dtimer_flops = c->dtimer_bytes = 0;
  c->dtimer_launches = 0;
  return DUET_OK;
}

extern "C" duet_status duet_profile_read(duet_ctx* c, duet_kernel_stats* out) {
  clear_error();
  if (!c || !out) DUET_FAIL(DUET_ERR_INVALID_ARG, "ctx/out is NULL");
  for (const auto& r : c->prof_pending) {
    const auto& ev = c->prof_pool[r.idx];
    CUDA_TRY(cudaEventSynchronize(ev.second));
    float ms = 0;
    CUDA_TRY(cudaEventElapsedTime(&ms, ev.first, ev.second));
    auto& a = c->prof_acc[r.cls];
    a.launches += 1;
    a.seconds += ms * 1e-3;
    a.flops += r.flops;
    a.bytes += r.bytes;
  }
  c->prof_pending.clear();
  c->prof_used = 0;
  if (c->dev_timer) {  // decode attention timed on the device inside the decode graphs
    CUDA_TRY(cudaSetDevice(c->device));
    CUDA_TRY(cudaDeviceSynchronize());
    unsigned long long t[8];
    CUDA_TRY(cudaMemcpy(t, c->dev_timer, sizeof t, cudaMemcpyDeviceToHost));
    if (t[4] > 0) {
      if ((int)t[4] != c->dtimer_launches)
        DUET_FAIL(DUET_ERR_CUDA, "device timer counted %llu decode-attention launches, %d were replayed", t[4],
                  c->dtimer_launches);
      auto& a = c->prof_acc[DUET_KCLASS_DECODE_ATTN];
      a.launches += (int32_t)t[4];
      a.seconds += (double)t[3] * 1e-9;
      a.flops += c->dtimer_flops;
      a.bytes += c->dtimer_bytes;
    }
    const unsigned long long init[8] = {~0ull, 0, 0, 0, 0, 0, 0, 0};
    CUDA_TRY(cudaMemcpy(c->dev_timer, init, sizeof init, cudaMemcpyHostToDevice));
    c->dtimer_flops = c->dtimer_bytes = 0;
    c->dtimer_launches = 0;
  }
  for (int i = 0; i < DUET_KCLASS_N; ++i) out[i] = c->prof_acc[i];
  return DUET_OK;
}

/*
 * duet.h — C ABI of libduet.so: the data-parallel hot path of DuetServe (arXiv 2511.04791)
 * on one B200 (sm_100a).
 *
 * Citations: "P:n" is line n of the paper text, with its section / equation /
 * algorithm; "S:n" a line of the CPU-simulator spec, used only for interface and
 * error conventions.  Readings of ambiguous passages are numbered as in DESIGN.md §Readings.
 *
 * Conventions (all entry points)
 *  - Status: DUET_OK (0) or a negative duet_status.  The message of the last failure on the
 *    calling thread is returned by duet_last_error(); it names the offending value.
 *  - Ownership: the caller owns every buffer it passes (host or device).  The library owns
 *    only a duet_ctx and the device workspace / pinned staging it sizes at duet_ctx_create
 *    from duet_ctx_limits; duet_step never allocates.
 *  - Host vs device: every pointer documented "host" is read by the CPU before the call
 *    returns; every pointer documented "device" is a CUDA device address on ctx's device.
 *  - Validation happens on the host before any launch; on error nothing is enqueued.
 *  - Thread safety: duet_predict_latency / duet_choose_split are pure and thread-safe
 *    (S:97).  A duet_ctx is used by one thread at a time.
 */
#ifndef DUET_H
#define DUET_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  DUET_OK = 0,
  DUET_ERR_INVALID_ARG = -1,   /* null pointer, negative size, unknown enum value              */
  DUET_ERR_OUT_OF_RANGE = -2,  /* an index / count outside its bound, bad page table    */
  DUET_ERR_CONFIG = -3,        /* non-positive profile entry, tp=0 or tp not
                                  dividing heads/ffn, inconsistent model spec          */
  DUET_ERR_UNSUPPORTED = -4,   /* a shape the kernels do not implement (e.g. head_dim != 64/128) */
  DUET_ERR_CUDA = -5,          /* a CUDA runtime / driver call failed                          */
  DUET_ERR_CAPACITY = -6,      /* a request exceeds the limits the ctx was created with        */
  DUET_ERR_NCCL = -7           /* libnccl missing or an NCCL call failed (tensor parallelism)  */
} duet_status;

/* Message of the last failure on this thread ("" if none).  Library-owned, valid until the
 * next call on this thread. */
const char* duet_last_error(void);
/* ABI version (bumped on any struct change). */
int32_t duet_abi_version(void);

/* ----------------------------------------------------------------- model & hardware */

/* Transformer dimensions (P:90-99 with readings #1-#6).
 *  d_model = n_q_heads * head_dim;  n_q_heads % n_kv_heads == 0;  elem_bytes s in {1,2,4}
 *  is the element size the roofline counts bytes with; ffn_gated=1 is SwiGLU
 *  (reading #3: gate-up projection d_o = 2m); tp = tensor-parallel degree N. */
typedef struct {
  int32_t n_layers, d_model, ffn_dim, n_q_heads, n_kv_heads, head_dim, vocab;
  int32_t elem_bytes, ffn_gated, qkv_bias, tp;
  double rope_theta, norm_eps;
} duet_model_spec;

/* Per-partition throughput tables Pi_SM(S), B_HBM(S) measured at init (§4.2).
 *  flops_at_sms / bw_at_sms: host arrays of total_sms+1 doubles indexed by SM count S
 *  (index 0 unused); FLOP/s and bytes/s; must be > 0 at every S the call evaluates.
 *  cand_sd_sms: host array of n_cand achievable decode-partition sizes S_d, ascending
 *  (reading #16: Alg. 1's range(1, S+1, 2) is replaced by what the partition launcher can
 *  provision; entries >= total_sms are skipped).
 *  nvlink_bw (B/s, per direction) and allreduce_alpha (s) feed the ring allreduce term
 *  (P:236-239); unused when tp == 1. */
typedef struct {
  int32_t total_sms;
  int32_t n_cand;
  const int32_t* cand_sd_sms;
  const double* flops_at_sms;
  const double* bw_at_sms;
  double nvlink_bw;
  double allreduce_alpha;
} duet_hw_profile;

enum { DUET_PHASE_PREFILL_FULL = 0, DUET_PHASE_PREFILL_CHUNK = 1, DUET_PHASE_DECODE = 2 };

/* One scheduled request: q new query tokens, c cached tokens.
 * Phase invariants: decode q==1 && c>0; prefill-full q>=1 && c==0; prefill-chunk q>=1 && c>0.
 * emits_logits: 1 if this entry produces logits (counts toward t_cls, reading #12). */
typedef struct { int32_t q, c, phase, emits_logits; } duet_req;

/* Latency breakdown in seconds.  t_block = ((t_linear + t_norm_act) + t_attn)
 * + t_allreduce ; t_total = L * t_block + t_cls. */
typedef struct {
  double t_linear, t_norm_act, t_attn, t_allreduce, t_block, t_cls, t_total;
} duet_latency;

enum { DUET_OPT_FORCE_SPATIAL = 1u, DUET_OPT_INCLUDE_CLS = 2u, DUET_OPT_VERBATIM_INFEASIBLE = 4u,
       DUET_OPT_BOUNDARY_TBT = 8u };

/* f_roofline(batch, Pi_SM(sms), B_HBM(sms)) — the attention-aware roofline model of §4.1
 * (P:194-250): token-level operators max(F/Pi, B/B) with F_lin = 2 n d_i d_o,
 * B_lin = (n d_i + d_i d_o + n d_o) s; attention per request
 * F = 4 h_q q (q+c) d_h + 2 h_q q (q+c), B = 2 h_q q d_h s + 2 h_kv (q+c) d_h s, max taken
 * per request then summed (reading #8: B_SM read as B_HBM(S)); two ring
 * allreduces per block when tp > 1; t_cls when opts has INCLUDE_CLS.
 * Evaluation order is fixed and the result is bit-identical to the
 * oracle (fp64, no contraction).
 *  batch: host array of n entries (n may be 0 -> all-zero result).
 *  sms: partition size S in [1, hw->total_sms].
 * Errors: INVALID_ARG (null), OUT_OF_RANGE (sms, an entry violating its phase invariant),
 *         CONFIG (spec invariants, tp divisibility, non-positive profile entry at sms). */
duet_status duet_predict_latency(const duet_model_spec* spec, const duet_hw_profile* hw,
                                 const duet_req* batch, int32_t n, int32_t sms, uint32_t opts,
                                 duet_latency* out);

enum { DUET_MODE_TEMPORAL = 0, DUET_MODE_SPATIAL = 1 };
enum { DUET_FLAG_INFEASIBLE = 1, DUET_FLAG_DEGENERATE = 2 };

/* Partition configuration C* = (S_p, S_d, k) of Alg. 1 with its predictions.
 * Temporal: s_p = total_sms, s_d = 0, k = 1, t_p = t_d = t_mixed, rho = sum(q)/t_mixed. */
typedef struct {
  int32_t mode, s_p, s_d, k, flags;
  double t_mixed, t_p, t_d, rho;
} duet_split;

/* Algorithm 1: t_mixed = f_roofline(all, S); temporal if t_mixed <= tau
 * (reading #19) unless FORCE_SPATIAL; else for S_d in cand ascending: t_d(S_d), skip if
 * > tau; t_p(S - S_d); k in {floor(t_p/t_d), floor(t_p/t_d)+1} clamped to [1, k_max]
 * (reading #17); rho = (k T_dec + T_pre) / max(k t_d, t_p); strict ">" keeps the
 * first maximum (reading #18).  Fallbacks are flagged, never silent: DEGENERATE
 * (one phase absent -> temporal), INFEASIBLE (no S_d meets tau -> argmin t_d; reading #20b: that
 * spatial split is kept only if its rho >= the temporal rho sum(q)/t_mixed, else the batch runs
 * temporally with the INFEASIBLE flag — VERBATIM_INFEASIBLE or FORCE_SPATIAL keep it spatial).
 * BOUNDARY_TBT (opt-in, reading #23): a candidate (S_d, k) must also keep the window-boundary gap
 * t_d + max(0, t_p - k t_d) <= tau (the paper constrains t_d only).
 * Errors: as duet_predict_latency, plus CONFIG for tbt_slo_s <= 0 or k_max < 1. */
duet_status duet_choose_split(const duet_model_spec* spec, const duet_hw_profile* hw,
                              const duet_req* batch, int32_t n, double tbt_slo_s, int32_t k_max,
                              uint32_t opts, duet_split* out);

/* f4 attention co-run choice of a temporal step (POD-Attention's overlap): the
 * prefill attention (F causal FLOPs) and the decode attention (B bytes) of one layer run either one
 * after the other on the full device, t_seq = F / fa(S) + B / bw(S), or side by side on the partition
 * (S - S_d, S_d), t = max(F / fa(S - S_d), B / bw(S_d)).  *s_d_out = the first candidate (ascending,
 * both sides >= min_sms) with the smallest t if that t < t_seq - overhead_s, else 0 (no co-run);
 * *t_out (nullable) = that t or t_seq.  fa_flops_at_sms / dec_bw_at_sms: [total_sms + 1] rates of the
 * library's prefill- and decode-attention kernels per partition size (duet_calibrate measures them
 * for the ctx; entries <= 0 are skipped).  Pure host function.
 * Errors: INVALID_ARG, CONFIG (full-device rate <= 0). */
typedef struct {
  int32_t total_sms, n_cand;
  const int32_t* cand_sd_sms;
  const double* fa_flops_at_sms;
  const double* dec_bw_at_sms;
  int32_t min_sms;
  double overhead_s;
} duet_corun_profile;
duet_status duet_corun_choose(const duet_corun_profile* p, double attn_flops_pre, double attn_bytes_dec,
                              int32_t* s_d_out, double* t_out);

/* ----------------------------------------------------------------- execution context */

typedef struct duet_ctx duet_ctx;

enum { DUET_DTYPE_BF16 = 0, DUET_DTYPE_FP32 = 1 };
enum {
  DUET_CTX_FINE_SPLIT = 1u,  /* 2-SM (TPC) partitions: CU_DEV_SM_RESOURCE_SPLIT_IGNORE_SM_COSCHEDULING;
                                default is the driver's 8-SM granularity (cuda.h green contexts) */
  DUET_CTX_NO_GRAPH = 2u,    /* launch decode kernels directly instead of replaying a CUDA graph */
  DUET_CTX_NO_CORUN = 4u,    /* temporal steps never co-run the prefill and decode attentions on an SM
                                split (f4; by default a measured-rate model decides per step, and the
                                environment variable DUET_CORUN=<S_d> / 0 forces / disables it) */
  DUET_CTX_NO_PREFILL_GRAPH = 8u /* spatial steps launch the prefill side's kernels one by one.  By default
                                the second spatial step with the same prefill shape (rows, sequences,
                                longest chunk, longest context, partition, buffers) captures the side's
                                L layers into a CUDA graph and later steps of that shape replay it
                                (prefill dispatch costs host time per kernel); at most 8 such
                                graphs are kept (LRU).  Never while live kernel timing is enabled. */
};

/* Capacity the workspace is sized for.  max_pos bounds every absolute token position
 * (RoPE table length).  dtype: element type of weights, activations and KV pools
 * (DUET_DTYPE_BF16 or DUET_DTYPE_FP32; fp32 runs SIMT kernels, bf16 tensor-core kernels). */
typedef struct {
  int32_t max_prefill_tokens, max_prefill_seqs, max_decode_reqs, max_k;
  int32_t max_pages_per_seq, max_pos;
  int32_t dtype;
  uint32_t flags;
} duet_ctx_limits;

/* Creates streams bound to disjoint SM partitions (green contexts: one pre-created pair per
 * achievable S_d — the pool P:112 describes), a full-device stream for temporal mode,
 * events, the RoPE table and the workspace.  device: CUDA ordinal.
 * Errors: INVALID_ARG, CONFIG (spec), UNSUPPORTED (head_dim, dtype), CUDA. */
duet_status duet_ctx_create(int32_t device, const duet_model_spec* spec,
                            const duet_ctx_limits* limits, duet_ctx** out);
duet_status duet_ctx_destroy(duet_ctx* ctx);

/* ----------------------------------------------------------------- iteration stream (§8(f) f2)
 * Host-side batch former + KV page allocator that turns a request trace into mixed iterations
 * (P:184 decode-first chunked prefill, P:302 R_prefill / R_decode, P:335 k-slot look-ahead; S:376
 * KV-capacity admission).  Deterministic, pure host, thread-compatible (one sched per thread).
 *  duet_sched_create: cfg = page size and pool size (pages), token budget per iteration (decode rows
 *    count one token each), max decode batch, max prefill sequences per iteration, k_max (look-ahead
 *    slots reserved per request), max pages per sequence (page-table pitch bound).
 *  duet_sched_add: a request (id, prompt and output length in tokens, arrival time, non-decreasing).
 *    CAPACITY if prompt + output + k_max tokens can never fit.
 *  duet_sched_next: forms the next iteration at time now_s: admits arrived requests FIFO while the
 *    free pages cover their whole prompt + output + k_max and the admitted, unfinished requests number
 *    fewer than max_batch; every running decode joins (so none is ever skipped), then prefill chunks
 *    fill the remaining budget, the oldest prompt first.  The arrays of
 *    *out (ids, q, c, page_table [n_prefill + n_decode][max_pages], prefill entries first) are owned by
 *    the sched and valid until the next call; an empty iteration (n_prefill = n_decode = 0) needs
 *    no commit — next_arrival_s says when the next request arrives (-1: none).
 *  duet_sched_commit: the iteration ran with k_done look-ahead decode steps (1 in temporal mode):
 *    prefill chunks advance (a completed prompt yields its first output token and joins the decodes),
 *    decodes produce min(k_done, remaining) tokens; finished requests return their pages.
 *    tokens_out: tokens produced (prefilled + generated); finished_out: requests completed.
 * Errors: INVALID_ARG (order of calls, ranges), OUT_OF_RANGE, CAPACITY. */
typedef struct {
  int32_t page_size, n_pages, token_budget, max_batch, max_prefill_seqs, k_max, max_pages_per_seq;
} duet_sched_cfg;
typedef struct {
  int32_t n_prefill, n_decode;
  const int64_t* ids;
  const int32_t* q;
  const int32_t* c;
  const int32_t* page_table;
  int32_t max_pages;
  double next_arrival_s;
  int32_t n_unfinished;
} duet_iteration;
typedef struct duet_sched duet_sched;
duet_status duet_sched_create(const duet_sched_cfg* cfg, duet_sched** out);
duet_status duet_sched_destroy(duet_sched* sched);
duet_status duet_sched_add(duet_sched* sched, int64_t id, int32_t prompt_len, int32_t output_len, double arrival_s);
duet_status duet_sched_next(duet_sched* sched, double now_s, duet_iteration* out);
duet_status duet_sched_commit(duet_sched* sched, int32_t k_done, int32_t* tokens_out, int32_t* finished_out);
duet_status duet_sched_free_pages(const duet_sched* sched, int32_t* out);

/* ----------------------------------------------------------------- tensor parallelism (§8 a9)
 * Head-sharded TP (reading #13).  A ctx created with spec->tp = N
 * computes the shard of rank r: h_q/N query heads, h_kv/N kv heads and ffn_dim/N FFN columns
 * (N must divide all three).  The caller passes that rank's weights to duet_step — w_qkv rows of
 * its q, k and v heads ([(h_q + 2 h_kv)/N d_h][d]), w_o columns of its q heads ([d][h_q/N d_h]),
 * w_gate_up rows [gate rows of its columns ; up rows] ([2 ffn_dim/N][d]), w_down columns
 * ([d][ffn_dim/N]); norm gains whole — and KV pools holding its kv heads ([n_pages][h_kv/N][P][d_h]).
 * The O and down projections then produce partial sums: rank 0 adds the residual and the
 * [rows][d] partials are all-reduced (sum) over NCCL right after each, on the side's own
 * communicator (decode and prefill/temporal sides run concurrently in spatial mode).
 *
 * duet_nccl_unique_id: an ncclUniqueId (128 bytes) into out (len >= 128); rank 0 creates two (one
 *   per side) and broadcasts them (e.g. with torch.distributed).
 * duet_ctx_set_comms: collective over the N ranks (each calls it with its rank and the same two
 *   ids): creates the ctx's decode-side and prefill-side communicators (ncclCommInitRankConfig with
 *   maxCTAs / nvlsCTAs capped — 4 on the decode side, 16 on the prefill side; env DUET_NCCL_MAXCTAS_DEC,
 *   DUET_NCCL_MAXCTAS_PRE, DUET_NCCL_NVLSCTAS — so a side's collectives stay a small share of its
 *   partition).  With spec->tp = 1 it creates single-rank communicators (the allreduce
 *   path, as a no-op copy).
 * duet_ctx_check_comms: polls ncclCommGetAsyncError on both communicators (NCCL if either reports an
 *   error; OK without communicators); duet_step does the same before it enqueues work on a TP ctx.
 * duet_calibrate_allreduce: alpha (s) and B_NVLink (B/s) of the P:237 ring model from timed
 *   allreduces of 16 B and 64 MiB on the prefill communicator (0, 0 when tp = 1).
 * libnccl.so.2 is resolved at run time (the one PyTorch loads).  Errors: INVALID_ARG,
 * OUT_OF_RANGE (rank), NCCL, CUDA. */
duet_status duet_nccl_unique_id(void* out, int32_t len);
duet_status duet_ctx_set_comms(duet_ctx* ctx, int32_t rank, const void* id_decode, const void* id_prefill);
duet_status duet_calibrate_allreduce(duet_ctx* ctx, double* alpha_s, double* bw_bytes_s);
duet_status duet_ctx_check_comms(duet_ctx* ctx);
/* 1 if the last temporal duet_step ran a layer's two attentions as the fused POD launch (SURVEY §8(f) f4,
 * prefill-attention and decode-attention CTAs in one grid instead of the green-context co-run;
 * opt-in with DUET_POD=1, used whenever the co-run model splits the step), else 0. */
int32_t duet_ctx_last_pod(duet_ctx* ctx);

/* ----------------------------------------------------------------- fused GEMM + allreduce (f3)
 * SURVEY §8(f) f3; P:233-236 (§4.1 Communication Operators: in a head-sharded TP block the O and FFN-down
 * outputs are partial sums over the N ranks, followed by an allreduce of the [n][d] rows, twice per
 * layer).  The row-parallel projection and its allreduce run as ONE CTA-pair tcgen05 kernel: the
 * epilogue of each 256 x 256 output tile t pushes the fp32 partial over peer memory (NVLink) into the
 * receive slot of the tile's owner rank t mod N and releases an arrival counter there; the owner sums the
 * N partials in rank order 0..N-1 (its own straight from TMEM), adds the residual, rounds once to bf16
 * and stores the rows into every rank's output (all-gather by push), releasing each rank's completion
 * counter.  Communication overlaps the remaining tiles' MMAs; no NCCL kernel runs in the partition.
 * Every wait polls local memory; every remote access is a store or a release-add; counters are re-armed
 * by their waiters, so a launch or a CUDA-graph replay needs no epoch.
 *
 * duet_ctx_ar_handle: allocates (once) the ctx's fused-allreduce arena — per side the receive slots, the
 *   counters and two [rows][d] bf16 outputs, sized from the limits — and writes its cudaIpcMemHandle_t
 *   (64 bytes) to out (len >= 64).  Needs duet_ctx_set_comms first (rank, group).  Every rank must have
 *   created its ctx with the same spec and limits (the arenas share one layout).
 * duet_ctx_ar_open: handles = [n][64] bytes, every rank's handle in rank order (an all-gather of
 *   duet_ctx_ar_handle); maps the peers' arenas (cudaIpcOpenMemHandle).  From then on duet_step runs the
 *   O and down projections of every > 128-row batch (the prefill side; temporal steps; a > 128-row decode
 *   side) through the fused kernel; batches of <= 128 rows keep the NCCL allreduce.  Every rank calls it
 *   before any rank's next duet_step.  With tp = 1 the kernel is the plain residual GEMM (bitwise).
 *   Errors: INVALID_ARG (no comms / no arena / n != tp / already open), CUDA (IPC).
 * duet_op_gemm_ar_emul: the fused kernel with n_ranks ranks (1..8) EMULATED in one grid on this GPU
 *   (each rank on total_sms / 2 / n_ranks CTA pairs, all resident: ranks that wait on one another must
 *   share a launch when there are fewer GPUs than ranks).  A: [n_ranks][M][K], B: [n_ranks][N][K]
 *   (rank r's shards stacked), R: [M][N], C: [n_ranks][M][N] (every rank's output); each must equal
 *   R + sum_r A_r B_r^T, and all ranks' outputs are bitwise equal.  M > 128, N % 32 == 0, K % 64 == 0,
 *   bf16 ctx, device pointers, 16-byte aligned.  Errors: INVALID_ARG, OUT_OF_RANGE, UNSUPPORTED, CUDA. */
duet_status duet_ctx_ar_handle(duet_ctx* ctx, void* out, int32_t len);
duet_status duet_ctx_ar_open(duet_ctx* ctx, int32_t n, const void* handles);
duet_status duet_op_gemm_ar_emul(duet_ctx* ctx, int32_t n_ranks, const void* A, const void* B, const void* R,
                                 void* C, int32_t M, int32_t N, int32_t K, void* stream);

/* The achievable decode-partition sizes, ascending (host array of capacity *n on input;
 * *n is set to the count).  total_sms: SMs of the device. */
duet_status duet_ctx_partitions(duet_ctx* ctx, int32_t* sd_sms, int32_t* n, int32_t* total_sms);

/* Per-layer weights, all device, dtype of the ctx, nn.Linear layout [out][in] (K-major):
 *  w_qkv [(h_q + 2 h_kv) d_h][d] (rows: q heads, k heads, v heads; reading #4)
 *  b_qkv [(h_q + 2 h_kv) d_h] or NULL;  w_o [d][h_q d_h];
 *  w_gate_up [2m][d] (rows: gate(m) then up(m); reading #3);  w_down [d][m];
 *  g_norm1, g_norm2 [d] (RMSNorm gains; reading #1). */
typedef struct {
  const void *w_qkv, *b_qkv, *w_o, *w_gate_up, *w_down, *g_norm1, *g_norm2;
} duet_layer_weights;

/* Prefill side (R_prefill): n_seqs sequences, rows grouped by sequence in order.
 *  q, c: host [n_seqs] new / cached tokens; sequence s occupies positions c[s]..c[s]+q[s]-1.
 *  page_table: host [n_seqs][max_pages] int32 pool pages; must cover c+q tokens.
 *  x: device [sum q][d] input rows; y: device [sum q][d] output rows (last layer). */
typedef struct {
  int32_t n_seqs;
  const int32_t* q;
  const int32_t* c;
  const int32_t* page_table;
  int32_t max_pages;
  const void* x;
  void* y;
} duet_prefill;

/* Optional LM head of the decode side (P:250 t_cls, P:335 sampled tokens): after
 * the last layer of every decode step, h = RMSNorm(y) * g_norm, logits = h . w_head^T (bf16, fp32
 * accumulation), token = argmax (greedy; the lowest index among equal maxima), and the next step's
 * input is embed[token] instead of y (closing the look-ahead window into an autoregressive loop).
 *  g_norm: device [d]; w_head: device [vocab][d] (nn.Linear layout); embed: device [vocab][d];
 *  tokens: device int32 [k][n_reqs] output.  All of the ctx dtype, vocab = spec->vocab; bf16 ctx only. */
typedef struct {
  const void* g_norm;
  const void* w_head;
  const void* embed;
  int32_t* tokens;
} duet_lm_head;

/* Decode side (R_decode) for a look-ahead window of k steps.
 *  c: host [n_reqs] cached tokens before step 1; step j (1..k) is at position c + j - 1.
 *  page_table: host [n_reqs][max_pages]; must cover c + k tokens (look-ahead slots).
 *  x: device [n_reqs][d] step-1 input; y: device [k][n_reqs][d] per-step last-layer outputs.
 *  head == NULL: step j>1 takes step j-1's last-layer output as input (synthetic feedback,
 *  reading #26); otherwise the greedy token's embedding (duet_lm_head). */
typedef struct {
  int32_t n_reqs;
  const int32_t* c;
  const int32_t* page_table;
  int32_t max_pages;
  const void* x;
  void* y;
  const duet_lm_head* head;
} duet_decode;

/* Paged KV cache (vLLM-style pages).  k_pool / v_pool: host arrays of
 * n_layers device pointers, each pool [n_pages][h_kv][page_size][d_h] of the ctx dtype.
 * slot(r, p) = (page_table[r][p / page_size], p % page_size) (C-3).  Pages must be distinct
 * within and across all requests of one call and < n_pages.  page_size must be 16. */
typedef struct {
  void* const* k_pool;
  void* const* v_pool;
  int32_t n_pages;
  int32_t page_size;
} duet_kv_pages;

/* One mixed serving iteration (the hot path).
 *  split->mode == TEMPORAL: GPU_temporal_sharing_execute (Alg. 1 l.4): one full-device
 *    stream runs the layer stack over the concatenated rows [prefill ; decode], k = 1.
 *  split->mode == SPATIAL: GPU_spatial_sharing_execute (Alg. 1 l.22, §4.3): the decode side
 *    runs k steps on the S_d-SM partition (launched first, as replays of a captured CUDA
 *    graph) while the prefill side runs on the remaining S_p SMs; both join on an
 *    event.  split->s_d must be one of duet_ctx_partitions.
 *  pre or dec may be NULL (or have 0 rows).  w: host array of n_layers weight sets.
 *  stream: the caller's cudaStream_t (NULL = legacy default stream).  All work is ordered
 *  after work already on `stream`, and `stream` waits for the step's completion: the call
 *  is asynchronous and never synchronizes the host.
 * Errors: INVALID_ARG, OUT_OF_RANGE (page tables, s_d not achievable), CAPACITY (limits),
 *         CUDA. */
duet_status duet_step(duet_ctx* ctx, const duet_layer_weights* w, const duet_prefill* pre,
                      const duet_decode* dec, const duet_kv_pages* kv, const duet_split* split,
                      void* stream);

/* Device-measured times of the last completed duet_step (CUDA events on the partition
 * streams; requires the step to have completed, e.g. after synchronizing `stream`).
 * Times in seconds: t_window = first launch -> join; t_decode = decode side (k steps);
 * t_prefill = prefill side.  Temporal: t_window = t_decode = t_prefill.  corun_s_d: SMs of the
 * decode group the two attentions of a temporal step co-ran on (f4; 0 = one after the other). */
typedef struct {
  double t_window, t_decode, t_prefill;
  int32_t mode, k, kernels, corun_s_d;
  int32_t prefill_graph; /* spatial: 1 if the prefill side replayed a captured graph (DUET_CTX_NO_PREFILL_GRAPH) */
} duet_step_times;
duet_status duet_last_step_times(duet_ctx* ctx, duet_step_times* out);

/* Measures Pi_SM(S) and B_HBM(S) for S = every partition size the ctx can provision (both
 * sides of every split, and the full device) with the library's own kernels, the recipe of
 * B_HBM(S) is the HBM bandwidth the library's memory-bound hot kernel (paged decode
 * attention, bf16; 64 requests whose K/V pages fill a >= 512 MiB buffer) achieves on S SMs — fp32
 * contexts use an 8 KiB-page cp.async streaming kernel — and Pi_SM(S) is the rate of a GEMM with the
 * model's gate-up shape (M = max_prefill_tokens clamped to 256..8192, N = 2 ffn_dim, K = d_model).
 * flops_at_sms / bw_at_sms: host arrays of total_sms+1 doubles; entries for sizes that
 * cannot be provisioned are filled by linear interpolation between measured neighbours.
 * Errors: INVALID_ARG, CUDA. */
duet_status duet_calibrate(duet_ctx* ctx, double* flops_at_sms, double* bw_at_sms, int32_t len);

/* duet_calibrate with the co-run, sustained refinement (reading R-f of DESIGN.md, "achievable"):
 * after the standalone pass and about a second of full-device GEMMs (the clocks settle at the power
 * cap), every split (S_d, S_p) runs two phases of ~pair_seconds each — the calibration GEMM on S_p while
 * the paged decode attention streams on S_d (-> flops_at_sms[S_p], bw_at_sms[S_d]), then the roles
 * swapped (-> flops_at_sms[S_d], bw_at_sms[S_p]); the full device runs each kernel alone, sustained.
 * Rates over launches 40-90 % of each side's loop, then smoothed over the measured sizes
 * (duet_profile_smooth).  Falls back to duet_calibrate's tables where a
 * size was not measured this way (fp32 contexts).  ~2 * n_partitions * pair_seconds + ~1.5 s.
 * Errors: as duet_calibrate, INVALID_ARG for pair_seconds <= 0. */
duet_status duet_calibrate_corun(duet_ctx* ctx, double* flops_at_sms, double* bw_at_sms, int32_t len,
                                 double pair_seconds);

/* Smooths one calibration table in place (reading R-g; duet_calibrate_corun applies it to both of its
 * tables over the sizes it measured): at the measured sizes (strictly ascending, 0 < size < len) the
 * per-SM rate rate[S]/S of every interior size becomes the median of its own and its two neighbours'
 * per-SM rates; the end points are kept.  Monotone runs of per-SM rates are left unchanged; one
 * outlying measurement (a 0.1-s phase on a power-capped GPU) is replaced.  Host-only.
 * Errors: INVALID_ARG (NULL, n < 0), OUT_OF_RANGE (sizes), CONFIG (a rate <= 0). */
duet_status duet_profile_smooth(const int32_t* sizes, int32_t n, double* rate_at_sms, int32_t len);

/* The hardware read-stream ceiling per partition size — the roofline denominator of a decode
 * partition, SURVEY §8(d) (not a predictor input): plain 16-byte LDG streaming of a >= 256 MiB buffer
 * from 2048 threads per SM on S SMs (median of 5), for S = every achievable partition side and the
 * full device; other entries 0.  bw_stream: host array of len >= total_sms + 1 doubles (B/s).
 * Errors: INVALID_ARG, CAPACITY, CUDA. */
duet_status duet_calibrate_stream(duet_ctx* ctx, double* bw_stream, int32_t len);

/* Live kernel timing (measurement, §8(d)): while enabled, duet_step records CUDA events on the
 * launching stream around every kernel it launches, per kernel class, together with the
 * algorithmic FLOPs and bytes of each launch (causal attention FLOPs,
 * weights/activations read once).  duet_profile_enable(ctx, mask) resets the counters and times the
 * classes whose bit (1 << DUET_KCLASS_*) is set in mask (0 = off; DUET_PROFILE_ALL = every class);
 * each timed launch costs two event records on its stream (~1 us), so a timed region usually enables
 * only the class it reports.  duet_profile_read synchronizes on the recorded events and returns
 * DUET_KCLASS_N entries. */
/* GEMM / OTHER count the prefill side of a spatial step and every kernel of a temporal step;
 * GEMM_DECODE / OTHER_DECODE the decode side of a spatial step.  Event-timed kernels are never inside
 * a CUDA graph: while GEMM_DECODE or OTHER_DECODE is enabled the decode side launches its kernels one
 * by one, while a prefill-side class is enabled the prefill side does.  DECODE_ATTN alone keeps the
 * decode graph: the graph is captured with a device-side timer in the decode-attention kernel (the
 * earliest CTA start to the latest CTA end of every launch, %globaltimer; the split-K combine, when
 * the batch splits, is not included), read by duet_profile_read. */
enum { DUET_KCLASS_GEMM = 0, DUET_KCLASS_PREFILL_ATTN = 1, DUET_KCLASS_DECODE_ATTN = 2, DUET_KCLASS_OTHER = 3,
       DUET_KCLASS_GEMM_DECODE = 4, DUET_KCLASS_OTHER_DECODE = 5, DUET_KCLASS_N = 6 };
#define DUET_PROFILE_ALL 0x3F
typedef struct { int32_t launches; double seconds, flops, bytes; } duet_kernel_stats;
duet_status duet_profile_enable(duet_ctx* ctx, int32_t class_mask);
duet_status duet_profile_read(duet_ctx* ctx, duet_kernel_stats* out);

/* ----------------------------------------------------------------- single operators
 * The kernels of duet_step, exposed for parity tests and microbenchmarks.  All pointers are
 * device; dtype is the ctx dtype; launched on `stream` over the full device. */

/* C[M][N] = epilogue(A[M][K] . B[N][K]^T); epi: 0 store (+ bias[N] if bias), 1 residual
 * C = R + acc, 2 SwiGLU: B has 2N rows [gate; up], C[m][j] = silu(acc_g) * acc_u. */
enum { DUET_EPI_STORE = 0, DUET_EPI_RESIDUAL = 1, DUET_EPI_SWIGLU = 2 };
duet_status duet_op_gemm(duet_ctx* ctx, const void* A, const void* B, void* C, const void* R,
                         const void* bias, int32_t M, int32_t N, int32_t K, int32_t epi,
                         void* stream);

/* h[n][d] = x * (mean(x^2) + eps)^(-1/2) * g   (reading #1). */
duet_status duet_op_rmsnorm(duet_ctx* ctx, const void* x, const void* g, void* h, int32_t n,
                            void* stream);

/* Paged decode attention alone (a5.4: split-K over pages + log-sum-exp combine, exactly the launch
 * duet_step makes), for parity checks at full size and partition microbenchmarks.
 *  q: device [n] rows of row stride q_stride elements (>= h_q d_h), head j at column j d_h, already
 *  rotated; o: device [n][h_q d_h].  Row r attends to positions 0..pos[r] of page-table row r
 *  (readings #2, #6, #7); their K/V must already be in the pools (no append).
 *  pos: host int32 [n]; page_table: host int32 [n][max_pages], covering pos + 1 tokens, pages distinct.
 *  k_pool / v_pool: device [n_pages][h_kv][16][d_h] of one layer.  s_d: 0 = full device on `stream`,
 *  else the decode group of the partition with s_d SMs (duet_ctx_partitions), ordered after and
 *  joined back into `stream`.  n <= max_decode_reqs, pos < max_pos.
 * Errors: INVALID_ARG, OUT_OF_RANGE (pages, positions, s_d), CAPACITY, UNSUPPORTED, CUDA. */
duet_status duet_op_decode_attn(duet_ctx* ctx, const void* q, int32_t q_stride, void* o, int32_t n,
                                const int32_t* pos, const int32_t* page_table, int32_t max_pages,
                                const void* k_pool, const void* v_pool, int32_t n_pages, int32_t s_d,
                                void* stream);

/* Causal prefill attention alone (a6.4, the launch of duet_step): n_seqs sequences, sequence s has
 * q_len[s] query rows (rows grouped by sequence in order) at positions c[s] .. c[s] + q_len[s] - 1 and
 * attends to every position <= its own (the prefix fully, reading #7); K/V of all those positions
 * must already be in the pools.  q: device [sum q_len] rows of stride q_stride; o: device
 * [sum q_len][h_q d_h].  q_len, c: host int32 [n_seqs]; page_table: host [n_seqs][max_pages].
 *  s_p: 0 = full device, else the prefill side (remainder) of the partition with that many SMs.
 * Errors: as duet_op_decode_attn. */
duet_status duet_op_prefill_attn(duet_ctx* ctx, const void* q, int32_t q_stride, void* o, int32_t n_seqs,
                                 const int32_t* q_len, const int32_t* c, const int32_t* page_table,
                                 int32_t max_pages, const void* k_pool, const void* v_pool, int32_t n_pages,
                                 int32_t s_p, void* stream);

/* Token times (TBT per decode step, the window-boundary gap): every decode step of a
 * spatial window, and the decode rows of a temporal step, write %globaltimer (ns, one device-wide
 * clock) into a 4096-slot device ring when that step's tokens are complete, in stream order.
 * duet_token_times synchronizes the device, returns the number of stamps written since the last reset
 * in *n and copies the first min(*n, cap) of them to out_ns (both nullable), then clears the ring
 * when reset != 0.  Consecutive stamps of one decode batch are its inter-token gaps, including the
 * gap across a window boundary.  Errors: INVALID_ARG, CAPACITY (> 4096 stamps since the reset), CUDA. */
duet_status duet_token_times(duet_ctx* ctx, int32_t reset, uint64_t* out_ns, int32_t cap, int32_t* n);

#ifdef __cplusplus
}
#endif

#endif /* DUET_H */

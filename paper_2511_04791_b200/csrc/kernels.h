// Internal launcher interface between the step orchestration (duet_ctx.cu) and the sm_100a
// kernels (kernels_*.cu).  Not part of the C ABI.
#pragma once
#include <cuda_runtime.h>
#include <cstdint>

namespace duet {

enum class DT : int { BF16 = 0, F32 = 1 };

inline size_t dt_size(DT t) { return t == DT::BF16 ? 2 : 4; }

// ---------------------------------------------------------------- GEMM
// C[M][N] (ldc) = epi(A[M][K] (lda) . B[N][K]^T (ldb)).  Both operands K-major (nn.Linear).
//  EPI_STORE:    C = acc (+ bias[n])
//  EPI_RESIDUAL: C = R[m][n] (ldr) + acc
//  EPI_SWIGLU:   B has rows [gate(N) ; up(N)] (gate row j at j, up row j at N + j);
//                C[m][j] = silu(acc_gate) * acc_up
//  EPI_QKV_ROPE: C = acc (+ bias) for the q heads after RoPE; k heads (RoPE) and v heads are written to
//                their paged KV slots instead (QKV GEMM + RoPE + KV append fused; CTA-pair kernel only)
//  EPI_RESIDUAL_AR: row-parallel GEMM + allreduce fused: every rank's
//                C = R + sum over the tp ranks of their A_r . B_r^T; the partial tiles are exchanged
//                inside the epilogue over peer memory (GemmAr; CTA-pair kernel only)
enum { EPI_STORE = 0, EPI_RESIDUAL = 1, EPI_SWIGLU = 2, EPI_QKV_ROPE = 3, EPI_RESIDUAL_AR = 4 };

// Fused GEMM + allreduce (EPI_RESIDUAL_AR).  Each 256 x 256 output tile has one owner rank (rotating along
// every CTA pair's tile sequence, identical on all ranks).  Every non-owner pushes its fp32 partial tile into the owner's receive
// slot and releases a per-(tile, warp) arrival counter there; the owner sums the n partials in rank order
// 0..n-1 (its own from TMEM), adds R, rounds once to bf16 and stores the rows into every rank's output
// (all-gather by push), releasing each rank's completion counter; one CTA per rank waits for its
// completion counter before the grid ends.  All waits poll local memory; every remote access is a
// store or a release-add.  Counters are reset by their waiter, so a launch (or a graph replay) needs no
// epoch.  Pointers of rank r: on a real TP group peer-mapped (cudaIpc), for emulation local buffers.
constexpr int kMaxTp = 8;
struct GemmAr {
  int n = 1;              // ranks (<= kMaxTp)
  int rank = 0;           // this rank (emul = 0)
  int emul = 0;           // 1: all n ranks run in this one grid (one GPU; A / B stacked per rank)
  float* slots[kMaxTp];   // rank r's receive slots [owned tile][sender][256 cols][256 rows] fp32
  void* out[kMaxTp];      // rank r's output C (same pitch ldc on every rank)
  unsigned* cnt[kMaxTp];  // rank r's arrival counters [owned tile][8], zero between launches
  unsigned* done[kMaxTp]; // rank r's completion counter, zero between launches
  size_t slot_tiles = 0;  // owned-tile capacity of every rank's slots / counters (gemm_ar_slot_tiles)
};
// owned-tile slots, receive-slot floats and counters one rank needs for an M x N output over n ranks on
// any grid of <= num_sms / 2 CTA pairs
size_t gemm_ar_slot_tiles(int M, int N, int n, int num_sms);
size_t gemm_ar_slot_floats(int M, int N, int n, int num_sms);
size_t gemm_ar_counters(int M, int N, int n, int num_sms);

struct GemmArgs {
  const void* A;
  const void* B;
  void* C;
  const void* R;
  const void* bias;
  int M, N, K;
  int lda, ldb, ldc, ldr;
  int epi;
  // split-K workspace (fp32 partials) for weight-streaming (swap-AB) launches; nullptr -> no split-K.
  // A split launch is two kernels (GEMM writing partials, then an ordered reduction + epilogue).
  float* ws = nullptr;
  size_t ws_floats = 0;
  // rows >= row_split read the residual from R2 and store to C2 (row - row_split), same pitches: the
  // temporal batch [prefill rows ; decode rows] without copying it between the caller's buffers
  // (CTA-pair kernel only; kernels.h gemm2_supported)
  const void* R2 = nullptr;
  void* C2 = nullptr;
  int row_split = 1 << 30;
  // EPI_QKV_ROPE: the RoPE / KV-append operands (kernels.h RopeKvArgs; head_dim 128, page size 16)
  const struct RopeKvArgs* rope = nullptr;
  // EPI_RESIDUAL_AR: the tp group (C is ignored: outputs go to ar->out[r])
  const struct GemmAr* ar = nullptr;
  // nullable device int: the rows of this launch, read on the device (M is then the buffers' capacity;
  // CTA-pair kernel only, never split-K) — graphs that replay for any row count (f4)
  const int* m_dev = nullptr;
};
// fp32 partial floats a split-K launch of this shape needs (0 when it runs unsplit)
size_t gemm_tc_splitk_need(int M, int N, int K, int epi);
// fp32 partial floats a CTA-pair (M > 128) launch of this shape needs (0 when it runs unsplit)
size_t gemm2_splitk_need(int M, int N, int K, int epi);

// num_sms: SMs of the partition the launch runs in (persistent grid sizing).
// Returns the number of kernels launched (0 on a launch error, checked by the caller).
int launch_gemm(DT dt, const GemmArgs& a, int num_sms, cudaStream_t st);
int launch_gemm_simt(DT dt, const GemmArgs& a, cudaStream_t st);
int launch_gemm_tc(const GemmArgs& a, int num_sms, cudaStream_t st);
bool gemm_tc_supported(const GemmArgs& a);
// CTA-pair (cta_group::2) 256x256 tiles for M > 128 on partitions of >= 2 SMs (kernels_gemm2.cu)
bool gemm2_supported(const GemmArgs& a, int num_sms);
int launch_gemm2(const GemmArgs& a, int num_sms, cudaStream_t st);

// ---------------------------------------------------------------- RMSNorm
// h[n][d] = x * rsqrt(mean(x^2) + eps) * g     (reading #1)
int launch_rmsnorm(DT dt, const void* x, const void* g, void* h, int n, int d, float eps, cudaStream_t st,
                   const void* x2 = nullptr, int row_split = 1 << 30,  // rows >= row_split from x2
                   const int* n_dev = nullptr);  // nullable: rows on the device (n is then the capacity)

// ---------------------------------------------------------------- RoPE + paged KV append
// qkv rows [n][(hq + 2 hkv) dh]; row i at position pos[i], page-table row tok_row[i].
// q heads are rotated in place; rotated k and v go to slot (table[row][p/P], p%P) of the
// layer's pools [n_pages][hkv][P][dh].  rope: [max_pos][dh/2] float2 (cos, sin).
struct RopeKvArgs {
  void* qkv;
  const void* bias;  // [(hq + 2 hkv) dh] or nullptr: added before rotation
  int n, hq, hkv, dh;
  const int* pos;
  const int* tok_row;
  const int* table;
  int max_pages, page_size;
  void* k_pool;
  void* v_pool;
  const float2* rope;
};
int launch_rope_kv(DT dt, const RopeKvArgs& a, cudaStream_t st);

// ---------------------------------------------------------------- decode attention
// o[r][hq*dh] = softmax(q_r . K / sqrt(dh)) . V over positions 0..pos[r] of request r
// (tok_row[r] selects its page-table row).  Split-K over pages with an LSE combine.
struct DecodeAttnArgs {
  const void* q;  // row stride q_stride (elements); head j at column j*dh
  int q_stride;
  void* o;        // [n][hq*dh]
  int n, hq, hkv, dh;
  const int* pos;
  const int* tok_row;
  const int* table;
  int max_pages, page_size;
  const void* k_pool;
  const void* v_pool;
  float* part_o;    // workspace [n][hq][max_splits][dh]
  float* part_ml;   // workspace [n][hq][max_splits][2]
  int max_splits;
  int num_sms;
  int max_len;      // upper bound of pos[r] + 1 over the batch (host-known), for split sizing
  int n_pages;      // pool extent (TMA maps)
  // device-side launch timing (live kernel timing inside CUDA graphs): [0] earliest CTA start,
  // [1] latest CTA end (%globaltimer ns), [2] CTAs done, [3] sum of launch durations (ns), [4] launches;
  // the last CTA of a launch adds end - start to [3] and re-arms [0..2].  nullptr = off.
  unsigned long long* dev_timer = nullptr;
  // nullable device [n]: the request each CTA column z takes (longest first: a shorter last wave); the
  // results do not depend on it (every request is computed by its own CTAs)
  const int* order = nullptr;
};
int launch_decode_attn(DT dt, const DecodeAttnArgs& a, cudaStream_t st);
bool decode_tc_supported(const DecodeAttnArgs& a);
int launch_decode_tc(const DecodeAttnArgs& a, int pages_per_split, int n_splits, cudaStream_t st);

// ---------------------------------------------------------------- prefill attention
// Causal attention of the chunk rows over prefix + chunk (reading #7): sequence s has rows
// [row0[s], row0[s] + qlen[s]) at positions cpre[s] + i and reads KV from page-table row
// seq_row[s]; the chunk's own K/V are already in the pages.
struct PrefillAttnArgs {
  const void* q;
  int q_stride;
  void* o;
  int n_seqs, hq, hkv, dh;
  const int* row0;
  const int* qlen;
  const int* cpre;
  const int* seq_row;
  const int* table;
  int max_pages, page_size;
  const void* k_pool;
  const void* v_pool;
  int max_q;   // host-known max qlen (grid sizing)
  int total_q; // host-known sum of qlen
  int num_sms;
  // per-row view (SIMT path): row i at position tok_pos[i], page-table row tok_row[i]
  const int* tok_pos;
  const int* tok_row;
  int max_len;  // host-known max(c + q) over the sequences
  // tensor-core path: pool extent and rows of the q buffer (TMA maps)
  int n_pages;
  int total_rows;
  // nullable device [rows, sequences, longest chunk]: a launch sized for the capacity (n_seqs, max_q) reads
  // the step's own shape (shape-agnostic prefill graphs, f4; tcgen05 kernel)
  const int* shape_dev = nullptr;
};
int launch_prefill_attn(DT dt, const PrefillAttnArgs& a, cudaStream_t st);
bool fa_prefill_supported(const PrefillAttnArgs& a);
int launch_fa_prefill(const PrefillAttnArgs& a, cudaStream_t st);
bool fa_tc_supported(const PrefillAttnArgs& a);
int launch_fa_tc(const PrefillAttnArgs& a, cudaStream_t st);
// POD-style fused prefill + decode attention (f4, kernels_pod.cu): one launch, the first CTAs run the
// persistent tcgen05 prefill attention, the last n_dec_ctas the paged decode attention (+ the LSE combine
// as a second kernel when the batch splits); bf16, d_h 128.  Returns kernels launched, < 0 if unsupported.
int launch_pod_attn(DT dt, const PrefillAttnArgs& pa, const DecodeAttnArgs& da, int n_dec_ctas, cudaStream_t st);
int launch_pod_tc(const PrefillAttnArgs& pa, const DecodeAttnArgs& da, int pps, int n_splits, int n_dec_ctas,
                  cudaStream_t st);
// CTA-pair (cta_group::2) version, opt-in with DUET_FA2=1 (measured slower than the one-CTA kernel)
bool fa2_tc_supported(const PrefillAttnArgs& a);
int launch_fa2_tc(const PrefillAttnArgs& a, cudaStream_t st);

// ---------------------------------------------------------------- decode window bookkeeping
// End of one decode step (P:335 look-ahead): y_out[step][r] = y[r]; xin[r] = y[r];
// pos[r] += 1; step += 1.  Reads *step on device so a captured graph can be replayed k times.
// greedy token of each row's bf16 logits [n][vocab] -> tokens[(step ? *step : 0) * n + r]; x_next[r] =
// embed[token] (x_next may be NULL)
int launch_argmax_embed(const void* logits, int vocab, const void* embed, void* x_next, int d, int* tokens,
                        const int* step, int n, cudaStream_t st);
// ts / ts_cnt (nullable): token-time ring of kTokTsSlots %globaltimer stamps; the bump kernel of every step
// writes slot (*ts_cnt)++ (the time the step's tokens are complete).  launch_stamp writes one stamp.
constexpr int kTokTsSlots = 4096;
int launch_decode_advance(DT dt, const void* y, void* xin, void* y_out, int n, int d, int* pos, int* step,
                          cudaStream_t st, unsigned long long* ts = nullptr, int* ts_cnt = nullptr);
int launch_stamp(unsigned long long* ts, int* cnt, cudaStream_t st);

// Streaming-read kernel for B_HBM(S) calibration: reads n_bytes, writes one word per CTA.
int launch_stream_read(const void* buf, size_t n_bytes, unsigned long long* sink, int num_sms, cudaStream_t st);
int launch_stream_pages(const void* buf, size_t n_bytes, unsigned long long* sink, int num_sms, cudaStream_t st);
// hashed values in [-1, 1) (calibration operands)
int launch_fill_hash(DT dt, void* p, size_t n_elems, uint32_t seed, cudaStream_t st);
// dst <- src on the SMs (src may be mapped pinned host memory: zero-copy over PCIe); no copy engine
int launch_copy_bytes(void* dst, const void* src, size_t bytes, int num_sms, cudaStream_t st);

}  // namespace duet

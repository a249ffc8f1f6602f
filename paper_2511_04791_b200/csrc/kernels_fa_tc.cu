// Causal prefill attention over the paged KV cache on 5th-generation tensor cores (tcgen05 / TMEM).
//
// Chunked prefill (§4.1; readings #2, #6, #7): a chunk of q tokens at positions
// c..c+q-1 attends to its c-token prefix and to itself causally.  One CTA = the same 128 query rows
// of TWO query heads of one GQA group (reading #6: they read the same kv head), so every K/V tile is
// gathered once for two score tiles; keys stream in 128-key tiles (8 pages of 16 tokens), so the
// score MMA is 128x128x16 (an N = 64 UMMA reads 6 KiB of operands for half the work and runs at ~44%
// of the tensor rate, N = 128 at ~88%: profiles/r01_probe_umma_rate.txt).
//   warp 0        Q tiles by TMA (2 heads x two 64-column SWIZZLE_128B boxes)
//   warp 1        TMEM allocator (all 512 columns: per head S_j/P_j 128 | O 128) + tcgen05.mma issuer,
//                 per head: PV_j (A = P_j straight from TMEM, B = V from smem, MN-major), then
//                 S_{j+1} = Q K_{j+1}^T over the same TMEM columns (MMAs execute in issue order)
//   warps 2..5    softmax of head A, one thread per query row (= TMEM lane): two passes over the 128
//                 S columns (max, then exp2 -> bf16 P written in place with tcgen05.st) — no
//                 shared-memory round trip, no proxy fence
//   warps 6..9    softmax of head B — each SM sub-partition runs one warp of each head, so one head's
//                 exp work overlaps the other head's MMAs
//   warps 10..13  loaders (2 warps per tensor): cp.async gathers of the scattered 4 KiB page blocks
//                 into a 2-stage K ring and a 3-stage V ring, each thread's copies tracked by the stage
//                 mbarrier (cp.async.mbarrier.arrive.noinc); a TMA box costs its issuing thread
//                 ~0.25 us on B200 (profiles/r01_probe_tma_bw.txt) and a page would need four
// The running max is re-based (O rescaled in TMEM) only when it grows by more than 2^8; the decision is
// taken per warp because tcgen05.ld/st are warp-collective.  Keys past the causal end of a tile are
// zero-filled (cp.async src-size 0) and masked.  An odd last head of a group runs alone (has_b = 0).
#include <cuda.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "dev_common.cuh"
#include "kernels.h"

namespace duet {
namespace fatc {

constexpr int BQ = 128, BKV = 128, DH = 128, PAGE = 16;
constexpr int Q_SUB = BQ * 128;            // [128 rows][64 cols] SW128 sub-tile = 16 KiB
constexpr int KV_SUB = BKV * 128;          // [128 keys][64 cols] = 16 KiB
constexpr int Q_BYTES = 2 * Q_SUB;         // 32 KiB per head
constexpr int KV_BYTES = 2 * KV_SUB;       // 32 KiB per tensor per stage
constexpr int OFF_Q = 0;                   // head A, head B
constexpr int OFF_K = OFF_Q + 2 * Q_BYTES;
// K ring KS stages, V ring VS stages (the Q tiles take 64 KiB, so KS + VS <= 5)
template <int KS, int VS> struct Ring {
  static constexpr int OFF_V = OFF_K + KS * KV_BYTES;
  static constexpr int OFF_BAR = OFF_V + VS * KV_BYTES;
  static constexpr int OFF_TRACE = OFF_BAR + 256;   // DUET_FA_TRACE: per-tile clock stamps of CTA (0,0,0)
  static constexpr int SMEM = OFF_TRACE + 10 * 16 * 4 + 1024;
  static_assert(SMEM <= 227 * 1024, "smem");
  
};
constexpr int TRACE_EV = 10, TRACE_MAXJ = 16;

constexpr int THREADS = 14 * 32;
constexpr int TMEM_COLS = 512;             // per head: S_j / P_j (128) | O (128)
constexpr float RESCALE_THRESHOLD = 8.0f;  // log2 domain

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(const CUtensorMap* map, uint64_t* bar, void* dst, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
          smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1)
      : "memory");
}
// K-major SW128 descriptor (rows of 128 B, 8-row atoms of 1 KiB): LBO unused (1), SBO = 1 KiB
__device__ __forceinline__ uint64_t desc_k(uint32_t saddr) {
  return (uint64_t)((saddr & 0x3FFFF) >> 4) | ((uint64_t)1 << 16) | ((uint64_t)64 << 32) | ((uint64_t)1 << 46) |
         ((uint64_t)2 << 61);
}
// MN-major SW128 descriptor: 64-element MN blocks LBO = KV_SUB apart, 8-row K groups SBO = 1 KiB
__device__ __forceinline__ uint64_t desc_mn(uint32_t saddr) {
  return (uint64_t)((saddr & 0x3FFFF) >> 4) | ((uint64_t)(KV_SUB >> 4) << 16) | ((uint64_t)64 << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
// kind::f16, D f32, A = B = bf16, M = 128, N; b_mn selects an MN-major B operand (bit 16)
__host__ __device__ constexpr uint32_t idesc(int n, bool b_mn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((b_mn ? 1u : 0u) << 16) | ((uint32_t)(n >> 3) << 17) |
         ((uint32_t)(128 >> 4) << 24);
}
__device__ __forceinline__ void umma(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(id), "r"(acc));
}
// D (TMEM) += A (TMEM, row = lane, bf16 pairs along columns) . B (smem descriptor)
__device__ __forceinline__ void umma_ts(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n"
      "}\n" ::"r"(d),
      "r"(a_tmem), "l"(b), "r"(id), "r"(acc));
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tc_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
// 2^x on the SFU without the denormal range fix-up exp2f adds (arguments are <= 8 here; underflow -> 0)
__device__ __forceinline__ float fast_exp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// packed fp32x2 arithmetic (FFMA2 / FADD2 on sm_100)
__device__ __forceinline__ uint64_t pack_f2(float lo, float hi) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
  return r;
}
__device__ __forceinline__ void unpack_f2(uint64_t v, float& lo, float& hi) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
}
__device__ __forceinline__ uint64_t ffma2(uint64_t a, uint64_t b, uint64_t c) {
  uint64_t d;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
  return d;
}
__device__ __forceinline__ uint64_t fadd2(uint64_t a, uint64_t b) {
  uint64_t d;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
  return d;
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,"
      "%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
// two 32-column loads in flight, one wait (the softmax's TMEM reads are on its critical path)
__device__ __forceinline__ void tmem_ld32x2(uint32_t taddr0, uint32_t taddr1, uint32_t (&r)[32], uint32_t (&q)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,"
      "%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr0));
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,"
      "%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(q[0]), "=r"(q[1]), "=r"(q[2]), "=r"(q[3]), "=r"(q[4]), "=r"(q[5]), "=r"(q[6]), "=r"(q[7]), "=r"(q[8]),
        "=r"(q[9]), "=r"(q[10]), "=r"(q[11]), "=r"(q[12]), "=r"(q[13]), "=r"(q[14]), "=r"(q[15]), "=r"(q[16]),
        "=r"(q[17]), "=r"(q[18]), "=r"(q[19]), "=r"(q[20]), "=r"(q[21]), "=r"(q[22]), "=r"(q[23]), "=r"(q[24]),
        "=r"(q[25]), "=r"(q[26]), "=r"(q[27]), "=r"(q[28]), "=r"(q[29]), "=r"(q[30]), "=r"(q[31])
      : "r"(taddr1));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"
      "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]),
      "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]),
      "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
  asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ void tmem_st32_nowait(uint32_t taddr, const uint32_t (&r)[32]) {
  asm volatile(
      "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,"
      "%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
      "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]), "r"(r[8]), "r"(r[9]),
      "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15]), "r"(r[16]), "r"(r[17]), "r"(r[18]),
      "r"(r[19]), "r"(r[20]), "r"(r[21]), "r"(r[22]), "r"(r[23]), "r"(r[24]), "r"(r[25]), "r"(r[26]), "r"(r[27]),
      "r"(r[28]), "r"(r[29]), "r"(r[30]), "r"(r[31])
      : "memory");
}

struct Params {
  const int* row0;
  const int* qlen;
  const int* cpre;
  const int* seq_row;
  const int* table;
  int max_pages, hq, hkv, n_qtiles, n_pairs, trace, n_seqs;
  const int* shape_dev;  // nullable: [rows, sequences, longest chunk] on the device (n_qtiles, n_seqs: capacity)
  bf16* o;
  const bf16* k_pool;
  const bf16* v_pool;
};

// Work item = (sequence, 128-row query tile, GQA head pair).  Items are ordered heavy first (query tile
// from the last, then sequence, then pair); a persistent CTA takes items k = 0, 1, ... of a snake order
// over the grid (round r gives CTA b the item r G + b for even r, r G + G - 1 - b for odd r), so the heavy
// and light items of consecutive rounds balance; with G = the item count every CTA takes one item (the
// one-item-per-CTA launch).  Every warp role walks the same sequence and skips the same empty items.
struct Item {
  int s_id, qt, pair, qlen, row0, cpre, q0, kvh, head_a, n_heads, kv_end, n_kt;
  const int* tab;
};
// cta / n_ctas: this CTA among the CTAs running prefill attention (the grid, or the prefill part of the
// fused POD launch, kernels_pod.cu)
__device__ __forceinline__ bool item_at(const Params& p, int k, Item& it, bool& live, int cta, int n_ctas) {
  // a launch sized for the capacity (device-side shapes, f4) enumerates the step's own sequences and query
  // tiles: shape_dev = [rows, sequences, longest chunk] of the step's metadata
  const int n_seqs = p.shape_dev ? p.shape_dev[1] : p.n_seqs;
  const int n_qtiles = p.shape_dev ? (p.shape_dev[2] + BQ - 1) / BQ : p.n_qtiles;
  const int G = n_ctas, T = n_qtiles * n_seqs * p.n_pairs;
  const int idx = k * G + ((k & 1) ? G - 1 - cta : cta);
  if (idx >= T) return false;
  it.pair = idx % p.n_pairs;
  it.s_id = (idx / p.n_pairs) % n_seqs;
  it.qt = n_qtiles - 1 - idx / (p.n_pairs * n_seqs);
  it.qlen = p.qlen[it.s_id];
  live = it.qt * BQ < it.qlen;
  if (!live) return true;
  const int Gq = p.hq / p.hkv, ppg = (Gq + 1) / 2;
  it.kvh = it.pair / ppg;
  it.head_a = it.kvh * Gq + (it.pair % ppg) * 2;
  it.n_heads = it.head_a + 1 < (it.kvh + 1) * Gq ? 2 : 1;
  it.row0 = p.row0[it.s_id];
  it.cpre = p.cpre[it.s_id];
  it.tab = p.table + (size_t)p.seq_row[it.s_id] * p.max_pages;
  it.q0 = it.qt * BQ;
  const int q_last = min(it.q0 + BQ, it.qlen) - 1;
  it.kv_end = it.cpre + q_last + 1;
  it.n_kt = (it.kv_end + BKV - 1) / BKV;
  return true;
}

template <int K_STAGES, int V_STAGES>
__device__ __forceinline__ void fa_tc_body(const CUtensorMap* mq, const Params& p, const int cta, const int n_ctas) {
  using RG = Ring<K_STAGES, V_STAGES>;
  constexpr int OFF_V = RG::OFF_V, OFF_BAR = RG::OFF_BAR, OFF_TRACE = RG::OFF_TRACE;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* bar = (uint64_t*)(smem + OFF_BAR);
  uint64_t* q_full = bar;                   // 1
  uint64_t* k_full = bar + 1;               // [K_STAGES] K ring: freed by the S MMAs
  uint64_t* k_empty = k_full + K_STAGES;
  uint64_t* v_full = k_empty + K_STAGES;    // [V_STAGES] V ring: freed by the PV MMAs
  uint64_t* v_empty = v_full + V_STAGES;
  uint64_t* s_full = v_empty + V_STAGES;    // [head]
  uint64_t* p_full = s_full + 2;            // [head]
  uint64_t* o_done = p_full + 2;            // [head]: the last PV of a work item
  uint64_t* q_empty = o_done + 2;           // 1: the item's last S MMAs completed (Q tiles reusable)
  uint32_t* tmem_slot = (uint32_t*)(q_empty + 1);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (warp == 0 && lane == 0) {
    mbar_init(q_full, 1);
    mbar_init(q_empty, 1);
    for (int i = 0; i < K_STAGES; ++i) {
      mbar_init(&k_full[i], 64);  // one cp.async-tracked (noinc) arrive per loader thread of the tensor
      mbar_init(&k_empty[i], 1);
    }
    for (int i = 0; i < V_STAGES; ++i) {
      mbar_init(&v_full[i], 64);
      mbar_init(&v_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&p_full[i], 4);
      mbar_init(&o_done[i], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "n"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_before();
  __syncthreads();
  tc_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();  // set-up above overlaps the previous kernel's tail
  // timeline debugging (DUET_FA_TRACE=1): event e of tile j, clock() relative to kernel start
  uint32_t* trace = (uint32_t*)(smem + OFF_TRACE);
  bool tr = (p.trace & 1) && cta == 0;  // CTA 0's first work item
  const uint32_t t_start = (uint32_t)clock();
  auto stamp = [&](int e, int j) {
    if (tr && lane == 0 && j < TRACE_MAXJ) trace[e * TRACE_MAXJ + j] = (uint32_t)clock() - t_start;
  };
  // head h: S_j (fp32, 128 columns), overwritten in place by P_j (bf16 pairs, columns 0..63); O
  auto T_S = [&](int h) { return tmem + h * 256; };
  auto T_O = [&](int h) { return tmem + h * 256 + BKV; };

  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------ Q tiles (TMA, two 64-column boxes per head); the
      // next item's tiles load as soon as the current item's last S MMAs have read them
      int ni = 0;
      Item it;
      bool live;
      for (int k = 0; item_at(p, k, it, live, cta, n_ctas); ++k) {
        if (!live) continue;
        mbar_wait(q_empty, (ni & 1) ^ 1);
        mbar_expect_tx(q_full, it.n_heads * Q_BYTES);
        for (int h = 0; h < it.n_heads; ++h) {
          tma_load_2d(mq, q_full, smem + OFF_Q + h * Q_BYTES, (it.head_a + h) * DH, it.row0 + it.q0);
          tma_load_2d(mq, q_full, smem + OFF_Q + h * Q_BYTES + Q_SUB, (it.head_a + h) * DH + 64, it.row0 + it.q0);
        }
        ++ni;
      }
    }
  } else if (warp >= 10) {
    // ------------------------------------------------ loaders: warps 10-11 stream K, warps 12-13 stream V
    // (separate rings: a K slot frees when the S MMAs of its tile complete, long before its V slot)
    const int tensor = (warp - 10) >> 1;           // 0 = K, 1 = V
    const int lt = threadIdx.x - (10 + 2 * tensor) * 32;  // 0..63
    const bf16* pool = tensor ? p.v_pool : p.k_pool;
    uint64_t* full = tensor ? v_full : k_full;
    uint64_t* empty = tensor ? v_empty : k_empty;
    const int off_ring = tensor ? OFF_V : OFF_K;
    const int nst = tensor ? V_STAGES : K_STAGES;
    const size_t page_stride = (size_t)p.hkv * PAGE * DH;
    // chunk c = lt + 64 i (i < 32) of a [128 keys][16 chunks] tile: key row rr = lt/16 + 4 i, 16-B
    // column ch = lt % 16 (fixed per thread); page-in-tile = i / 4, row-in-page = lt/16 + 4 (i % 4).
    // The per-thread address pattern is hoisted: per tile only the 8 page-table entries are read.
    const int ch = lt & 15, r0 = lt >> 4;
    const uint32_t so0 = (uint32_t)((ch >> 3) * KV_SUB);
    int g = 0;  // tiles streamed by this CTA so far (ring position across work items)
    Item it;
    bool live;
    for (int k = 0; item_at(p, k, it, live, cta, n_ctas); ++k) {
     if (!live) continue;
     const int kv_end = it.kv_end;
     const int* tab = it.tab;
     const size_t col_off = (size_t)it.kvh * PAGE * DH + ch * 8;
     for (int j = 0; j < it.n_kt; ++j, ++g) {
      const int st = g % nst;
      mbar_wait(&empty[st], ((g / nst) & 1) ^ 1);
      if (warp == 10) stamp(0, j);
      const uint32_t dst = smem_u32(smem + off_ring + st * KV_BYTES) + so0;
      if (p.trace & 2) {  // timing experiment only (DUET_FA_TRACE=noload): no K/V traffic, garbage result
        mbar_arrive(&full[st]);
        continue;
      }
      const int pg_base = j * (BKV / PAGE);
#pragma unroll
      for (int pp = 0; pp < BKV / PAGE; ++pp) {  // 8 pages of the tile
        const int kp = (pg_base + pp) * PAGE;    // first key of the page
        const bool page_live = kp < kv_end;
        const bf16* src_pg = pool + (page_live ? (size_t)tab[pg_base + pp] * page_stride + col_off : 0);
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const int rip = r0 + 4 * q;            // row in page
          const int rr = pp * PAGE + rip;        // row in tile
          const bool v = page_live && kp + rip < kv_end;
          const uint32_t so = (uint32_t)(rr * 128 + (((ch & 7) ^ (rr & 7)) << 4));
          asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst + so),
                       "l"(src_pg + (v ? rip * DH : 0)), "r"(v ? 16 : 0)
                       : "memory");
        }
      }
      // the barrier phase completes when every loader thread's copies of this tile have landed
      asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(&full[st])) : "memory");
     }
     tr = false;
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
  } else if (warp == 1) {
    // ------------------------------------------------ MMA issuer
    // tcgen05.mma from one thread executes in issue order: S_{j+1}^h (written over P_j^h) is issued right
    // after PV_j^h (which reads P_j^h), and a commit tracks every earlier MMA, so s_full also
    // certifies that PV_{j-1} has completed.  Across work items: S_0 of the next item follows the last
    // PV of the current one (the softmax warps drain O meanwhile; the next item's PV_0, which overwrites
    // O, waits for p_full, which those warps arrive on only after their epilogue read O).
    constexpr uint32_t ID_S = idesc(BKV, false), ID_PV = idesc(DH, true);
    int ni = 0, gk = 0, gv = 0;      // items, K tiles, V tiles consumed by this CTA
    int gp[2] = {0, 0};              // P tiles per head
    Item it;
    bool live;
    for (int k = 0; item_at(p, k, it, live, cta, n_ctas); ++k) {
      if (!live) continue;
      const int n_kt = it.n_kt, n_heads = it.n_heads;
      mbar_wait(q_full, ni & 1);
      auto wait_k = [&](int j) {
        mbar_wait(&k_full[gk % K_STAGES], (gk / K_STAGES) & 1);
        stamp(1, j);
        fence_async_smem();  // the loaders' cp.async (generic proxy) writes -> visible to the MMA (async proxy)
        tc_after();
      };
      auto issue_s = [&](int j, int h) {  // S_j^h = Q^h K_j^T
        if (lane == 0) {
          const uint32_t sk = smem_u32(smem + OFF_K + (gk % K_STAGES) * KV_BYTES);
          const uint32_t sq = smem_u32(smem + OFF_Q + h * Q_BYTES);
#pragma unroll
          for (int kk = 0; kk < DH / 16; ++kk)
            umma(T_S(h), desc_k(sq + (kk >> 2) * Q_SUB + (kk & 3) * 32), desc_k(sk + (kk >> 2) * KV_SUB + (kk & 3) * 32),
                 ID_S, kk > 0);
          umma_commit(&s_full[h]);
          if (h == n_heads - 1) {
            umma_commit(&k_empty[gk % K_STAGES]);
            if (j == n_kt - 1) umma_commit(q_empty);  // the item's last S: its Q tiles may be replaced
          }
        }
        __syncwarp();
      };
      wait_k(0);
      for (int h = 0; h < n_heads; ++h) issue_s(0, h);
      ++gk;
      stamp(2, 0);
      for (int j = 0; j < n_kt; ++j, ++gv) {
        const int st = gv % V_STAGES;
        mbar_wait(&v_full[st], (gv / V_STAGES) & 1);
        fence_async_smem();
        const uint32_t sv = smem_u32(smem + OFF_V + st * KV_BYTES);
        if (j + 1 < n_kt) wait_k(j + 1);
        for (int h = 0; h < n_heads; ++h) {
          mbar_wait(&p_full[h], gp[h] & 1);
          ++gp[h];
          tc_after();
          if (lane == 0) {
#pragma unroll
            for (int kk = 0; kk < BKV / 16; ++kk)  // 16 keys per UMMA k-step: A = P (TMEM, 8 columns), B = V
              umma_ts(T_O(h), T_S(h) + kk * 8, desc_mn(sv + kk * 16 * 128), ID_PV, (j > 0 || kk > 0));
            if (j == n_kt - 1) umma_commit(&o_done[h]);
            if (h == n_heads - 1) umma_commit(&v_empty[st]);
          }
          __syncwarp();
          if (j + 1 < n_kt) issue_s(j + 1, h);
        }
        if (j + 1 < n_kt) ++gk;
        stamp(3, j);
        if (j + 1 < n_kt) stamp(2, j + 1);
      }
      ++ni;
      if (tr && lane == 0) trace[10 * TRACE_MAXJ] = (uint32_t)n_kt;  // the traced item's key tiles
      tr = false;
    }
  } else {
    // ------------------------------------------------ softmax warps: one thread per query row
    const int h = (warp - 2) >> 2;  // head A (warps 2..5) or B (6..9)
    const int quad = warp & 3;
    const int r = quad * 32 + lane;                          // row in tile = TMEM lane
    const float sc = rsqrtf((float)DH) * 1.4426950408889634f;
    const uint32_t lane_base = (uint32_t)(quad * 32) << 16;
    const uint32_t t_s = T_S(h) + lane_base;
    int gs = 0, ni_h = 0;  // S tiles and work items of this head so far
    Item it;
    bool live;
    for (int k = 0; item_at(p, k, it, live, cta, n_ctas); ++k) {
      if (!live || h >= it.n_heads) continue;  // an odd last head of a group runs alone (no head B)
      const int n_kt = it.n_kt, q0 = it.q0, qlen = it.qlen, row0 = it.row0, head_a = it.head_a;
      const int pos = min(it.cpre + q0 + r, it.kv_end - 1);  // clamp rows past the chunk
      float m_used = -INFINITY, l = 0.f;
      for (int j = 0; j < n_kt; ++j, ++gs) {
        mbar_wait(&s_full[h], gs & 1);
        if (warp == 2) stamp(4, j);
        if (warp == 6) stamp(7, j);
        tc_after();
        const int lim = pos - j * BKV;  // keys 0..lim of this tile are visible to this row
        const bool full_tile = lim >= BKV - 1;
        // One pass over S in two 64-column chunks (online softmax at chunk granularity): each chunk is
        // read from TMEM once, its max taken in registers, the exponentials taken against the running
        // reference m_used, and P written over the chunk's S columns.  The reference is re-based only
        // when a chunk's max exceeds it by more than 2^8: O and l are rescaled (PV_{j-1} is complete:
        // s_full tracks it) and, for the second chunk, so is the first chunk's P already in TMEM.
        // (The two-pass version read S twice: TMEM traffic that also slowed the MMAs, FA_TRACE.)
        float l0 = 0.f, l1 = 0.f;
#pragma unroll 1
        for (int c = 0; c < 2; ++c) {
          uint32_t v0[32], v1[32], pk[32];
          tmem_ld32x2(t_s + c * 64, t_s + c * 64 + 32, v0, v1);
          if (!full_tile) {  // keys past the row's causal end -> -inf: exp2 gives 0, the max ignores them
#pragma unroll
            for (int e = 0; e < 32; ++e) {
              if (c * 64 + e > lim) v0[e] = 0xff800000u;
              if (c * 64 + 32 + e > lim) v1[e] = 0xff800000u;
            }
          }
          float mx = -INFINITY;
#pragma unroll
          for (int e = 0; e < 32; e += 2)
            mx = fmaxf(mx, fmaxf(fmaxf(__uint_as_float(v0[e]), __uint_as_float(v0[e + 1])),
                                 fmaxf(__uint_as_float(v1[e]), __uint_as_float(v1[e + 1]))));
          const float m_new = fmaxf(m_used, mx * sc);  // sc > 0: the max commutes with the scaling
          const bool mine = m_new > m_used + RESCALE_THRESHOLD;
          if (__any_sync(0xffffffffu, mine)) {  // rare after the first chunk of a row
            const float f = mine ? exp2f(m_used - m_new) : 1.f;  // 0 while m_used = -inf (nothing to scale)
            l *= f;
            l0 *= f;
            l1 *= f;
            if (j >= 1) {
#pragma unroll 1
              for (int cc = 0; cc < DH; cc += 32) {
                uint32_t v[32];
                tmem_ld32(T_O(h) + lane_base + cc, v);
#pragma unroll
                for (int e = 0; e < 32; ++e) v[e] = __float_as_uint(__uint_as_float(v[e]) * f);
                tmem_st32(T_O(h) + lane_base + cc, v);
              }
            }
            if (c == 1) {  // the first chunk's P (bf16 pairs in columns 0..31) against the new reference
              asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
              uint32_t v[32];
              tmem_ld32(t_s, v);
#pragma unroll
              for (int e = 0; e < 32; ++e) {
                const float2 q = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&v[e]));
                __nv_bfloat162 t = __floats2bfloat162_rn(q.x * f, q.y * f);
                v[e] = *reinterpret_cast<uint32_t*>(&t);
              }
              tmem_st32(t_s, v);
            }
            if (mine) m_used = m_new;
          }
          // the chunk's 64 exponentials, packed f32x2 (masked keys hold -inf: p = 0, a row's first chunk
          // always has its key 0 visible, so m_used is finite whenever a -inf is exponentiated)
          const uint64_t sc2 = pack_f2(sc, sc), nm2 = pack_f2(-m_used, -m_used);
          uint64_t acc2 = pack_f2(0.f, 0.f);
#pragma unroll
          for (int e = 0; e < 64; e += 2) {
            const uint32_t* src = e < 32 ? v0 : v1;
            const int ee = e & 31;
            const uint64_t t2 = ffma2(pack_f2(__uint_as_float(src[ee]), __uint_as_float(src[ee + 1])), sc2, nm2);
            float t0, t1;
            unpack_f2(t2, t0, t1);
            const float p0 = fast_exp2(t0), p1 = fast_exp2(t1);
            acc2 = fadd2(acc2, pack_f2(p0, p1));
            __nv_bfloat162 t = __floats2bfloat162_rn(p0, p1);
            pk[e / 2] = *reinterpret_cast<uint32_t*>(&t);
          }
          float a0, a1;
          unpack_f2(acc2, a0, a1);
          l0 += a0;
          l1 += a1;
          tmem_st32_nowait(t_s + c * 32, pk);  // completion awaited once, before p_full
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        l += l0 + l1;
        if (warp == 2) stamp(5, j);
        if (warp == 6) stamp(8, j);
        tc_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[h]);
        if (warp == 2) stamp(6, j);
        if (warp == 6) stamp(9, j);
      }
      {  // the CTA's last work item: only its epilogue is left
        Item nx;
        bool nlive = false;
        int kk = k + 1;
        while (item_at(p, kk, nx, nlive, cta, n_ctas) && !nlive) ++kk;
        if (!nlive) pdl_trigger();
      }
      // epilogue: O / l -> bf16 -> global
      mbar_wait(&o_done[h], ni_h & 1);
      ++ni_h;
      tc_after();
      const bool row_ok = q0 + r < qlen;
      const float inv = l > 0.f ? 1.f / l : 0.f;
      bf16* dst = p.o + (size_t)(row0 + q0 + r) * p.hq * DH + (size_t)(head_a + h) * DH;
#pragma unroll 1
      for (int c = 0; c < DH; c += 32) {
        uint32_t v[32];
        tmem_ld32(T_O(h) + lane_base + c, v);
        if (row_ok) {
#pragma unroll
          for (int q4 = 0; q4 < 4; ++q4) {
            float o8[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) o8[e] = __uint_as_float(v[q4 * 8 + e]) * inv;
            store16<bf16>(dst + c + q4 * 8, o8);
          }
        }
      }
      tr = false;
    }
  }
  tc_before();
  __syncthreads();
  if ((p.trace & 1) && cta == 0 && threadIdx.x == 0) {
    const int n_kt = (int)trace[10 * TRACE_MAXJ];
    printf("FA_TRACE n_kt=%d (clock cycles; ev: 0 load-issue 1 kv_full 2 S-issued 3 PV-issued 4 s_full 5 exps-done 6 P-published)\n", n_kt);
    for (int j = 0; j < n_kt && j < TRACE_MAXJ; ++j)
      printf("FA_TRACE j=%2d %8u %8u %8u %8u | A %8u %8u %8u | B %8u %8u %8u\n", j, trace[j], trace[TRACE_MAXJ + j],
             trace[2 * TRACE_MAXJ + j], trace[3 * TRACE_MAXJ + j], trace[4 * TRACE_MAXJ + j], trace[5 * TRACE_MAXJ + j],
             trace[6 * TRACE_MAXJ + j], trace[7 * TRACE_MAXJ + j], trace[8 * TRACE_MAXJ + j], trace[9 * TRACE_MAXJ + j]);
  }
  if (warp == 1) {
    tc_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(TMEM_COLS));
  }
}

template <int K_STAGES, int V_STAGES>
__global__ void __launch_bounds__(THREADS, 1) fa_tc_kernel(const __grid_constant__ CUtensorMap map_q, Params p) {
  fa_tc_body<K_STAGES, V_STAGES>(&map_q, p, (int)blockIdx.x, (int)gridDim.x);
}

#ifndef DUET_BODIES_ONLY
typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* f = nullptr;
    if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &f, 12000, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (EncodeTiledFn)f;
  }
  return fn;
}
static bool make_map(CUtensorMap* m, const void* base, uint64_t rows, uint64_t cols, uint64_t ld_elems,
                     uint32_t box_rows) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {ld_elems * 2};
  cuuint32_t box[2] = {64, box_rows};
  cuuint32_t es[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

#endif  // DUET_BODIES_ONLY
}  // namespace fatc
#ifndef DUET_BODIES_ONLY

bool fa_tc_supported(const PrefillAttnArgs& a) {
  return a.dh == fatc::DH && a.page_size == fatc::PAGE && a.q_stride % 8 == 0 && fatc::encode_fn() != nullptr &&
         a.total_rows > 0;
}

int launch_fa_tc(const PrefillAttnArgs& a, cudaStream_t st) {
  // DUET_FA_RING = "KSxVS": K / V ring depths (A/B); K 3 / V 2 and K 2 / V 3 measure the same
  // (profiles/r02_fa_ring_ab.txt: the MMA warp's K waits are the per-CTA pipeline fill, not ring depth)
  static int ks = 3, vs = 2;
  static bool attr = false;
  if (!attr) {
    if (const char* e = getenv("DUET_FA_RING")) sscanf(e, "%dx%d", &ks, &vs);
    cudaFuncSetAttribute(fatc::fa_tc_kernel<2, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, fatc::Ring<2, 3>::SMEM);
    cudaFuncSetAttribute(fatc::fa_tc_kernel<3, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, fatc::Ring<3, 2>::SMEM);
    attr = true;
  }
  CUtensorMap mq;
  if (!fatc::make_map(&mq, a.q, (uint64_t)a.total_rows, (uint64_t)a.q_stride, (uint64_t)a.q_stride, 128)) return -1;
  fatc::Params p{a.row0, a.qlen, a.cpre, a.seq_row, a.table, a.max_pages, a.hq, a.hkv, 0, 0, 0, 0, nullptr,
                 (bf16*)a.o, (const bf16*)a.k_pool, (const bf16*)a.v_pool};
  const int G = a.hq / a.hkv;
  p.n_qtiles = (a.max_q + fatc::BQ - 1) / fatc::BQ;
  p.n_pairs = a.hkv * ((G + 1) / 2);
  p.n_seqs = a.n_seqs;
  p.shape_dev = a.shape_dev;
  static const char* trace = getenv("DUET_FA_TRACE");
  // DUET_FA_TRACE: any value prints the timeline of CTA (0,0,0); "noload" skips the K/V loads instead
  // (timing experiment, garbage output); "tn" does both
  p.trace = trace ? (trace[0] == 'n' ? 2 : (trace[0] == 't' && trace[1] == 'n' ? 3 : 1)) : 0;
  // persistent: one CTA per SM of the partition walks a snake order of the work items (the next item's Q
  // load, first K / V tiles and S_0 overlap the current item's last PV and epilogue); DUET_FA_PERSIST=0
  // launches one CTA per item (the round-1 grid, A/B)
  static const bool persist = !getenv("DUET_FA_PERSIST") || atoi(getenv("DUET_FA_PERSIST")) != 0;
  const int items = p.n_qtiles * a.n_seqs * p.n_pairs;
  dim3 grid(persist ? std::min(items, std::max(a.num_sms, 1)) : items);
  if (ks == 2 && vs == 3) launch_pdl(fatc::fa_tc_kernel<2, 3>, grid, fatc::THREADS, fatc::Ring<2, 3>::SMEM, st, mq, p);
  else launch_pdl(fatc::fa_tc_kernel<3, 2>, grid, fatc::THREADS, fatc::Ring<3, 2>::SMEM, st, mq, p);
  return 1;
}

#endif  // DUET_BODIES_ONLY
}  // namespace duet

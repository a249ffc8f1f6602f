// Causal prefill attention over the paged KV cache on a CTA PAIR (tcgen05 cta_group::2).
//
// Same computation as kernels_fa_tc.cu (chunked prefill, §4.1; readings #2, #6, #7):
// the chunk's rows attend causally to the c-token prefix and to themselves.  Why a pair: the one-CTA
// kernel is bound by shared memory — a 128x128x16 score UMMA with Q and K both in shared memory reads
// 8 KiB per 64 cycles, the full 128 B/clk port, next to the loaders' 64 KiB of writes per KV tile.
// Here two CTAs of a cluster (one TPC) hold 256 consecutive query rows of the same two heads (CTA r:
// rows 128 r .. 128 r + 127 of the pair block) and split every KV tile between them:
//   S = Q K^T   UMMA 256 x 128 x 16: A = each CTA's own Q rows, B = K — CTA r holds keys 64 r .. 64 r + 63
//   O += P V    UMMA 256 x 128 x 16: A = P from each CTA's TMEM, B = V — CTA r holds dims 64 r .. 64 r + 63
// so each SM reads 6 instead of 8 KiB per score k-step, 2 instead of 4 KiB per PV k-step, and gathers
// 32 instead of 64 KiB per KV tile (~160 instead of ~256 KiB of shared-memory traffic per tile).
//   warp 0        Q tiles of this CTA by TMA (2 heads x two 64-column SW128 boxes)
//   warp 1        TMEM (512 columns, cta_group::2: per head S_j/P_j 128 | O 128); in the leader CTA
//                 lane 0 issues every MMA of the pair and commits to both CTAs' barriers (multicast)
//   warps 2..9    softmax, one thread per query row (= TMEM lane) of this CTA: warps 2-5 head A,
//                 6-9 head B — as in the one-CTA kernel; P is published to the leader's p_pair barrier
//   warps 10..13  loaders: cp.async gathers of this CTA's half of each K / V tile (K ring 3, V ring 4)
//   warp 14       forwarder: waits this CTA's local "tile landed" barriers and arrives on the leader's
//                 pair barriers (a cp.async completion can only signal a barrier of its own CTA)
// The last KV tile of the pair block is masked out for CTA 0's rows (causal): ~1/n_kt of the MMAs.
#include <cuda.h>

#include <cstdio>
#include <cstdlib>

#include "dev_common.cuh"
#include "kernels.h"

namespace duet {
namespace fa2 {

constexpr int BQ = 128, BKV = 128, DH = 128, PAGE = 16, K_STAGES = 3, V_STAGES = 4;
constexpr int Q_SUB = BQ * 128;                  // [128 rows][64 cols] SW128 = 16 KiB
constexpr int Q_BYTES = 2 * Q_SUB;               // 32 KiB per head
constexpr int K_SUB = 64 * 128;                  // this CTA's 64 keys x 64 dims = 8 KiB
constexpr int K_BYTES = 2 * K_SUB;               // 16 KiB per stage (two dim halves)
constexpr int V_BYTES = BKV * 128;               // 128 keys x this CTA's 64 dims = 16 KiB per stage
constexpr int OFF_Q = 0;
constexpr int OFF_K = OFF_Q + 2 * Q_BYTES;
constexpr int OFF_V = OFF_K + K_STAGES * K_BYTES;
constexpr int OFF_BAR = OFF_V + V_STAGES * V_BYTES;
constexpr int SMEM = OFF_BAR + 512 + 1024;
constexpr int THREADS = 15 * 32;
constexpr int TMEM_COLS = 512;
constexpr float RESCALE_THRESHOLD = 8.0f;  // log2 domain
static_assert(SMEM <= 227 * 1024, "smem");

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
__device__ __forceinline__ uint32_t mapa(uint32_t saddr, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(saddr), "r"(rank));
  return r;
}
__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
// arrive on a barrier of (possibly) the other CTA of the cluster, release at cluster scope
__device__ __forceinline__ void mbar_arrive_remote(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr) : "memory");
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
// wait on a barrier whose arrivals come from the other CTA too (acquire at cluster scope)
__device__ __forceinline__ void mbar_wait_cluster(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%0], %1;\n"
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
// K-major SW128 descriptor (rows of 128 B, 8-row atoms of 1 KiB): SBO = 1 KiB
__device__ __forceinline__ uint64_t desc_k(uint32_t saddr) {
  return (uint64_t)((saddr & 0x3FFFF) >> 4) | ((uint64_t)1 << 16) | ((uint64_t)64 << 32) | ((uint64_t)1 << 46) |
         ((uint64_t)2 << 61);
}
// MN-major SW128 descriptor of this CTA's [128 keys][64 dims] V tile: one 64-element MN block, 8-row K
// groups SBO = 1 KiB apart
__device__ __forceinline__ uint64_t desc_mn(uint32_t saddr) {
  return (uint64_t)((saddr & 0x3FFFF) >> 4) | ((uint64_t)(V_BYTES >> 4) << 16) | ((uint64_t)64 << 32) |
         ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
// kind::f16, D f32, A = B = bf16, M = 256 (pair), N; b_mn selects an MN-major B operand
__host__ __device__ constexpr uint32_t idesc(int n, bool b_mn) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((b_mn ? 1u : 0u) << 16) | ((uint32_t)(n >> 3) << 17) |
         ((uint32_t)(256 >> 4) << 24);
}
__device__ __forceinline__ void umma2(uint32_t d, uint64_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(d),
      "l"(a), "l"(b), "r"(id), "r"(acc));
}
// D (TMEM) += A (TMEM of each CTA, row = lane, bf16 pairs along columns) . B (smem descriptor)
__device__ __forceinline__ void umma2_ts(uint32_t d, uint32_t a_tmem, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n"
      "}\n" ::"r"(d),
      "r"(a_tmem), "l"(b), "r"(id), "r"(acc));
}
// arrive on the barrier at this offset in BOTH CTAs once every earlier MMA of the pair has completed
__device__ __forceinline__ void commit_both(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}
__device__ __forceinline__ void tc_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ float fast_exp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
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

struct Params {
  const int* row0;
  const int* qlen;
  const int* cpre;
  const int* seq_row;
  const int* table;
  int max_pages, hq, hkv, n_qblocks, n_pairs;
  bf16* o;
  const bf16* k_pool;
  const bf16* v_pool;
};

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(THREADS, 1)
    fa2_kernel(const __grid_constant__ CUtensorMap map_q, Params p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* bar = (uint64_t*)(smem + OFF_BAR);
  uint64_t* q_full = bar;                    // local: Q TMA bytes
  uint64_t* k_full = q_full + 1;             // [K_STAGES] local: this CTA's K half landed (cp.async)
  uint64_t* k_empty = k_full + K_STAGES;     // [K_STAGES] both: the S MMAs of the tile completed
  uint64_t* v_full = k_empty + K_STAGES;     // [V_STAGES] local
  uint64_t* v_empty = v_full + V_STAGES;     // [V_STAGES] both: the PV MMAs completed
  uint64_t* s_full = v_empty + V_STAGES;     // [head] both: S_j in TMEM
  uint64_t* o_done = s_full + 2;             // [head] both: the last PV
  uint64_t* q_pair = o_done + 2;             // leader: both CTAs' Q landed (2 arrivals)
  uint64_t* k_pair = q_pair + 1;             // [K_STAGES] leader: both K halves landed
  uint64_t* v_pair = k_pair + K_STAGES;      // [V_STAGES] leader
  uint64_t* p_pair = v_pair + V_STAGES;      // [head] leader: both CTAs' P_j published (8 warps)
  uint32_t* tmem_slot = (uint32_t*)(p_pair + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  const int pair = blockIdx.x >> 1;
  const int qb = p.n_qblocks - 1 - blockIdx.y;  // heavy (late) blocks first
  const int s_id = blockIdx.z;
  const int qlen = p.qlen[s_id];
  if (qb * 2 * BQ >= qlen) return;              // uniform over the pair: neither CTA syncs
  const int G = p.hq / p.hkv;
  const int pairs_per_group = (G + 1) / 2;
  const int kvh = pair / pairs_per_group;
  const int head_a = kvh * G + (pair % pairs_per_group) * 2;
  const bool has_b = head_a + 1 < (kvh + 1) * G;
  const int n_heads = has_b ? 2 : 1;
  const int row0 = p.row0[s_id], cpre = p.cpre[s_id];
  const int* tab = p.table + (size_t)p.seq_row[s_id] * p.max_pages;
  const int q0 = qb * 2 * BQ + (int)rank * BQ;  // this CTA's first row
  const int q_last = min(qb * 2 * BQ + 2 * BQ, qlen) - 1;  // the pair's last row
  const int kv_end = cpre + q_last + 1;
  const int n_kt = (kv_end + BKV - 1) / BKV;

  if (warp == 0 && lane == 0) {
    mbar_init(q_full, 1);
    for (int i = 0; i < K_STAGES; ++i) {
      mbar_init(&k_full[i], 64);
      mbar_init(&k_empty[i], 1);
      mbar_init(&k_pair[i], 2);
    }
    for (int i = 0; i < V_STAGES; ++i) {
      mbar_init(&v_full[i], 64);
      mbar_init(&v_empty[i], 1);
      mbar_init(&v_pair[i], 2);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&o_done[i], 1);
      mbar_init(&p_pair[i], 8);
    }
    mbar_init(q_pair, 2);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "n"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_before();
  cluster_sync();  // barriers initialised and TMEM allocated in both CTAs before any remote access
  tc_after();
  const uint32_t tmem = *tmem_slot;
  pdl_wait();
  auto T_S = [&](int h) { return tmem + h * 256; };
  auto T_O = [&](int h) { return tmem + h * 256 + BKV; };
  auto leader_addr = [&](uint64_t* b) { return mapa(smem_u32(b), 0); };

  if (warp == 0) {
    if (lane == 0) {  // ---------------- this CTA's Q rows (TMA; rows past the tensor end are zero-filled)
      mbar_expect_tx(q_full, n_heads * Q_BYTES);
      for (int h = 0; h < n_heads; ++h) {
        tma_load_2d(&map_q, q_full, smem + OFF_Q + h * Q_BYTES, (head_a + h) * DH, row0 + q0);
        tma_load_2d(&map_q, q_full, smem + OFF_Q + h * Q_BYTES + Q_SUB, (head_a + h) * DH + 64, row0 + q0);
      }
    }
  } else if (warp == 14) {
    if (lane == 0) {  // ---------------- forwarder: this CTA's landed tiles -> the leader's pair barriers
      mbar_wait(q_full, 0);
      mbar_arrive_remote(leader_addr(q_pair));
      for (int j = 0; j < n_kt; ++j) {
        mbar_wait(&k_full[j % K_STAGES], (j / K_STAGES) & 1);
        fence_async_smem();  // the loaders' generic-proxy writes -> visible to the async proxy (UMMA)
        mbar_arrive_remote(leader_addr(&k_pair[j % K_STAGES]));
        mbar_wait(&v_full[j % V_STAGES], (j / V_STAGES) & 1);
        fence_async_smem();
        mbar_arrive_remote(leader_addr(&v_pair[j % V_STAGES]));
      }
    }
  } else if (warp >= 10) {
    // ---------------- loaders: warps 10-11 this CTA's 64 keys of every K tile, 12-13 its 64 dims of V
    const int tensor = (warp - 10) >> 1;  // 0 = K, 1 = V
    const int lt = threadIdx.x - (10 + 2 * tensor) * 32;
    const bf16* pool = tensor ? p.v_pool : p.k_pool;
    uint64_t* full = tensor ? v_full : k_full;
    uint64_t* empty = tensor ? v_empty : k_empty;
    const int nst = tensor ? V_STAGES : K_STAGES;
    const size_t page_stride = (size_t)p.hkv * PAGE * DH;
    const size_t head_off = (size_t)kvh * PAGE * DH;
    // K: chunk (kr, ch): key kr = r0 + 4 i (of this CTA's 64), 16-B column ch = lt % 16 (128 dims)
    // V: chunk (kr, ch): key kr = r0 + 8 i (of 128), 16-B column ch = lt % 8 of this CTA's 64 dims
    const int ch = tensor ? (lt & 7) : (lt & 15);
    const int r0 = tensor ? (lt >> 3) : (lt >> 4);
    const int kstep = tensor ? 8 : 4;
    const int key_base = tensor ? 0 : 64 * (int)rank;          // key offset of this CTA's rows in the tile
    const int dim_off = tensor ? 64 * (int)rank + 8 * ch : 8 * ch;
    for (int j = 0; j < n_kt; ++j) {
      const int st = j % nst;
      mbar_wait(&empty[st], ((j / nst) & 1) ^ 1);
      const uint32_t dst = smem_u32(smem + (tensor ? OFF_V + st * V_BYTES : OFF_K + st * K_BYTES));
#pragma unroll 4
      for (int i = 0; i < 16; ++i) {
        const int kr = r0 + kstep * i;                   // row of this CTA's tile part
        const int key = j * BKV + key_base + kr;         // key position in the sequence
        const bool v = key < kv_end;
        const bf16* src = v ? pool + (size_t)tab[key / PAGE] * page_stride + head_off + (key % PAGE) * DH + dim_off
                            : pool;
        const uint32_t so = tensor ? (uint32_t)(kr * 128 + ((ch ^ (kr & 7)) << 4))
                                   : (uint32_t)((ch >> 3) * K_SUB + kr * 128 + (((ch & 7) ^ (kr & 7)) << 4));
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst + so), "l"(src), "r"(v ? 16 : 0)
                     : "memory");
      }
      asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(&full[st])) : "memory");
    }
    asm volatile("cp.async.wait_all;" ::: "memory");
  } else if (warp == 1) {
    if (leader && lane == 0) {
      // ---------------- MMA issuer of the pair (in issue order: S_{j+1}^h overwrites P_j^h after PV_j^h)
      constexpr uint32_t ID_S = idesc(BKV, false), ID_PV = idesc(DH, true);
      mbar_wait_cluster(q_pair, 0);
      tc_after();
      auto wait_k = [&](int j) {
        mbar_wait_cluster(&k_pair[j % K_STAGES], (j / K_STAGES) & 1);
        tc_after();
      };
      auto issue_s = [&](int j, int h) {  // S_j^h = Q^h K_j^T
        const uint32_t sk = smem_u32(smem + OFF_K + (j % K_STAGES) * K_BYTES);
        const uint32_t sq = smem_u32(smem + OFF_Q + h * Q_BYTES);
#pragma unroll
        for (int kk = 0; kk < DH / 16; ++kk)
          umma2(T_S(h), desc_k(sq + (kk >> 2) * Q_SUB + (kk & 3) * 32), desc_k(sk + (kk >> 2) * K_SUB + (kk & 3) * 32),
                ID_S, kk > 0);
        commit_both(&s_full[h]);
        if (h == n_heads - 1) commit_both(&k_empty[j % K_STAGES]);
      };
      wait_k(0);
      for (int h = 0; h < n_heads; ++h) issue_s(0, h);
      for (int j = 0; j < n_kt; ++j) {
        const int st = j % V_STAGES;
        mbar_wait_cluster(&v_pair[st], (j / V_STAGES) & 1);
        tc_after();
        const uint32_t sv = smem_u32(smem + OFF_V + st * V_BYTES);
        if (j + 1 < n_kt) wait_k(j + 1);
        for (int h = 0; h < n_heads; ++h) {
          mbar_wait_cluster(&p_pair[h], j & 1);
          tc_after();
#pragma unroll
          for (int kk = 0; kk < BKV / 16; ++kk)  // 16 keys per k-step: A = P (TMEM, 8 columns), B = V half
            umma2_ts(T_O(h), T_S(h) + kk * 8, desc_mn(sv + kk * 16 * 128), ID_PV, (j > 0 || kk > 0));
          if (j == n_kt - 1) commit_both(&o_done[h]);
          if (h == n_heads - 1) commit_both(&v_empty[st]);
          if (j + 1 < n_kt) issue_s(j + 1, h);
        }
      }
    }
  } else {
    // ---------------- softmax warps of this CTA: one thread per query row
    const int h = (warp - 2) >> 2;
    if (h < n_heads) {
      const int quad = warp & 3;
      const int r = quad * 32 + lane;
      const int pos = min(cpre + q0 + r, kv_end - 1);  // rows past the chunk clamp (never stored)
      const float sc = rsqrtf((float)DH) * 1.4426950408889634f;
      const uint32_t lane_base = (uint32_t)(quad * 32) << 16;
      const uint32_t t_s = T_S(h) + lane_base;
      const uint32_t p_leader = leader_addr(&p_pair[h]);
      float m_used = -INFINITY, l = 0.f;
      for (int j = 0; j < n_kt; ++j) {
        mbar_wait(&s_full[h], j & 1);
        tc_after();
        const int lim = pos - j * BKV;  // keys 0..lim of this tile are visible to this row
        const bool full_tile = lim >= BKV - 1;
        float mx = -INFINITY;
#pragma unroll 1
        for (int c = 0; c < 2; ++c) {
          uint32_t v0[32], v1[32];
          tmem_ld32x2(t_s + c * 64, t_s + c * 64 + 32, v0, v1);
          if (full_tile) {
#pragma unroll
            for (int e = 0; e < 32; e += 2)
              mx = fmaxf(mx, fmaxf(fmaxf(__uint_as_float(v0[e]), __uint_as_float(v0[e + 1])),
                                   fmaxf(__uint_as_float(v1[e]), __uint_as_float(v1[e + 1]))));
          } else {
#pragma unroll
            for (int e = 0; e < 32; ++e) {
              if (c * 64 + e <= lim) mx = fmaxf(mx, __uint_as_float(v0[e]));
              if (c * 64 + 32 + e <= lim) mx = fmaxf(mx, __uint_as_float(v1[e]));
            }
          }
        }
        const float m_new = fmaxf(m_used, mx * sc);
        const bool mine = m_new > m_used + RESCALE_THRESHOLD;
        if (__any_sync(0xffffffffu, mine)) {
          if (j >= 1) {
            const float f = mine ? exp2f(m_used - m_new) : 1.f;
            l *= f;
#pragma unroll 1
            for (int c = 0; c < DH; c += 32) {
              uint32_t v[32];
              tmem_ld32(T_O(h) + lane_base + c, v);
#pragma unroll
              for (int e = 0; e < 32; ++e) v[e] = __float_as_uint(__uint_as_float(v[e]) * f);
              tmem_st32(T_O(h) + lane_base + c, v);
            }
          }
          if (mine) m_used = m_new;
        }
        float l0 = 0.f, l1 = 0.f;
#pragma unroll 1
        for (int c = 0; c < 2; ++c) {
          uint32_t v0[32], v1[32], pk[32];
          tmem_ld32x2(t_s + c * 64, t_s + c * 64 + 32, v0, v1);
          if (full_tile) {
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
          } else {
#pragma unroll
            for (int hh = 0; hh < 2; ++hh) {
#pragma unroll
              for (int e = 0; e < 32; e += 2) {
                const float s0 = __uint_as_float(hh ? v1[e] : v0[e]), s1 = __uint_as_float(hh ? v1[e + 1] : v0[e + 1]);
                const int k0 = c * 64 + hh * 32 + e;
                const float p0 = (k0 <= lim) ? fast_exp2(fmaf(s0, sc, -m_used)) : 0.f;
                const float p1 = (k0 + 1 <= lim) ? fast_exp2(fmaf(s1, sc, -m_used)) : 0.f;
                l0 += p0;
                l1 += p1;
                __nv_bfloat162 t2 = __floats2bfloat162_rn(p0, p1);
                pk[hh * 16 + e / 2] = *reinterpret_cast<uint32_t*>(&t2);
              }
            }
          }
          tmem_st32(t_s + c * 32, pk);
        }
        l += l0 + l1;
        tc_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_remote(p_leader);
      }
      pdl_trigger();
      mbar_wait(&o_done[h], 0);
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
    }
  }
  tc_before();
  cluster_sync();  // no CTA leaves while its peer may still signal its barriers or its MMAs run
  if (warp == 1) {
    tc_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(TMEM_COLS));
  }
}

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
static bool make_map(CUtensorMap* m, const void* base, uint64_t rows, uint64_t cols, uint64_t ld_elems) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {cols, rows};
  cuuint64_t strides[1] = {ld_elems * 2};
  cuuint32_t box[2] = {64, (cuuint32_t)BQ};
  cuuint32_t es[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

}  // namespace fa2

bool fa2_tc_supported(const PrefillAttnArgs& a) {
  // opt-in (DUET_FA2=1) until it beats the one-CTA kernel: 0.81x of it at q = 8192, 0.8x at q = 2048
  // (profiles/r02_fa2_pair_ab.txt)
  static const bool on = getenv("DUET_FA2") && atoi(getenv("DUET_FA2")) != 0;
  return on && a.dh == fa2::DH && a.page_size == fa2::PAGE && a.q_stride % 8 == 0 && fa2::encode_fn() != nullptr &&
         a.total_rows > 0 && a.num_sms >= 2 && ((uintptr_t)a.q & 15) == 0;
}

int launch_fa2_tc(const PrefillAttnArgs& a, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(fa2::fa2_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, fa2::SMEM);
    attr = true;
  }
  CUtensorMap mq;
  if (!fa2::make_map(&mq, a.q, (uint64_t)a.total_rows, (uint64_t)a.q_stride, (uint64_t)a.q_stride)) return -1;
  fa2::Params p{a.row0, a.qlen, a.cpre, a.seq_row, a.table, a.max_pages, a.hq, a.hkv, 0, 0,
                (bf16*)a.o, (const bf16*)a.k_pool, (const bf16*)a.v_pool};
  const int G = a.hq / a.hkv;
  p.n_qblocks = (a.max_q + 2 * fa2::BQ - 1) / (2 * fa2::BQ);
  p.n_pairs = a.hkv * ((G + 1) / 2);
  dim3 grid(2 * p.n_pairs, p.n_qblocks, a.n_seqs);
  launch_pdl(fa2::fa2_kernel, grid, fa2::THREADS, fa2::SMEM, st, mq, p);
  return 1;
}

}  // namespace duet

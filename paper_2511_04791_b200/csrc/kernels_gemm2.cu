// CTA-pair (cta_group::2) tcgen05 GEMM for the token-major linear operators of the layer when the
// batch has more than 128 rows (prefill chunks, temporal mode): QKV, O, gate-up + SwiGLU, down
// (§2, §4.1).  C[M][N] = epi(X[M][K] . W[N][K]^T), bf16 in, fp32 in TMEM.
//
// Two CTAs of a cluster (one TPC) compute a 256-row x 256-column tile with UMMA 256x256x16:
//   * each CTA TMA-loads its own 128 rows of X and its own 128 rows of W (for SwiGLU: CTA 0 the gate
//     rows, CTA 1 the matching up rows) into the same shared-memory offsets; both loads signal the
//     leader CTA's `full` mbarrier (.cta_group::2 TMA);
//   * the leader's single MMA thread issues tcgen05.mma.cta_group::2, which reads A from both CTAs'
//     shared memory (M halves) and B from both (N halves) and writes each CTA's 128 rows x 256
//     columns of fp32 into that CTA's TMEM; tcgen05.commit ... multicast::cluster frees the stage in
//     both CTAs and publishes the accumulator to both epilogues;
//   * each CTA's 4 epilogue warps drain their own TMEM rows and signal the leader's `tempty`.
// Per SM this halves the shared-memory operand traffic of the 1-CTA 128x256 tile (each UMMA reads
// 16 KiB per SM instead of 24 KiB per 128x256x16, and TMA writes 32 instead of 48 KiB per k-block),
// the limit of the 1-CTA kernel (profiles/r01_probe_umma_rate.txt, profiles/r01_ncu_full_cfg2.md).
// Tiles are assigned statically, every output is reduced over K in one fixed order.
// Tile width BN = 256 (UMMA 256x256x16) or 128 (UMMA 256x128x16, each CTA loads 64 W rows) — the
// narrow tile for grids the wide one leaves under-filled: a 256-row decode batch's O / down / QKV
// projections have 16-24 wide tiles for the 32-37 CTA pairs of a decode partition.  The choice
// depends on the shape only (split invariance); the per-element K order is the same for both.
#include <cuda.h>

#include <algorithm>
#include <cstdlib>

#include "dev_common.cuh"
#include "kernels.h"

namespace duet {
namespace tc2 {

constexpr int BM = 128, BK = 64, PAIR_M = 256;
constexpr int A_BYTES = BM * BK * 2;      // this CTA's 128 rows of X
template <int BN> struct Cfg {
  static constexpr int B_ROWS = BN / 2;                 // this CTA's rows of W
  static constexpr int B_BYTES = B_ROWS * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int STAGES = BN == 256 ? 6 : 8;
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 + 256;
  static constexpr int TMEM_COLS = 2 * BN;              // two accumulators
};
constexpr int THREADS = 192;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
// shared::cluster address of the same variable in CTA `rank` of the cluster
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
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
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
// TMA box into this CTA's shared memory, completion bytes counted on the leader CTA's mbarrier
__device__ __forceinline__ void tma_load_2cta(const CUtensorMap* map, uint32_t leader_bar, void* dst, int c0, int c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], "
      "[%2];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(leader_bar), "r"(c0), "r"(c1)
      : "memory");
}
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  return (uint64_t)((saddr & 0x3FFFF) >> 4) | ((uint64_t)1 << 16) | ((uint64_t)64 << 32) | ((uint64_t)1 << 46) |
         ((uint64_t)2 << 61);
}
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}
__device__ __forceinline__ void umma2(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                      uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate));
}
// arrive on the mbarrier at this offset in both CTAs once every earlier MMA of the pair completed
__device__ __forceinline__ void commit_both(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
          smem_u32(bar)),
      "h"((uint16_t)3)
      : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float (&v)[32]) {
  uint32_t r[32];
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,%17,%18,%19,"
      "%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
        "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]), "=r"(r[16]),
        "=r"(r[17]), "=r"(r[18]), "=r"(r[19]), "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]),
        "=r"(r[25]), "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
  for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

struct Params {
  int M, N, K;
  int num_m2, num_n, num_tiles;
  bf16* C;
  const bf16* R;
  const bf16* bias;
  int ldc, ldr;
  int n_up_off;  // SwiGLU: row offset of the up rows in W (= N)
  const bf16* R2;
  bf16* C2;
  int row_split;  // rows >= row_split: residual from R2, output to C2 (row - row_split)
  // EPI_QKV_ROPE (RoPE, reading #5; paged KV append before attention; C-3 slots)
  const int* pos;
  const int* tok_row;
  const int* table;
  int max_pages, hq, hkv;
  bf16* k_pool;
  bf16* v_pool;
  const float2* rope;
  // split-K (STORE / RESIDUAL epilogues of under-filled grids): work unit u = tile (u % num_tiles) x
  // K chunk (u / num_tiles) of kb_per k-blocks; chunk s writes fp32 partials to ws[s][M][N] and
  // gemm2_reduce_kernel sums the chunks in order 0..ksplit-1 and applies the epilogue
  int ksplit, kb_per;
  float* ws;
  // EPI_RESIDUAL_AR (f3): the tp group; emulation (ar.emul) runs rank r on pairs [r ppr, (r + 1) ppr) and
  // reads its operands at X rows r * xrows and W rows r * wrows of the stacked inputs
  GemmAr ar;
  int ar_ppr, ar_xrows, ar_wrows;
  const int* m_dev;  // nullable: rows from device memory (M is then the capacity)
};

// system-scope release / acquire on the counters of the fused allreduce (peer memory over NVLink)
__device__ __forceinline__ void red_release_sys(unsigned* p, unsigned v) {
  asm volatile("red.release.sys.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire_sys(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_sys(unsigned* p, unsigned v) {
  asm volatile("st.relaxed.sys.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// Tile order (grouped rasterization): tiles run in groups of GROUP_M 256-row blocks; inside a group the
// row block varies fastest, so the pairs of one wave share a few weight column blocks (read once from
// HBM, multicast through L2) and revisit a bounded set of X row blocks (<= GROUP_M x 256 rows, which
// stays L2-resident).  With the plain row-fastest order over all rows an X larger than L2 — the down
// projection's 8192 x 14336 activation at cfg3, 235 MB — was re-read from HBM for every column block
// (profiles/ncu_traffic.json: 1.34x the algorithmic bytes at cfg2, ~16x X at cfg3).
constexpr int GROUP_M = 8;
__device__ __forceinline__ void tile_coords(int t, int num_m2, int num_n, int& mp, int& nb) {
  const int g = t / (GROUP_M * num_n);
  const int first = g * GROUP_M;
  const int gm = min(num_m2 - first, GROUP_M);
  const int local = t - g * GROUP_M * num_n;
  mp = first + local % gm;
  nb = local / gm;
}

// PROD = 2: the X tiles and the W tiles are requested by two producer warps (0 and 6); PROD = 4: four
// (X even / odd k-blocks: warps 0 / 7, W: 6 / 8).  One TMA-issuing thread streams ~55 GB/s per SM
// (~0.28 us per box, profiles/r01_probe_tma_bw.txt): a narrow (128-column) tile's k-block needs 24 KiB in
// 0.18 us of MMA, so the 256-row decode GEMMs ran TMA-issue-bound at 31-47 % tensor pipe (ncu)
template <int EPI, int BN, int PROD>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(THREADS + (PROD - 1) * 32, 1)
    gemm2_kernel(const __grid_constant__ CUtensorMap map_x, const __grid_constant__ CUtensorMap map_w, Params p) {
  using CF = Cfg<BN>;
  constexpr int STAGES = CF::STAGES, STAGE_BYTES = CF::STAGE_BYTES, B_BYTES = CF::B_BYTES, B_ROWS = CF::B_ROWS;
  constexpr int TMEM_COLS = CF::TMEM_COLS, BN_PAIR = BN;
  constexpr int OUT_COLS = EPI == EPI_SWIGLU ? BN / 2 : BN;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * A_BYTES;
  uint64_t* full = (uint64_t*)(smem + STAGES * STAGE_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = (uint32_t*)(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t rank = cluster_rank();
  const bool leader = rank == 0;
  int pair = blockIdx.x >> 1, n_pairs = gridDim.x >> 1;
  // EPI_RESIDUAL_AR: this CTA's rank (emulation: the grid holds every rank's pairs) and the row offsets
  // of that rank's operands in the stacked X / W
  int ar_r = 0, xoff = 0, woff = 0;
  if constexpr (EPI == EPI_RESIDUAL_AR) {
    if (p.ar.emul) {
      ar_r = pair / p.ar_ppr;
      pair -= ar_r * p.ar_ppr;
      n_pairs = p.ar_ppr;
      xoff = ar_r * p.ar_xrows;
      woff = ar_r * p.ar_wrows;
    } else {
      ar_r = p.ar.rank;
    }
  }
  const int num_k = p.K / BK;
  // device-side row count (the prefill side's graph replays for any chunk size, f4; Params.m_dev): p.M is
  // then the buffers' capacity (TMA maps, grid), the rows this launch covers are read after the previous
  // kernels' writes are visible
  int M_ = p.M, num_m2_ = p.num_m2, num_tiles_ = p.num_tiles;
  if (p.m_dev) {
    pdl_wait();
    M_ = *p.m_dev;
    num_m2_ = (M_ + PAIR_M - 1) / PAIR_M;
    num_tiles_ = num_m2_ * p.num_n;
  }
  const int num_units = num_tiles_ * p.ksplit;

  if (warp == 0 && lane == 0) {
    for (int i = 0; i < STAGES; ++i) {
      mbar_init(&full[i], 1);   // leader: its producer's expect_tx (bytes of both CTAs)
      mbar_init(&empty[i], 1);  // both: the leader's multicast commit
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 8);  // leader: 4 local + 4 peer epilogue warps
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "n"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;");
  }
  tc_fence_before();
  cluster_sync();  // barriers initialised and TMEM allocated in both CTAs before any remote access
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // set-up above overlaps the previous kernel's tail; its outputs are read below.  The producer waits
  // later: the weights (never written by an earlier kernel) of its first stages are requested first.
  // producer roles (PROD >= 2): warp 0 / 7 request X tiles, warp 6 / 8 W tiles; with PROD = 4 each of a
  // pair takes the k-blocks of one parity (every box costs its issuing thread ~0.28 us, a narrow tile's
  // k-block only ~0.18 us of MMA)
  int role = -1, par = -1;  // role 0 = X (+ the leader's expect_tx), 1 = W; par = k-block parity (-1: all)
  if (PROD >= 2) {
    if (warp == 0) { role = 0; par = PROD == 4 ? 0 : -1; }
    else if (warp == 6) { role = 1; par = PROD == 4 ? 0 : -1; }
    else if (PROD == 4 && warp == 7) { role = 0; par = 1; }
    else if (PROD == 4 && warp == 8) { role = 1; par = 1; }
  }
  if (warp != 0 && role < 0) pdl_wait();

  auto w_row_of = [&](int nb) {
    return EPI == EPI_SWIGLU ? (rank ? p.n_up_off : 0) + nb * B_ROWS : woff + nb * BN_PAIR + (int)rank * B_ROWS;
  };
  if (role >= 0) {
    if (lane == 0) {
      // ---------------- X producer(s): X tiles + the leader's expect_tx of both CTAs' stage bytes;
      // W producer(s): weight tiles only — weights are never written by an earlier kernel, so no
      // pdl_wait (a W tile may land before the stage's expect_tx: the tx count goes transiently negative)
      asm volatile("prefetch.tensormap [%0];" ::"l"(role == 0 ? &map_x : &map_w) : "memory");
      if (role == 0) pdl_wait();
      int s = 0;
      uint32_t ph = 0, g = 0;
      for (int u = pair; u < num_units; u += n_pairs) {
        const int t = u % num_tiles_, kb0 = (u / num_tiles_) * p.kb_per, kb1 = min(num_k, kb0 + p.kb_per);
        int mp, nb;
        tile_coords(t, num_m2_, p.num_n, mp, nb);
        const int row_x = xoff + mp * PAIR_M + (int)rank * BM;
        const int row_w = w_row_of(nb);
        for (int kb = kb0; kb < kb1; ++kb, ++g) {
          if (par < 0 || (int)(g & 1) == par) {
            mbar_wait(&empty[s], ph ^ 1);
            const uint32_t lbar = mapa(smem_u32(&full[s]), 0);
            if (role == 0) {
              if (leader) mbar_expect_tx(&full[s], 2 * STAGE_BYTES);
              tma_load_2cta(&map_x, lbar, sA + s * A_BYTES, kb * BK, row_x);
            } else {
              tma_load_2cta(&map_w, lbar, sB + s * B_BYTES, kb * BK, row_w);
            }
          }
          if (++s == STAGES) {
            s = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (warp == 0) {
    if (lane == 0) {
      // ---------------- TMA producer (both CTAs): own X rows and own W rows; leader's `full` counts both
      asm volatile("prefetch.tensormap [%0];" ::"l"(&map_x) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(&map_w) : "memory");
      auto w_row = [&](int nb) {
        return EPI == EPI_SWIGLU ? (rank ? p.n_up_off : 0) + nb * B_ROWS : woff + nb * BN_PAIR + (int)rank * B_ROWS;
      };
      int pre = 0;
#ifndef DUET_NO_WPREFETCH
      if (pair < num_units && !p.m_dev) {  // fresh ring: the first STAGES stages are free
        const int kb00 = (pair / num_tiles_) * p.kb_per;
        const int nkb0 = min(num_k, kb00 + p.kb_per) - kb00;
        pre = nkb0 < STAGES ? nkb0 : STAGES;
        int mp0, nb0;
        tile_coords(pair % num_tiles_, num_m2_, p.num_n, mp0, nb0);
        const int row_w0 = w_row(nb0);
        for (int i = 0; i < pre; ++i) {
          if (leader) mbar_expect_tx(&full[i], 2 * STAGE_BYTES);
          tma_load_2cta(&map_w, mapa(smem_u32(&full[i]), 0), sB + i * B_BYTES, (kb00 + i) * BK, row_w0);
        }
      }
#endif
      pdl_wait();
      int s = 0;
      uint32_t ph = 0;
      for (int u = pair; u < num_units; u += n_pairs) {
        const int t = u % num_tiles_, kb0 = (u / num_tiles_) * p.kb_per, kb1 = min(num_k, kb0 + p.kb_per);
        int mp, nb;
        tile_coords(t, num_m2_, p.num_n, mp, nb);
        const int row_x = xoff + mp * PAIR_M + (int)rank * BM;
        const int row_w = w_row(nb);
        for (int kb = kb0; kb < kb1; ++kb) {
          const uint32_t lbar = mapa(smem_u32(&full[s]), 0);
          if (u == pair && kb - kb0 < pre) {  // weights already requested before pdl_wait
            tma_load_2cta(&map_x, lbar, sA + s * A_BYTES, kb * BK, row_x);
          } else {
            mbar_wait(&empty[s], ph ^ 1);
            if (leader) mbar_expect_tx(&full[s], 2 * STAGE_BYTES);
            tma_load_2cta(&map_x, lbar, sA + s * A_BYTES, kb * BK, row_x);
            tma_load_2cta(&map_w, lbar, sB + s * B_BYTES, kb * BK, row_w);
          }
          if (++s == STAGES) {
            s = 0;
            ph ^= 1;
          }
        }
      }
    }
  } else if (warp == 1) {
    if (leader && lane == 0) {
      // ---------------- MMA issuer (leader only): UMMA 256 x 256 x 16 over the CTA pair
      constexpr uint32_t idesc = idesc_bf16(PAIR_M, BN_PAIR);
      int s = 0;
      uint32_t ph = 0;
      int i = 0;
      for (int u = pair; u < num_units; u += n_pairs, ++i) {
        const int kb0 = (u / num_tiles_) * p.kb_per, kb1 = min(num_k, kb0 + p.kb_per);
        const int acc = i & 1;
        mbar_wait(&tempty[acc], ((i >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * BN_PAIR;
        for (int kb = kb0; kb < kb1; ++kb) {
          mbar_wait(&full[s], ph);
          tc_fence_after();
          const uint32_t a0 = smem_u32(sA + s * A_BYTES), b0 = smem_u32(sB + s * B_BYTES);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k)
            umma2(d_tmem, sw128_desc(a0 + k * 32), sw128_desc(b0 + k * 32), idesc, (kb != kb0 || k != 0));
          commit_both(&empty[s]);
          if (++s == STAGES) {
            s = 0;
            ph ^= 1;
          }
        }
        commit_both(&tfull[acc]);
      }
    }
  } else if (warp >= 2 && warp <= 5) {
    // ---------------- epilogue warps 2..5 (both CTAs): this CTA's 128 rows, TMEM quadrant = warp % 4
    const int quad = warp & 3;
    const int lane_row = quad * 32 + lane;
    const uint32_t leader_tempty0 = mapa(smem_u32(&tempty[0]), 0);
    int i = 0;
    for (int u = pair; u < num_units; u += n_pairs, ++i) {
      const int t = u % num_tiles_, sk = u / num_tiles_;
      const int acc = i & 1;
      int mp, nb;
      tile_coords(t, num_m2_, p.num_n, mp, nb);
      // EPI_QKV_ROPE: this row's position, KV page and cos/sin row are fetched while the tile's MMAs
      // still run (the dependent pos -> table / rope loads are off the epilogue's critical path)
      int r_pos = 0, r_page = 0;
      if constexpr (EPI == EPI_QKV_ROPE) {
        const int row_ = mp * PAIR_M + (int)rank * BM + quad * 32 + lane;
        if (row_ < M_) {
          r_pos = p.pos[row_];
          r_page = p.table[(size_t)p.tok_row[row_] * p.max_pages + (r_pos >> 4)];
          const char* cs_ = reinterpret_cast<const char*>(p.rope + (size_t)r_pos * 64);
#pragma unroll
          for (int j = 0; j < 4; ++j) asm volatile("prefetch.global.L1 [%0];" ::"l"(cs_ + j * 128));
        }
      }
      mbar_wait(&tfull[acc], (i >> 1) & 1);
      if (u + n_pairs >= num_units) pdl_trigger();  // last unit: only the epilogue is left
      tc_fence_after();
      const uint32_t tbase = tmem_base + ((uint32_t)(quad * 32) << 16) + acc * BN_PAIR;
      const int row = mp * PAIR_M + (int)rank * BM + lane_row;
      const int n0 = nb * OUT_COLS;
      if constexpr (EPI == EPI_STORE || EPI == EPI_RESIDUAL) {
        if (p.ksplit > 1) {  // fp32 partial of K chunk sk; the reduce kernel applies the epilogue
#pragma unroll 1
          for (int c = 0; c < OUT_COLS; c += 32) {
            float v[32];
            tmem_ld32(tbase + c, v);
            if (row < M_ && n0 + c < p.N) {
              float* dst = p.ws + ((size_t)sk * M_ + row) * p.N + n0 + c;
              if (n0 + c + 32 <= p.N) {
#pragma unroll
                for (int q = 0; q < 8; ++q)
                  *reinterpret_cast<float4*>(dst + 4 * q) = make_float4(v[4 * q], v[4 * q + 1], v[4 * q + 2], v[4 * q + 3]);
              } else {
#pragma unroll
                for (int e = 0; e < 32; ++e)
                  if (n0 + c + e < p.N) dst[e] = v[e];
              }
            }
          }
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive_cluster(leader_tempty0 + acc * 8);
          continue;
        }
      }
      if constexpr (EPI == EPI_RESIDUAL_AR) {
        // f3: each tile belongs to one owner rank.  This warp's 32 rows x 256 columns of the partial either go to
        // the owner's receive slot (sender) or are summed with the n - 1 received partials (owner).
        // ownership rotates along each pair's unit sequence (owner = (i + pair) mod E), so every pair — on
        // every rank — does the owner's reduction on 1 / E of its tiles (owner = t mod E would leave a pair
        // owning all or none of its tiles whenever E divides the pair count); ot indexes the owner's slots
        const int E = p.ar.n, owner = (i + pair) % E, ot = (i / E) * n_pairs + pair;
        const int wslot = (int)rank * 4 + quad;       // 8 (CTA, warp) row groups per tile
        const int trow = (int)rank * BM + lane_row;   // row within the 256-row tile
        if (owner != ar_r) {
          // slot layout [column][row] (column-major tile): for each column the warp's 32 rows are one
          // coalesced 128-B segment, on the store here and on the owner's load
          float* dst = p.ar.slots[owner] + ((size_t)ot * E + ar_r) * PAIR_M * BN + trow;
#pragma unroll 1
          for (int c = 0; c < BN; c += 32) {
            float v[32];
            tmem_ld32(tbase + c, v);
#pragma unroll
            for (int e = 0; e < 32; ++e) __stcg(dst + (size_t)(c + e) * PAIR_M, v[e]);
          }
          // the warp's rows are ordered before lane 0's system-scope fence by the warp barrier (cumulativity),
          // one fence per warp and tile instead of one per lane
          __syncwarp();
          if (lane == 0) {
            __threadfence_system();
            red_release_sys(p.ar.cnt[owner] + (size_t)ot * 8 + wslot, 1u);
          }
        } else {
          unsigned* cnt = p.ar.cnt[ar_r] + (size_t)ot * 8 + wslot;
          if (lane == 0) {
            while (ld_acquire_sys(cnt) < (unsigned)(E - 1)) {
            }
            st_relaxed_sys(cnt, 0u);  // re-armed: no sender touches it again before this grid ends
          }
          __syncwarp();
          const bool row_ok = row < M_;
          const float* slot0 = p.ar.slots[ar_r] + (size_t)ot * E * PAIR_M * BN + trow;
#pragma unroll 1
          for (int c = 0; c < BN; c += 32) {
            float v[32], sum[32];
            tmem_ld32(tbase + c, v);
#pragma unroll
            for (int e = 0; e < 32; ++e) sum[e] = 0.f;
            for (int sr = 0; sr < E; ++sr) {  // fixed rank order: every rank receives the same sum
              if (sr == ar_r) {
#pragma unroll
                for (int e = 0; e < 32; ++e) sum[e] += v[e];
              } else {
                const float* src = slot0 + (size_t)sr * PAIR_M * BN + (size_t)c * PAIR_M;
                float f[32];
#pragma unroll
                for (int e = 0; e < 32; ++e) f[e] = __ldcg(src + (size_t)e * PAIR_M);
#pragma unroll
                for (int e = 0; e < 32; ++e) sum[e] += f[e];
              }
            }
            const bool col_ok = row_ok && n0 + c < p.N;  // N % 32 == 0 (gemm2_supported)
            if (col_ok) {
              const bf16* rsrc = p.R + (size_t)row * p.ldr + n0 + c;
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                float rf[8];
                load16<bf16>(rsrc + q * 8, rf);
#pragma unroll
                for (int e = 0; e < 8; ++e) sum[q * 8 + e] += rf[e];
              }
              for (int dr = 0; dr < E; ++dr) {  // all-gather by push
                bf16* dst = (bf16*)p.ar.out[dr] + (size_t)row * p.ldc + n0 + c;
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                  float o8[8];
#pragma unroll
                  for (int e = 0; e < 8; ++e) o8[e] = sum[q * 8 + e];
                  store16<bf16>(dst + q * 8, o8);
                }
              }
            }
          }
          __syncwarp();
          if (lane == 0) {
            __threadfence_system();
            for (int dr = 0; dr < E; ++dr) red_release_sys(p.ar.done[dr], 1u);
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(leader_tempty0 + acc * 8);
        continue;
      }
      if constexpr (EPI == EPI_QKV_ROPE) {
        // the tile's BN columns are BN / 128 whole heads (d_h = 128): rotate (i, i + 64) pairs of q and k
        // heads at this row's position; q stays in C, k and v go to their KV slots
        {  // tcgen05.ld is warp-collective: every lane loads, only rows < M store
          const bool row_ok = row < M_;
          const int pos = r_pos;
          const int page = r_page;
          const int slot = pos & 15;
          const float2* cs = p.rope + (size_t)pos * 64;
#pragma unroll 1
          for (int hh = 0; hh < BN / 128; ++hh) {
            const int head = (n0 >> 7) + hh;
            if (head * 128 >= p.N) break;
            const bool is_q = head < p.hq, is_k = !is_q && head < p.hq + p.hkv;
            bf16* dst = is_q ? p.C + (size_t)row * p.ldc + head * 128
                             : (is_k ? p.k_pool : p.v_pool) +
                                   (((size_t)page * p.hkv + (head - p.hq - (is_k ? 0 : p.hkv))) * 16 + slot) * 128;
#pragma unroll 1
            for (int c = 0; c < 64; c += 32) {
              float x0[32], x1[32];
              tmem_ld32(tbase + hh * 128 + c, x0);
              tmem_ld32(tbase + hh * 128 + 64 + c, x1);
              if (p.bias) {
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                  float b0[8], b1[8];
                  load16<bf16>(p.bias + head * 128 + c + q * 8, b0);
                  load16<bf16>(p.bias + head * 128 + 64 + c + q * 8, b1);
#pragma unroll
                  for (int e = 0; e < 8; ++e) {
                    x0[q * 8 + e] += b0[e];
                    x1[q * 8 + e] += b1[e];
                  }
                }
              }
              if (head < p.hq + p.hkv) {
#pragma unroll
                for (int e = 0; e < 32; e += 2) {  // two (cos, sin) pairs per 16-B load
                  const float4 r = __ldg(reinterpret_cast<const float4*>(cs + c + e));
                  const float a0 = x0[e], b0 = x1[e], a1 = x0[e + 1], b1 = x1[e + 1];
                  x0[e] = a0 * r.x - b0 * r.y;
                  x1[e] = b0 * r.x + a0 * r.y;
                  x0[e + 1] = a1 * r.z - b1 * r.w;
                  x1[e + 1] = b1 * r.z + a1 * r.w;
                }
              }
              if (row_ok) {
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                  float o0[8], o1[8];
#pragma unroll
                  for (int e = 0; e < 8; ++e) {
                    o0[e] = x0[q * 8 + e];
                    o1[e] = x1[q * 8 + e];
                  }
                  store16<bf16>(dst + c + q * 8, o0);
                  store16<bf16>(dst + 64 + c + q * 8, o1);
                }
              }
            }
          }
        }
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive_cluster(leader_tempty0 + acc * 8);
        continue;
      }
#pragma unroll 1
      for (int c = 0; c < OUT_COLS; c += 32) {
        float v[32];
        tmem_ld32(tbase + c, v);
        if constexpr (EPI == EPI_SWIGLU) {
          float u[32];
          tmem_ld32(tbase + OUT_COLS + c, u);  // up columns follow the gate columns
#pragma unroll
          for (int e = 0; e < 32; ++e) v[e] = silu_f(v[e]) * u[e];
        }
        if (row < M_ && n0 + c < p.N) {
          const bool hi = row >= p.row_split;
          const int rrow = hi ? row - p.row_split : row;
          bf16* dst = (hi ? p.C2 : p.C) + (size_t)rrow * p.ldc + n0 + c;
          const bf16* rbase = hi ? p.R2 : p.R;
          if (n0 + c + 32 <= p.N) {
            if constexpr (EPI == EPI_RESIDUAL) {
              const bf16* rsrc = rbase + (size_t)rrow * p.ldr + n0 + c;
#pragma unroll
              for (int q = 0; q < 4; ++q) {
                float rf[8];
                load16<bf16>(rsrc + q * 8, rf);
#pragma unroll
                for (int e = 0; e < 8; ++e) v[q * 8 + e] += rf[e];
              }
            } else if constexpr (EPI == EPI_STORE) {
              if (p.bias) {
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                  float bf[8];
                  load16<bf16>(p.bias + n0 + c + q * 8, bf);
#pragma unroll
                  for (int e = 0; e < 8; ++e) v[q * 8 + e] += bf[e];
                }
              }
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              float o8[8];
#pragma unroll
              for (int e = 0; e < 8; ++e) o8[e] = v[q * 8 + e];
              store16<bf16>(dst + q * 8, o8);
            }
          } else {
#pragma unroll
            for (int e = 0; e < 32; ++e) {
              if (n0 + c + e >= p.N) continue;
              float o = v[e];
              if constexpr (EPI == EPI_RESIDUAL) o += __bfloat162float(rbase[(size_t)rrow * p.ldr + n0 + c + e]);
              if constexpr (EPI == EPI_STORE)
                if (p.bias) o += __bfloat162float(p.bias[n0 + c + e]);
              dst[e] = __float2bfloat16_rn(o);
            }
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive_cluster(leader_tempty0 + acc * 8);  // the leader's tempty[acc]
    }
  }
  if constexpr (EPI == EPI_RESIDUAL_AR) {
    // one CTA per rank holds the grid open until every tile of the result has arrived in this rank's output
    // (pushed by the tiles' owners), then re-arms the counter for the next launch
    if (warp == 2 && lane == 0 && rank == 0 && pair == 0) {
      unsigned* d = p.ar.done[ar_r];
      while (ld_acquire_sys(d) < (unsigned)(num_tiles_ * 8)) {
      }
      st_relaxed_sys(d, 0u);
    }
  }
  tc_fence_before();
  cluster_sync();  // no CTA leaves while its peer may still signal its barriers or read its smem
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "n"(TMEM_COLS));
  }
}

// Split-K reduction + epilogue: every thread sums 8 consecutive outputs over the K chunks in order
// 0..ksplit-1 (fixed order: results do not depend on the grid) and applies bias / residual.
template <int EPI>
__global__ void __launch_bounds__(256) gemm2_reduce_kernel(Params p) {
  pdl_wait();
  const int n8 = p.N / 8;
  const long idx = (long)blockIdx.x * blockDim.x + threadIdx.x;
  if (idx >= (long)p.M * n8) return;
  const int row = (int)(idx / n8), col = (int)(idx % n8) * 8;
  float v[8];
  {
    const float* src = p.ws + (size_t)row * p.N + col;
    const float4 a = __ldcg(reinterpret_cast<const float4*>(src)), b = __ldcg(reinterpret_cast<const float4*>(src + 4));
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w; v[4] = b.x; v[5] = b.y; v[6] = b.z; v[7] = b.w;
  }
  for (int s = 1; s < p.ksplit; ++s) {
    const float* src = p.ws + ((size_t)s * p.M + row) * p.N + col;
    const float4 a = __ldcg(reinterpret_cast<const float4*>(src)), b = __ldcg(reinterpret_cast<const float4*>(src + 4));
    v[0] += a.x; v[1] += a.y; v[2] += a.z; v[3] += a.w; v[4] += b.x; v[5] += b.y; v[6] += b.z; v[7] += b.w;
  }
  const bool hi = row >= p.row_split;
  const int rrow = hi ? row - p.row_split : row;
  if constexpr (EPI == EPI_RESIDUAL) {
    float r[8];
    load16<bf16>((hi ? p.R2 : p.R) + (size_t)rrow * p.ldr + col, r);
#pragma unroll
    for (int e = 0; e < 8; ++e) v[e] += r[e];
  } else if (p.bias) {
    float b[8];
    load16<bf16>(p.bias + col, b);
#pragma unroll
    for (int e = 0; e < 8; ++e) v[e] += b[e];
  }
  store16<bf16>((hi ? p.C2 : p.C) + (size_t)rrow * p.ldc + col, v);
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
static bool make_map(CUtensorMap* m, const void* base, int rows, int cols, int ld, int box_rows) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 2};
  cuuint32_t box[2] = {(cuuint32_t)BK, (cuuint32_t)box_rows};
  cuuint32_t es[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// K chunks for an under-filled grid, from the shape alone (split invariance): a STORE / RESIDUAL GEMM
// with fewer tiles than the full device has CTA pairs (74) is cut into ceil(74 / tiles) <= 8 chunks of
// >= 8 k-blocks — e.g. the 256-row decode batch's O and down projections (32 narrow tiles, a second
// wave of 4 tiles on a 56-SM partition) — provided the caller's workspace holds the fp32 partials.
static int splitk_count(int epi, int tiles, int num_k, int M, int N, const float* ws, size_t ws_floats) {
  static const bool off = getenv("DUET_GEMM2_SPLITK") && atoi(getenv("DUET_GEMM2_SPLITK")) == 0;
  // DUET_GEMM2_SPLIT_UNITS: work units aimed at (A/B; <= 148, the workspace is sized for 148)
  static const int target = getenv("DUET_GEMM2_SPLIT_UNITS") ? std::min(148, atoi(getenv("DUET_GEMM2_SPLIT_UNITS"))) : 74;
  if (off || !ws || (epi != EPI_STORE && epi != EPI_RESIDUAL) || tiles >= 74 || N % 8) return 1;
  int ks = (target + tiles - 1) / tiles;
  if (ks > 8) ks = 8;
  while (ks > 1 && num_k / ks < 8) --ks;
  if (ks > 1 && (size_t)ks * M * N > ws_floats) return 1;
  return ks;
}

template <int EPI, int BN, int PROD>
static int launch(const GemmArgs& a, int num_sms, cudaStream_t st) {
  using CF = Cfg<BN>;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(gemm2_kernel<EPI, BN, PROD>, cudaFuncAttributeMaxDynamicSharedMemorySize, CF::SMEM);
    attr = true;
  }
  CUtensorMap mx, mw;
  // f3 emulation: the E ranks' X and W are stacked row-wise ([E][M][K], [E][N][K])
  const int n_emul = (EPI == EPI_RESIDUAL_AR && a.ar && a.ar->emul) ? a.ar->n : 1;
  const int w_rows = EPI == EPI_SWIGLU ? 2 * a.N : a.N * n_emul;
  if (!make_map(&mx, a.A, a.M * n_emul, a.K, a.lda, BM) || !make_map(&mw, a.B, w_rows, a.K, a.ldb, CF::B_ROWS))
    return -1;
  Params p{};
  p.M = a.M;
  p.N = a.N;
  p.K = a.K;
  p.num_m2 = (a.M + PAIR_M - 1) / PAIR_M;
  constexpr int out_cols = EPI == EPI_SWIGLU ? BN / 2 : BN;
  p.num_n = (a.N + out_cols - 1) / out_cols;
  p.num_tiles = p.num_m2 * p.num_n;
  p.C = (bf16*)a.C;
  p.R = (const bf16*)a.R;
  p.bias = (const bf16*)a.bias;
  p.ldc = a.ldc;
  p.ldr = a.ldr;
  p.n_up_off = a.N;
  p.R2 = (const bf16*)a.R2;
  p.C2 = (bf16*)a.C2;
  p.row_split = a.row_split;
  if constexpr (EPI == EPI_QKV_ROPE) {
    p.pos = a.rope->pos;
    p.tok_row = a.rope->tok_row;
    p.table = a.rope->table;
    p.max_pages = a.rope->max_pages;
    p.hq = a.rope->hq;
    p.hkv = a.rope->hkv;
    p.k_pool = (bf16*)a.rope->k_pool;
    p.v_pool = (bf16*)a.rope->v_pool;
    p.rope = a.rope->rope;
  }
  const int num_k = a.K / BK;
  p.m_dev = a.m_dev;
  const int ks = a.m_dev ? 1 : splitk_count(EPI, p.num_tiles, num_k, a.M, a.N, a.ws, a.ws_floats);
  p.kb_per = (num_k + ks - 1) / ks;
  p.ksplit = (num_k + p.kb_per - 1) / p.kb_per;
  p.ws = a.ws;
  const int units = p.num_tiles * p.ksplit;
  int pairs = units < num_sms / 2 ? units : num_sms / 2;
  if constexpr (EPI == EPI_RESIDUAL_AR) {
    if (!a.ar || BN != 256 || p.ksplit != 1) return -1;
    p.ar = *a.ar;
    const int per_rank = n_emul > 1 ? std::min(units, num_sms / 2 / n_emul) : pairs;
    const int upp = (units + per_rank - 1) / per_rank;  // units of the busiest pair
    if ((size_t)((upp + a.ar->n - 1) / a.ar->n) * per_rank > a.ar->slot_tiles) return -1;  // owned-slot capacity
    if (n_emul > 1) {  // every emulated rank's pairs resident at once (their owners wait on each other)
      pairs = std::min(units, num_sms / 2 / n_emul);
      if (pairs < 1) return -1;
      p.ar_xrows = a.M;
      p.ar_wrows = a.N;
    }
    p.ar_ppr = pairs;
    pairs *= n_emul;
  }
  launch_pdl(gemm2_kernel<EPI, BN, PROD>, 2 * pairs, THREADS + (PROD - 1) * 32, CF::SMEM, st, mx, mw, p);
  if (p.ksplit > 1) {
    if constexpr (EPI == EPI_STORE || EPI == EPI_RESIDUAL) {
      const long n = (long)a.M * (a.N / 8);
      launch_pdl(gemm2_reduce_kernel<EPI>, (unsigned)((n + 255) / 256), 256, 0, st, p);
      return 2;
    }
  }
  return 1;
}

// Tile width: 256 by default — under-filled grids split K instead (splitk_count).  The 128-column tile
// (DUET_GEMM2_BN=128) fills more pairs but its k-block is half the MMA work for the same X tile: on the
// 256-row decode batch at 56 SMs the narrow tiles averaged 72.6 us per GEMM launch, the wide tiles with
// split-K 66.5 us (profiles/r02_gemm2_tile_ab.txt).  DUET_GEMM2_BN = 128 / 256 forces one width (A/B).
template <int EPI>
static int launch_w(const GemmArgs& a, int num_sms, cudaStream_t st) {
  if constexpr (EPI == EPI_RESIDUAL_AR) {
    return launch<EPI, 256, 2>(a, num_sms, st);  // 256 x 256 receive slots
  } else {
    static const int force = getenv("DUET_GEMM2_BN") ? atoi(getenv("DUET_GEMM2_BN")) : 0;
    const bool narrow = force == 128;
    // DUET_GEMM2_PROD = 1 / 2 / 4: producer warps (A/B); default 2 (4 measured equal, 1 within 1 %)
    static const int prod = getenv("DUET_GEMM2_PROD") ? atoi(getenv("DUET_GEMM2_PROD")) : 2;
    if (prod == 1) return narrow ? launch<EPI, 128, 1>(a, num_sms, st) : launch<EPI, 256, 1>(a, num_sms, st);
    if (prod == 4) return narrow ? launch<EPI, 128, 4>(a, num_sms, st) : launch<EPI, 256, 4>(a, num_sms, st);
    return narrow ? launch<EPI, 128, 2>(a, num_sms, st) : launch<EPI, 256, 2>(a, num_sms, st);
  }
}

}  // namespace tc2

size_t gemm2_splitk_need(int M, int N, int K, int epi) {
  if (M <= 128 || K % tc2::BK || (epi != EPI_STORE && epi != EPI_RESIDUAL) || N % 8) return 0;
  size_t need = 0;
  for (int cols : {128, 256}) {  // either tile width (DUET_GEMM2_BN may force one)
    const long tiles = (long)((M + tc2::PAIR_M - 1) / tc2::PAIR_M) * ((N + cols - 1) / cols);
    if (tiles >= 74) continue;
    int ks = (int)((148 + tiles - 1) / tiles);
    if (ks > 8) ks = 8;
    while (ks > 1 && (K / tc2::BK) / ks < 8) --ks;
    if (ks > 1) need = std::max(need, (size_t)ks * M * N);
  }
  return need;
}

size_t gemm_ar_slot_tiles(int M, int N, int n, int num_sms) {
  // the owner's slot index is (i / n) * pairs + pair for unit i of a pair: < ceil(ceil(tiles / P) / n) * P,
  // bounded over every grid size P <= num_sms / 2 by ceil(tiles / n) + 2 P
  const size_t tiles = (size_t)((M + tc2::PAIR_M - 1) / tc2::PAIR_M) * ((N + 255) / 256);
  return (tiles + n - 1) / n + (size_t)num_sms;
}
size_t gemm_ar_slot_floats(int M, int N, int n, int num_sms) {
  return gemm_ar_slot_tiles(M, N, n, num_sms) * n * tc2::PAIR_M * 256;
}
size_t gemm_ar_counters(int M, int N, int n, int num_sms) { return gemm_ar_slot_tiles(M, N, n, num_sms) * 8; }

bool gemm2_supported(const GemmArgs& a, int num_sms) {
  static const bool on = !getenv("DUET_GEMM2") || atoi(getenv("DUET_GEMM2")) != 0;  // A/B switch
  auto mis = [](const void* p) { return ((uintptr_t)p & 15) != 0; };  // TMA / 16-B epilogue alignment
  if (mis(a.A) || mis(a.B) || mis(a.C) || mis(a.R) || mis(a.R2) || mis(a.C2)) return false;
  if (a.epi == EPI_RESIDUAL_AR) {
    if (!a.ar || a.ar->n < 1 || a.ar->n > kMaxTp || !a.R || a.N % 32 || a.row_split < a.M || a.C2 || a.R2) return false;
    for (int r = 0; r < a.ar->n; ++r)
      if (!a.ar->slots[r] || !a.ar->cnt[r] || !a.ar->done[r] || !a.ar->out[r] || mis(a.ar->out[r])) return false;
  }
  return on && a.M > 128 && num_sms >= 2 && a.K % tc2::BK == 0 && a.lda % 8 == 0 && a.ldb % 8 == 0 &&
         a.ldc % 8 == 0 && (!a.R || a.ldr % 8 == 0) && (a.epi != EPI_SWIGLU || a.N % 128 == 0) &&
         (a.epi != EPI_QKV_ROPE || a.N % 128 == 0);
}

int launch_gemm2(const GemmArgs& a, int num_sms, cudaStream_t st) {
  if (a.epi == EPI_QKV_ROPE) return a.rope ? tc2::launch_w<EPI_QKV_ROPE>(a, num_sms, st) : -1;
  if (a.epi == EPI_SWIGLU) return tc2::launch_w<EPI_SWIGLU>(a, num_sms, st);
  if (a.epi == EPI_RESIDUAL) return tc2::launch_w<EPI_RESIDUAL>(a, num_sms, st);
  if (a.epi == EPI_RESIDUAL_AR) return tc2::launch_w<EPI_RESIDUAL_AR>(a, num_sms, st);
  return tc2::launch_w<EPI_STORE>(a, num_sms, st);
}

}  // namespace duet

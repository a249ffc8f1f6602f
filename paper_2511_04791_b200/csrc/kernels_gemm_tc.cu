// tcgen05 / TMEM / TMA GEMM for sm_100a — the token-level linear operators of the layer
// (QKV, O, gate-up, down; §2, §4.1), bf16 in, fp32 accumulation in
// tensor memory, fused epilogues (bias, residual add, SwiGLU).
//
// C[M][N] = epi(X[M][K] . W[N][K]^T), X (activations) and W (weights) K-major (nn.Linear layout).
// Persistent, warp-specialized, one CTA per SM (cta_group::1):
//   warp 0      TMA producer (SWIZZLE_128B tiles, S-stage mbarrier ring)
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer
//   warps 2..5  epilogue: tcgen05.ld (32 lanes x 32 columns) -> fused op -> global
// Two TMEM accumulators let the epilogue of tile i overlap the MMAs of tile i+1.
//
// Two orientations:
//   normal  (prefill, temporal; M > 128): UMMA 128 x BN x 16, the 128 TMEM lanes are 128 token rows,
//           columns are BN output features.
//   swap-AB (decode side, M <= 128): UMMA 128 x NT x 16 with the 128 lanes = 128 *weight rows* and
//           NT (64 or 128) columns = the tokens, so a skinny decode batch does not pad the MMA M
//           dimension to 128 — the decode GEMMs stay weight-streaming (HBM) bound on a small
//           partition.  SwiGLU in swap mode issues two MMAs per k-step (gate rows
//           and the matching up rows into two TMEM column ranges), so the epilogue is thread-local.
// Tiles are assigned statically (tile = blockIdx.x + j * gridDim.x) and every output element is
// reduced over K in one fixed order: results do not depend on the grid, i.e. on the SM partition.
#include <cuda.h>

#include <algorithm>
#include <cstdlib>

#include "dev_common.cuh"
#include "kernels.h"

namespace duet {

namespace tc {

constexpr int BM = 128, BK = 64;

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
__device__ __forceinline__ void tma_load_2d_hint(const CUtensorMap* map, uint64_t* bar, void* dst, int c0, int c1,
                                                 uint64_t policy) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1, {%3, %4}], "
      "[%2], %5;" ::"r"(smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "l"(policy)
      : "memory");
}
__device__ __forceinline__ void prefetch_map(const CUtensorMap* map) {
  asm volatile("prefetch.tensormap [%0];" ::"l"(map) : "memory");
}

// UMMA shared-memory descriptor: K-major, SWIZZLE_128B (rows of 128 B, 8-row atoms of 1 KiB):
// start >> 4 | LBO = 1 (unused for swizzled K-major) | SBO = 1024 B >> 4 | version 1 | layout 2.
__device__ __forceinline__ uint64_t sw128_desc(uint32_t saddr) {
  return (uint64_t)((saddr & 0x3FFFF) >> 4) | ((uint64_t)1 << 16) | ((uint64_t)64 << 32) | ((uint64_t)1 << 46) |
         ((uint64_t)2 << 61);
}

// Instruction descriptor, kind::f16: D = f32 (bits 4-5 = 1), A = B = bf16 (bits 7-9, 10-12 = 1),
// both K-major, N >> 3 at bits 17-22, M >> 4 at bits 24-28.
__host__ __device__ constexpr uint32_t idesc_bf16(int M, int N) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void umma_bf16(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc, uint32_t idesc,
                                          uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(d_tmem),
      "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate));
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }

// 32 lanes x 32 consecutive fp32 columns -> 32 registers per thread
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

// Tile configuration.
//   normal: smem A = 128 token rows, smem B = BN weight rows (SwiGLU: BN/2 gate + BN/2 up rows);
//           accumulator 128 x BN; output tile 128 x (SwiGLU ? BN/2 : BN).
//   swap:   smem A = 128 weight rows (SwiGLU: two such tiles, gate and up), smem B = BN token rows;
//           accumulator 128 x BN (SwiGLU: 2 x BN); output tile BN tokens x 128 features.
template <int BN, int EPI, bool SWAP>
struct Cfg {
  static constexpr int A_TILES = (SWAP && EPI == EPI_SWIGLU) ? 2 : 1;
  // swap mode streams weights from HBM on a possibly small SM partition.  A TMA instruction costs its
  // issuing thread ~0.1-0.25 us on B200 (profiles/r01_probe_tma_bw.txt: one issuer sustains ~60 GB/s
  // per SM, two exactly twice that), so swap tiles run two CTAs per SM with two producer warps each
  // (four issuers per SM) taking alternate pipeline stages.
  static constexpr int NPROD = SWAP ? 2 : 1;                 // producer warps: 0 (and 6)
  static constexpr int THREADS = 192 + (NPROD - 1) * 32;
  static constexpr int CTAS = SWAP ? 2 : 1;                  // CTAs per SM
  static constexpr int A_BYTES = A_TILES * BM * BK * 2;
  static constexpr int B_BYTES = BN * BK * 2;
  static constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr int SMEM_BUDGET = CTAS == 2 ? 104 * 1024 : 200 * 1024;
  static constexpr int STAGES = SMEM_BUDGET / STAGE_BYTES > 8 ? 8 : SMEM_BUDGET / STAGE_BYTES;
  static constexpr int ACC_COLS = (SWAP && EPI == EPI_SWIGLU) ? 2 * BN : BN;
  static constexpr int TMEM_COLS = 2 * ACC_COLS <= 32 ? 32 : (2 * ACC_COLS <= 64 ? 64 : (2 * ACC_COLS <= 128 ? 128 : (2 * ACC_COLS <= 256 ? 256 : 512)));
  static constexpr int SMEM = STAGES * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;
  static_assert(2 * ACC_COLS <= 512, "TMEM");
};

// Split-K (swap tiles only).  A skinny decode GEMM has only N/128 weight-row tiles (32 for the O and
// down projections of Llama-3-8B), fewer than the CTAs of even a 24-SM partition, so the K range is
// cut into `ksplit` chunks of `kb_per` 64-wide blocks: a work unit is (tile, chunk).  The chunking
// depends only on the GEMM shape — never on the grid — and each tile's fp32 partials are summed in
// chunk order 0..ksplit-1 by whichever CTA finishes the tile's last chunk, so results stay
// independent of the SM partition (and of arrival order).
constexpr int SPLITK_TARGET_UNITS = 148;   // >= one unit per SM of the full GPU; >= 3 per CTA on a 24-SM partition
constexpr int SPLITK_MIN_KB = 8;           // >= 512 of K per chunk
constexpr int SPLITK_MAX = 8;              // partial bytes <= ~15% of the weight bytes at Llama-3-8B shapes
constexpr int SPLITK_MAX_TILES = 40;       // split only tile-starved shapes (O, down: 32 tiles); with 48+
                                           // tiles (QKV, gate-up) the reduction costs more than it balances

struct Params {
  int M, N, K;        // C is M x N; N = output features (SwiGLU: width of act)
  int num_m, num_n, num_tiles;
  int ksplit, kb_per, num_units;
  bf16* C;
  const bf16* R;
  const bf16* bias;
  int ldc, ldr;
  int n_up_off;       // SwiGLU: row offset of the up rows in W (= N)
  float* ws;          // split-K partials [num_tiles][ksplit][ACC_COLS][128]
};

// swap-mode output: thread = feature n, 32 consecutive tokens m0..m0+31 (bias / residual fused)
template <int EPI, class P>
__device__ __forceinline__ void swap_store(const P& p, const float (&v)[32], int m0, int n) {
  float badd = 0.f;
  if constexpr (EPI == EPI_STORE)
    if (p.bias) badd = __bfloat162float(p.bias[n]);
#pragma unroll
  for (int e = 0; e < 32; ++e) {
    const int m = m0 + e;
    if (m < p.M) {
      float o = v[e];
      if constexpr (EPI == EPI_RESIDUAL) o += __bfloat162float(p.R[(size_t)m * p.ldr + n]);
      if constexpr (EPI == EPI_STORE) o += badd;
      p.C[(size_t)m * p.ldc + n] = __float2bfloat16_rn(o);
    }
  }
}

template <int BN, int EPI, bool SWAP>
__global__ void __launch_bounds__(Cfg<BN, EPI, SWAP>::THREADS, Cfg<BN, EPI, SWAP>::CTAS)
    gemm_tc_kernel(const __grid_constant__ CUtensorMap map_x, const __grid_constant__ CUtensorMap map_w, Params p) {
  using CF = Cfg<BN, EPI, SWAP>;
  constexpr int S = CF::STAGES;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint8_t* sA = smem;
  uint8_t* sB = smem + S * CF::A_BYTES;
  uint64_t* full = (uint64_t*)(smem + S * CF::STAGE_BYTES);
  uint64_t* empty = full + S;
  uint64_t* tfull = empty + S;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = (uint32_t*)(tempty + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int num_k = p.K / BK;
  // unit u -> tile u % num_tiles, K chunk u / num_tiles: blocks [kb0, kb1)
  auto unit_k = [&](int u, int& tile, int& kb0, int& kb1) {
    tile = u % p.num_tiles;
    const int ch = u / p.num_tiles;
    kb0 = ch * p.kb_per;
    kb1 = min(num_k, kb0 + p.kb_per);
  };

  if (warp == 0 && lane == 0) {
    prefetch_map(&map_x);
    prefetch_map(&map_w);
    for (int i = 0; i < S; ++i) {
      mbar_init(&full[i], 1);
      mbar_init(&empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&tfull[i], 1);
      mbar_init(&tempty[i], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tmem_slot)),
                 "n"(CF::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // set-up above overlaps the previous kernel's tail.  Producers wait later: the weight tiles of their
  // first ring pass (never written by an earlier kernel) are requested before the wait.
  if (!(warp == 0 || warp >= 6)) pdl_wait();

  if (warp == 0 || warp >= 6) {
    if (lane == 0) {
      // ---------------- TMA producer(s): producer `pr` issues the k-blocks it with it % NPROD == pr
      const int pr = warp == 0 ? 0 : warp - 5;
      uint64_t pol_w = 0;
      if constexpr (SWAP)  // weights are streamed once per step: evict-first keeps split-K partials in L2
        asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_w));
      auto load_w = [&](int s, int kb, int nb) {
        if constexpr (SWAP) {
          uint8_t* a_dst = sA + s * CF::A_BYTES;
          const int j0 = nb * BM;
          tma_load_2d_hint(&map_w, &full[s], a_dst, kb * BK, j0, pol_w);
          if constexpr (EPI == EPI_SWIGLU)
            tma_load_2d_hint(&map_w, &full[s], a_dst + BM * BK * 2, kb * BK, p.n_up_off + j0, pol_w);
        } else {
          uint8_t* b_dst = sB + s * CF::B_BYTES;
          if constexpr (EPI == EPI_SWIGLU) {
            const int j0 = nb * (BN / 2);
            tma_load_2d(&map_w, &full[s], b_dst, kb * BK, j0);
            tma_load_2d(&map_w, &full[s], b_dst + (BN / 2) * BK * 2, kb * BK, p.n_up_off + j0);
          } else {
            tma_load_2d(&map_w, &full[s], b_dst, kb * BK, nb * BN);
          }
        }
      };
      auto load_x = [&](int s, int kb, int mb) {
        if constexpr (SWAP)
          tma_load_2d(&map_x, &full[s], sB + s * CF::B_BYTES, kb * BK, mb * BN);
        else
          tma_load_2d(&map_x, &full[s], sA + s * CF::A_BYTES, kb * BK, mb * BM);
      };
      int pre = 0;
#ifndef DUET_NO_WPREFETCH
      if ((int)blockIdx.x < p.num_units) {  // fresh ring: the first S stages are free
        int t, kb0, kb1;
        unit_k(blockIdx.x, t, kb0, kb1);
        pre = kb1 - kb0 < S ? kb1 - kb0 : S;
        for (int it = pr; it < pre; it += CF::NPROD) {
          mbar_expect_tx(&full[it], CF::STAGE_BYTES);
          load_w(it, kb0 + it, t / p.num_m);
        }
      }
#endif
      pdl_wait();
      int it = 0;
      for (int u = blockIdx.x; u < p.num_units; u += gridDim.x) {
        int t, kb0, kb1;
        unit_k(u, t, kb0, kb1);
        const int mb = t % p.num_m, nb = t / p.num_m;
        for (int kb = kb0; kb < kb1; ++kb, ++it) {
          if (it % CF::NPROD != pr) continue;
          const int s = it % S;
          if (it < pre) {  // weights already requested before pdl_wait
            load_x(s, kb, mb);
            continue;
          }
          mbar_wait(&empty[s], ((it / S) & 1) ^ 1);
          mbar_expect_tx(&full[s], CF::STAGE_BYTES);
          load_w(s, kb, nb);
          load_x(s, kb, mb);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---------------- MMA issuer
      constexpr uint32_t idesc = idesc_bf16(BM, BN);
      int it = 0, i = 0;
      for (int u = blockIdx.x; u < p.num_units; u += gridDim.x, ++i) {
        int t, kb0, kb1;
        unit_k(u, t, kb0, kb1);
        const int acc = i & 1;
        const uint32_t aph = (i >> 1) & 1;
        mbar_wait(&tempty[acc], aph ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * CF::ACC_COLS;
        for (int kb = kb0; kb < kb1; ++kb, ++it) {
          const int s = it % S;
          mbar_wait(&full[s], (it / S) & 1);
          tc_fence_after();
          const uint32_t a0 = smem_u32(sA + s * CF::A_BYTES);
          const uint32_t b0 = smem_u32(sB + s * CF::B_BYTES);
#pragma unroll
          for (int k = 0; k < BK / 16; ++k) {
            umma_bf16(d_tmem, sw128_desc(a0 + k * 32), sw128_desc(b0 + k * 32), idesc, (kb > kb0 || k) != 0);
            if constexpr (SWAP && EPI == EPI_SWIGLU)
              umma_bf16(d_tmem + BN, sw128_desc(a0 + BM * BK * 2 + k * 32), sw128_desc(b0 + k * 32), idesc,
                        (kb > kb0 || k) != 0);
          }
          umma_commit(&empty[s]);
        }
        umma_commit(&tfull[acc]);
      }
    }
  } else {
    // ---------------- epilogue warps 2..5: TMEM lane quadrant = warp % 4
    const int quad = warp & 3;
    const int lane_row = quad * 32 + lane;
    int i = 0;
    for (int u = blockIdx.x; u < p.num_units; u += gridDim.x, ++i) {
      int t, kb0, kb1;
      unit_k(u, t, kb0, kb1);
      const int acc = i & 1;
      const uint32_t aph = (i >> 1) & 1;
      const int mb = t % p.num_m, nb = t / p.num_m;
      mbar_wait(&tfull[acc], aph);
      if (u + (int)gridDim.x >= p.num_units) pdl_trigger();  // last unit: only the epilogue is left
      tc_fence_after();
      const uint32_t tbase = tmem_base + ((uint32_t)(quad * 32) << 16) + acc * CF::ACC_COLS;
      if constexpr (!SWAP) {
        // lane = token row, columns = output features
        const int row = mb * BM + lane_row;
        constexpr int OUT_COLS = EPI == EPI_SWIGLU ? BN / 2 : BN;
        const int n0 = nb * OUT_COLS;
#pragma unroll 1
        for (int c = 0; c < OUT_COLS; c += 32) {
          float v[32];
          tmem_ld32(tbase + c, v);
          if constexpr (EPI == EPI_SWIGLU) {
            float u[32];
            tmem_ld32(tbase + BN / 2 + c, u);
#pragma unroll
            for (int e = 0; e < 32; ++e) v[e] = silu_f(v[e]) * u[e];
          }
          if (row < p.M && n0 + c < p.N) {
            bf16* dst = p.C + (size_t)row * p.ldc + n0 + c;
            if (n0 + c + 32 <= p.N) {
              if constexpr (EPI == EPI_RESIDUAL) {
                const bf16* rsrc = p.R + (size_t)row * p.ldr + n0 + c;
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
                if constexpr (EPI == EPI_RESIDUAL) o += __bfloat162float(p.R[(size_t)row * p.ldr + n0 + c + e]);
                if constexpr (EPI == EPI_STORE)
                  if (p.bias) o += __bfloat162float(p.bias[n0 + c + e]);
                dst[e] = __float2bfloat16_rn(o);
              }
            }
          }
        }
      } else if (p.ksplit == 1) {
        // lane = output feature n, columns = tokens m
        const int n = nb * BM + lane_row;
        const bool n_ok = n < p.N;
#pragma unroll 1
        for (int c = 0; c < BN; c += 32) {
          const int m0 = mb * BN + c;
          if (m0 >= p.M) break;  // warp-uniform
          float v[32];
          tmem_ld32(tbase + c, v);
          if constexpr (EPI == EPI_SWIGLU) {
            float u[32];
            tmem_ld32(tbase + BN + c, u);
#pragma unroll
            for (int e = 0; e < 32; ++e) v[e] = silu_f(v[e]) * u[e];
          }
          if (n_ok) swap_store<EPI>(p, v, m0, n);
        }
      } else {
        // split-K: this chunk's fp32 partial, column-major [ACC_COLS][128 rows] so both this store
        // and the reduction kernel's loads are coalesced across the 128 weight rows
        const int ch = u / p.num_tiles;
        float* part = p.ws + ((size_t)t * p.ksplit + ch) * CF::ACC_COLS * BM + lane_row;
#pragma unroll 1
        for (int c = 0; c < CF::ACC_COLS; c += 32) {
          float v[32];
          tmem_ld32(tbase + c, v);
#pragma unroll
          for (int e = 0; e < 32; ++e) __stcg(part + (size_t)(c + e) * BM, v[e]);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base), "n"(CF::TMEM_COLS));
  }
}

// Split-K reduction + epilogue: one CTA (256 threads) per tile.  Thread t owns 4 consecutive weight
// rows n = 4 (t % 32) .. +3 and the token columns m = t / 32, t / 32 + 8, ...; for two columns at a
// time it issues all ksplit float4 loads before summing them in chunk order 0..ksplit-1 (a fixed
// order, independent of the grid and of which CTA computed which chunk), so ~16 loads per thread are
// in flight; then applies the fused epilogue and stores 4 bf16 (8 B) per thread per column.
template <int EPI>
__global__ void __launch_bounds__(256) splitk_reduce_kernel(Params p, int bn, int acc_cols) {
  pdl_wait();
  const int t = blockIdx.x;
  const int mb = t % p.num_m, nb = t / p.num_m;
  const int rq = threadIdx.x & 31, cg = threadIdx.x >> 5;
  const int n = nb * BM + 4 * rq;
  if (n >= p.N) return;
  const size_t chunk = (size_t)acc_cols * BM;
  const float* base = p.ws + (size_t)t * p.ksplit * chunk + 4 * rq;
  float bias4[4] = {0.f, 0.f, 0.f, 0.f};
  if constexpr (EPI == EPI_STORE)
    if (p.bias)
#pragma unroll
      for (int e = 0; e < 4; ++e) bias4[e] = n + e < p.N ? __bfloat162float(p.bias[n + e]) : 0.f;
  auto sum_col = [&](int col, float (&out)[4]) {
    float4 f[SPLITK_MAX];
#pragma unroll
    for (int k = 0; k < SPLITK_MAX; ++k)
      if (k < p.ksplit) f[k] = __ldcg(reinterpret_cast<const float4*>(base + k * chunk + (size_t)col * BM));
    float4 a = f[0];
#pragma unroll
    for (int k = 1; k < SPLITK_MAX; ++k)
      if (k < p.ksplit) {
        a.x += f[k].x;
        a.y += f[k].y;
        a.z += f[k].z;
        a.w += f[k].w;
      }
    out[0] = a.x;
    out[1] = a.y;
    out[2] = a.z;
    out[3] = a.w;
  };
#pragma unroll 2
  for (int ml = cg; ml < bn; ml += 8) {
    const int m = mb * bn + ml;
    if (m >= p.M) break;
    float v[4];
    sum_col(ml, v);
    if constexpr (EPI == EPI_SWIGLU) {
      float g[4];
      sum_col(bn + ml, g);
#pragma unroll
      for (int e = 0; e < 4; ++e) v[e] = silu_f(v[e]) * g[e];
    }
    bf16* dst = p.C + (size_t)m * p.ldc + n;
    if (n + 4 <= p.N) {
      if constexpr (EPI == EPI_RESIDUAL) {
        const __nv_bfloat162* r2 = reinterpret_cast<const __nv_bfloat162*>(p.R + (size_t)m * p.ldr + n);
        const float2 r0 = __bfloat1622float2(r2[0]), r1 = __bfloat1622float2(r2[1]);
        v[0] += r0.x;
        v[1] += r0.y;
        v[2] += r1.x;
        v[3] += r1.y;
      }
      if constexpr (EPI == EPI_STORE)
#pragma unroll
        for (int e = 0; e < 4; ++e) v[e] += bias4[e];
      __nv_bfloat162 o0 = __floats2bfloat162_rn(v[0], v[1]), o1 = __floats2bfloat162_rn(v[2], v[3]);
      uint2 pk;
      pk.x = *reinterpret_cast<uint32_t*>(&o0);
      pk.y = *reinterpret_cast<uint32_t*>(&o1);
      *reinterpret_cast<uint2*>(dst) = pk;
    } else {
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        if (n + e >= p.N) continue;
        float o = v[e];
        if constexpr (EPI == EPI_RESIDUAL) o += __bfloat162float(p.R[(size_t)m * p.ldr + n + e]);
        if constexpr (EPI == EPI_STORE) o += bias4[e];
        dst[e] = __float2bfloat16_rn(o);
      }
    }
  }
}

// ------------------------------------------------------------------------- host side

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

// 2-D bf16 map over a row-major [rows][cols] matrix with row pitch ld (elements); box = 64 x box_rows.
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

// K chunking of a split-K launch: a function of the shape only (see SPLITK_TARGET_UNITS)
static void splitk_plan(int num_tiles, int num_k, int* ks_out, int* kb_out) {
  int ks = num_tiles > SPLITK_MAX_TILES ? 1 : (SPLITK_TARGET_UNITS + num_tiles - 1) / num_tiles;
  ks = std::min(std::min(ks, SPLITK_MAX), num_k / SPLITK_MIN_KB);
  if (ks < 1) ks = 1;
  const int kb = (num_k + ks - 1) / ks;
  *ks_out = (num_k + kb - 1) / kb;
  *kb_out = kb;
}

template <int BN, int EPI, bool SWAP>
static int launch(const GemmArgs& a, int num_sms, cudaStream_t st) {
  using CF = Cfg<BN, EPI, SWAP>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(gemm_tc_kernel<BN, EPI, SWAP>, cudaFuncAttributeMaxDynamicSharedMemorySize, CF::SMEM);
    attr_set = true;
  }
  CUtensorMap mx, mw;
  const int w_rows = EPI == EPI_SWIGLU ? 2 * a.N : a.N;
  Params p{};
  p.M = a.M;
  p.N = a.N;
  p.K = a.K;
  if constexpr (!SWAP) {
    if (!make_map(&mx, a.A, a.M, a.K, a.lda, BM)) return -1;
    if (!make_map(&mw, a.B, w_rows, a.K, a.ldb, EPI == EPI_SWIGLU ? BN / 2 : BN)) return -1;
    const int out_cols = EPI == EPI_SWIGLU ? BN / 2 : BN;
    p.num_m = (a.M + BM - 1) / BM;
    p.num_n = (a.N + out_cols - 1) / out_cols;
  } else {
    if (!make_map(&mx, a.A, a.M, a.K, a.lda, BN)) return -1;
    if (!make_map(&mw, a.B, w_rows, a.K, a.ldb, BM)) return -1;
    p.num_m = (a.M + BN - 1) / BN;
    p.num_n = (a.N + BM - 1) / BM;
  }
  p.num_tiles = p.num_m * p.num_n;
  p.ksplit = 1;
  p.kb_per = a.K / BK;
  if constexpr (SWAP) {
    int ks, kb;
    splitk_plan(p.num_tiles, a.K / BK, &ks, &kb);
    const size_t need = (size_t)p.num_tiles * ks * BM * CF::ACC_COLS;
    static const bool splitk_on = !getenv("DUET_SPLITK") || atoi(getenv("DUET_SPLITK")) != 0;  // A/B switch
    if (splitk_on && ks > 1 && a.ws && need <= a.ws_floats) {
      p.ksplit = ks;
      p.kb_per = kb;
      p.ws = a.ws;
    }
  }
  p.num_units = p.num_tiles * p.ksplit;

  p.C = (bf16*)a.C;
  p.R = (const bf16*)a.R;
  p.bias = (const bf16*)a.bias;
  p.ldc = a.ldc;
  p.ldr = a.ldr;
  p.n_up_off = a.N;
  const int grid = p.num_units < CF::CTAS * num_sms ? p.num_units : CF::CTAS * num_sms;
  launch_pdl(gemm_tc_kernel<BN, EPI, SWAP>, grid, CF::THREADS, CF::SMEM, st, mx, mw, p);
  if (p.ksplit > 1) {
    launch_pdl(splitk_reduce_kernel<EPI>, p.num_tiles, 256, 0, st, p, BN, (int)CF::ACC_COLS);
    return 2;
  }
  return 1;
}

template <int EPI>
static int launch_epi(const GemmArgs& a, int num_sms, cudaStream_t st) {
  if (a.M <= 64) return launch<64, EPI, true>(a, num_sms, st);
  if (a.M <= 128) return launch<128, EPI, true>(a, num_sms, st);
  return launch<256, EPI, false>(a, num_sms, st);
}

}  // namespace tc

bool gemm_tc_supported(const GemmArgs& a) {
  // K in whole 64-element blocks; 16-byte aligned rows for TMA and vector epilogue loads
  if (a.K % tc::BK || a.M <= 0) return false;
  if (a.lda % 8 || a.ldb % 8 || a.ldc % 8 || (a.R && a.ldr % 8)) return false;
  // TMA maps and the 16-B vector epilogue need 16-byte aligned base pointers
  auto mis = [](const void* p) { return ((uintptr_t)p & 15) != 0; };
  if (mis(a.A) || mis(a.B) || mis(a.C) || mis(a.R) || mis(a.R2) || mis(a.C2)) return false;
  if (a.epi == EPI_SWIGLU && a.N % 128) return false;
  if (!tc::encode_fn()) return false;
  return true;
}

size_t gemm_tc_splitk_need(int M, int N, int K, int epi) {
  if (M <= 0 || M > 128 || K % tc::BK) return 0;
  const int bn = M <= 64 ? 64 : 128;
  const int num_tiles = ((M + bn - 1) / bn) * ((N + tc::BM - 1) / tc::BM);
  int ks, kb;
  tc::splitk_plan(num_tiles, K / tc::BK, &ks, &kb);
  if (ks <= 1) return 0;
  return (size_t)num_tiles * ks * tc::BM * (epi == EPI_SWIGLU ? 2 * bn : bn);
}

int launch_gemm_tc(const GemmArgs& a, int num_sms, cudaStream_t st) {
  if (a.epi == EPI_SWIGLU) return tc::launch_epi<EPI_SWIGLU>(a, num_sms, st);
  if (a.epi == EPI_RESIDUAL) return tc::launch_epi<EPI_RESIDUAL>(a, num_sms, st);
  return tc::launch_epi<EPI_STORE>(a, num_sms, st);
}

}  // namespace duet

// Causal prefill attention over the paged KV cache on 5th-generation tensor cores (tcgen05 / TMEM).
//
// Chunked prefill (§4.1; readings #2, #6, #7): a chunk of q tokens at positions
// c..c+q-1 attends to its c-token prefix and to itself causally.  One CTA = 128 query rows of one
// query head; the keys stream in 64-key tiles (4 pages of 16 tokens).
//   warp 0      Q tile by TMA (two 64-column SWIZZLE_128B boxes)
//   warp 1      TMEM allocator + tcgen05.mma issuer: S_j = Q K_j^T (UMMA 128x64x16, both operands
//               K-major) into one of two TMEM S buffers, then O += P_{j-1} V_{j-1} (A = P from smem,
//               B = V MN-major) — the MMAs of S_{j+1} overlap the softmax of tile j
//   warps 2..5  softmax, one thread per query row (= TMEM lane): max / exp2 / sum in registers, P
//               written to one of two smem buffers in the UMMA SW128 layout; the running max is re-based
//               (O rescaled in TMEM) only when it grows by more than 2^8, so P <= 256
//   warps 6..9  K/V loaders: cp.async gathers of the scattered 4 KiB page blocks into a 4-stage ring
//               (a TMA box costs its issuing thread ~0.25 us on B200 — profiles/r01_probe_tma_bw.txt —
//               and a page needs four), published LAG = 2 tiles behind the issue front
// Keys past the causal end of the tile are zero-filled (cp.async src-size 0) and masked.
#include <cuda.h>

#include "dev_common.cuh"
#include "kernels.h"

namespace duet {
namespace fatc {

constexpr int BQ = 128, BKV = 64, DH = 128, PAGE = 16, KV_STAGES = 4, LAG = 2;
constexpr int Q_SUB = BQ * 128;            // [128 rows][64 cols] SW128 sub-tile = 16 KiB
constexpr int KV_SUB = BKV * 128;          // [64 rows][64 cols] = 8 KiB
constexpr int Q_BYTES = 2 * Q_SUB;         // 32 KiB
constexpr int KV_BYTES = 2 * KV_SUB;       // 16 KiB per tensor per stage
constexpr int P_BYTES = BQ * BKV * 2;      // [128 rows][64 keys] = one SW128 sub-tile, 16 KiB
constexpr int OFF_Q = 0;
constexpr int OFF_K = OFF_Q + Q_BYTES;
constexpr int OFF_V = OFF_K + KV_STAGES * KV_BYTES;
constexpr int OFF_P = OFF_V + KV_STAGES * KV_BYTES;
constexpr int OFF_BAR = OFF_P + 2 * P_BYTES;
constexpr int SMEM = OFF_BAR + 256 + 1024;
constexpr int TMEM_COLS = 256;             // S0 (64) | S1 (64) | O (128)
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
  int max_pages, hq, hkv, n_qtiles;
  bf16* o;
  const bf16* k_pool;
  const bf16* v_pool;
};

__global__ void __launch_bounds__(320, 1) fa_tc_kernel(const __grid_constant__ CUtensorMap map_q, Params p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  uint64_t* bar = (uint64_t*)(smem + OFF_BAR);
  uint64_t* q_full = bar;                   // 1
  uint64_t* kv_full = bar + 1;              // [KV_STAGES]
  uint64_t* kv_empty = kv_full + KV_STAGES; // [KV_STAGES]
  uint64_t* s_full = kv_empty + KV_STAGES;  // [2]
  uint64_t* s_free = s_full + 2;            // [2]
  uint64_t* p_full = s_free + 2;            // [2]
  uint64_t* pv_done = p_full + 2;           // [2]  PV of the tile that used P buffer b
  uint32_t* tmem_slot = (uint32_t*)(pv_done + 2);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int qt = p.n_qtiles - 1 - blockIdx.x;  // heavy (late) tiles first
  const int head = blockIdx.y, s_id = blockIdx.z;
  const int qlen = p.qlen[s_id];
  if (qt * BQ >= qlen) return;
  const int G = p.hq / p.hkv, kvh = head / G;
  const int row0 = p.row0[s_id], cpre = p.cpre[s_id];
  const int* tab = p.table + (size_t)p.seq_row[s_id] * p.max_pages;
  const int q0 = qt * BQ;
  const int q_last = min(q0 + BQ, qlen) - 1;
  const int kv_end = cpre + q_last + 1;
  const int n_kt = (kv_end + BKV - 1) / BKV;

  if (warp == 0 && lane == 0) {
    mbar_init(q_full, 1);
    for (int i = 0; i < KV_STAGES; ++i) {
      mbar_init(&kv_full[i], 4);  // one arrive per loader warp
      mbar_init(&kv_empty[i], 1);
    }
    for (int i = 0; i < 2; ++i) {
      mbar_init(&s_full[i], 1);
      mbar_init(&s_free[i], 4);
      mbar_init(&p_full[i], 4);
      mbar_init(&pv_done[i], 1);
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
  const uint32_t T_S0 = tmem, T_S1 = tmem + BKV, T_O = tmem + 2 * BKV;

  if (warp == 0) {
    if (lane == 0) {
      // ------------------------------------------------ Q tile (TMA, two 64-column boxes)
      mbar_expect_tx(q_full, Q_BYTES);
      tma_load_2d(&map_q, q_full, smem + OFF_Q, head * DH, row0 + q0);
      tma_load_2d(&map_q, q_full, smem + OFF_Q + Q_SUB, head * DH + 64, row0 + q0);
    }
  } else if (warp >= 6) {
    // ------------------------------------------------ K/V loaders (4 warps, cp.async, 4-stage ring)
    const int lt = threadIdx.x - 6 * 32;  // 0..127
    const size_t page_stride = (size_t)p.hkv * PAGE * DH;
    // chunk c = lt + 128 i (i < 8) of a [64 keys][16 chunks] tile: key = c / 16, 16-B column = c % 16
    auto issue = [&](int j) {
      const int st = j % KV_STAGES;
      const uint32_t kd = smem_u32(smem + OFF_K + st * KV_BYTES), vd = smem_u32(smem + OFF_V + st * KV_BYTES);
#pragma unroll
      for (int i = 0; i < (BKV * 16) / 128; ++i) {
        const int c = lt + i * 128;
        const int rr = c >> 4, ch = c & 15;
        const int key = j * BKV + rr;
        const bool v = key < kv_end;
        const size_t off =
            v ? (size_t)tab[key / PAGE] * page_stride + ((size_t)kvh * PAGE + (key % PAGE)) * DH + ch * 8 : 0;
        const uint32_t so = (uint32_t)((ch >> 3) * KV_SUB + rr * 128 + (((ch & 7) ^ (rr & 7)) << 4));
        const int sz = v ? 16 : 0;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(kd + so), "l"(p.k_pool + off), "r"(sz)
                     : "memory");
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(vd + so), "l"(p.v_pool + off), "r"(sz)
                     : "memory");
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
    };
    int pub = 0;
    auto publish = [&]() {  // the oldest unpublished tile has landed -> visible to the async proxy
      fence_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(&kv_full[pub % KV_STAGES]);
      ++pub;
    };
    // LAG <= KV_STAGES - 2: tile j - KV_STAGES (whose consumption frees slot j) is always published first
    for (int j = 0; j < n_kt; ++j) {
      mbar_wait(&kv_empty[j % KV_STAGES], ((j / KV_STAGES) & 1) ^ 1);
      issue(j);
      if (j >= LAG) {
        asm volatile("cp.async.wait_group %0;" ::"n"(LAG) : "memory");
        publish();
      }
    }
    asm volatile("cp.async.wait_group 0;" ::: "memory");
    while (pub < n_kt) publish();
  } else if (warp == 1) {
    // ------------------------------------------------ MMA issuer
    constexpr uint32_t ID_S = idesc(BKV, false), ID_PV = idesc(DH, true);
    const uint32_t sq = smem_u32(smem + OFF_Q);
    mbar_wait(q_full, 0);
    for (int j = 0; j <= n_kt; ++j) {
      if (j < n_kt) {
        const int b = j & 1, st = j % KV_STAGES;
        if (j >= 2) mbar_wait(&s_free[b], ((j - 2) >> 1) & 1);
        mbar_wait(&kv_full[st], (j / KV_STAGES) & 1);
        tc_after();
        if (lane == 0) {
          const uint32_t sk = smem_u32(smem + OFF_K + st * KV_BYTES);
#pragma unroll
          for (int kk = 0; kk < DH / 16; ++kk) {
            umma(b ? T_S1 : T_S0, desc_k(sq + (kk >> 2) * Q_SUB + (kk & 3) * 32),
                 desc_k(sk + (kk >> 2) * KV_SUB + (kk & 3) * 32), ID_S, kk > 0);
          }
          umma_commit(&s_full[b]);
        }
        __syncwarp();
      }
      if (j >= 1) {
        const int jp = j - 1, b = jp & 1, st = jp % KV_STAGES;
        mbar_wait(&p_full[b], (jp >> 1) & 1);
        tc_after();
        if (lane == 0) {
          const uint32_t spp = smem_u32(smem + OFF_P + b * P_BYTES);
          const uint32_t sv = smem_u32(smem + OFF_V + st * KV_BYTES);
#pragma unroll
          for (int kk = 0; kk < BKV / 16; ++kk)  // 16 keys per UMMA k-step
            umma(T_O, desc_k(spp + kk * 32), desc_mn(sv + kk * 16 * 128), ID_PV, (jp > 0 || kk > 0));
          umma_commit(&kv_empty[st]);
          umma_commit(&pv_done[b]);
        }
        __syncwarp();
      }
    }
  } else {
    // ------------------------------------------------ softmax warps: one thread per query row
    const int quad = warp & 3;
    const int r = quad * 32 + lane;                          // row in tile = TMEM lane
    const int pos = min(cpre + q0 + r, kv_end - 1);          // clamp rows past the chunk
    const float sc = rsqrtf((float)DH) * 1.4426950408889634f;
    const uint32_t lane_base = (uint32_t)(quad * 32) << 16;
    const uint32_t sw = (uint32_t)(r & 7);
    float m_used = -INFINITY, l = 0.f;
    for (int j = 0; j < n_kt; ++j) {
      const int b = j & 1;
      const uint32_t T_S = b ? T_S1 : T_S0;
      mbar_wait(&s_full[b], (j >> 1) & 1);
      tc_after();
      const int kbase = j * BKV;
      uint32_t v0[32], v1[32];
      tmem_ld32(T_S + lane_base, v0);
      tmem_ld32(T_S + lane_base + 32, v1);
      tc_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&s_free[b]);  // S buffer b may be overwritten by S_{j+2}
      const int lim = pos - kbase;  // keys 0..lim of this tile are visible to this row
      float mx = -INFINITY;
      if (lim >= BKV - 1) {
#pragma unroll
        for (int e = 0; e < 32; ++e) mx = fmaxf(mx, fmaxf(__uint_as_float(v0[e]), __uint_as_float(v1[e])));
      } else {
#pragma unroll
        for (int e = 0; e < 32; ++e) {
          if (e <= lim) mx = fmaxf(mx, __uint_as_float(v0[e]));
          if (32 + e <= lim) mx = fmaxf(mx, __uint_as_float(v1[e]));
        }
      }
      const float m_new = fmaxf(m_used, mx * sc);  // sc > 0: the max commutes with the scaling
      // Re-base the rows whose max grew by more than 2^8.  tcgen05.ld/st are warp-collective
      // (.sync.aligned), so the decision is made per warp and rows that keep their max scale by 1.
      const bool mine = m_new > m_used + RESCALE_THRESHOLD;
      if (__any_sync(0xffffffffu, mine)) {
        if (j >= 1) {
          // O must be quiescent: wait for PV_{j-1} (all earlier ones completed before it)
          mbar_wait(&pv_done[(j - 1) & 1], ((j - 1) >> 1) & 1);
          tc_after();
          const float f = mine ? exp2f(m_used - m_new) : 1.f;
          l *= f;
#pragma unroll 1
          for (int c = 0; c < DH; c += 32) {
            uint32_t v[32];
            tmem_ld32(T_O + lane_base + c, v);
#pragma unroll
            for (int e = 0; e < 32; ++e) v[e] = __float_as_uint(__uint_as_float(v[e]) * f);
            tmem_st32(T_O + lane_base + c, v);
          }
        }
        if (mine) m_used = m_new;
      }
      // P buffer b is free once PV_{j-2} has completed
      if (j >= 2) {
        mbar_wait(&pv_done[b], ((j - 2) >> 1) & 1);
        tc_after();
      }
      uint8_t* prow = smem + OFF_P + b * P_BYTES + r * 128;
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        uint32_t pk[16];
#pragma unroll
        for (int e = 0; e < 32; e += 2) {
          const float s0 = __uint_as_float(h ? v1[e] : v0[e]), s1 = __uint_as_float(h ? v1[e + 1] : v0[e + 1]);
          const int k0 = h * 32 + e;
          const float p0 = (k0 <= lim) ? fast_exp2(fmaf(s0, sc, -m_used)) : 0.f;
          const float p1 = (k0 + 1 <= lim) ? fast_exp2(fmaf(s1, sc, -m_used)) : 0.f;
          l += p0 + p1;
          __nv_bfloat162 hh = __floats2bfloat162_rn(p0, p1);
          pk[e / 2] = *reinterpret_cast<uint32_t*>(&hh);
        }
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4) {
          const uint32_t chunk = (uint32_t)(h * 4 + q4);
          *reinterpret_cast<uint4*>(prow + ((chunk ^ sw) << 4)) =
              make_uint4(pk[q4 * 4], pk[q4 * 4 + 1], pk[q4 * 4 + 2], pk[q4 * 4 + 3]);
        }
      }
      fence_async_smem();
      tc_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&p_full[b]);
    }
    // epilogue: O / l -> bf16 -> global
    mbar_wait(&pv_done[(n_kt - 1) & 1], ((n_kt - 1) >> 1) & 1);
    tc_after();
    const bool row_ok = q0 + r < qlen;
    const float inv = l > 0.f ? 1.f / l : 0.f;
    bf16* dst = p.o + (size_t)(row0 + q0 + r) * p.hq * DH + (size_t)head * DH;
#pragma unroll 1
    for (int c = 0; c < DH; c += 32) {
      uint32_t v[32];
      tmem_ld32(T_O + lane_base + c, v);
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
  tc_before();
  __syncthreads();
  if (warp == 1) {
    tc_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "n"(TMEM_COLS));
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

}  // namespace fatc

bool fa_tc_supported(const PrefillAttnArgs& a) {
  return a.dh == fatc::DH && a.page_size == fatc::PAGE && a.q_stride % 8 == 0 && fatc::encode_fn() != nullptr &&
         a.total_rows > 0;
}

int launch_fa_tc(const PrefillAttnArgs& a, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(fatc::fa_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, fatc::SMEM);
    attr = true;
  }
  CUtensorMap mq;
  if (!fatc::make_map(&mq, a.q, (uint64_t)a.total_rows, (uint64_t)a.q_stride, (uint64_t)a.q_stride, 128)) return -1;
  fatc::Params p{a.row0,  a.qlen, a.cpre,       a.seq_row,           a.table, a.max_pages,
                 a.hq,    a.hkv,  0,            (bf16*)a.o,          (const bf16*)a.k_pool,
                 (const bf16*)a.v_pool};
  p.n_qtiles = (a.max_q + fatc::BQ - 1) / fatc::BQ;
  dim3 grid(p.n_qtiles, a.hq, a.n_seqs);
  fatc::fa_tc_kernel<<<grid, 320, fatc::SMEM, st>>>(mq, p);
  return 1;
}

}  // namespace duet

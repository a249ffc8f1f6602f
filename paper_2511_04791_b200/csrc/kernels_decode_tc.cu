// Paged decode attention on tensor cores (bf16, d_h = 128, GQA group G <= 8).
//
// Computed transposed, so that the 16 tokens of a page fill the MMA M dimension and the G query
// heads sharing a kv head (reading #6) fill N = 8:
//   S^T (16 keys x 8 heads)  = K_page (16 x 128) . Q^T (128 x 8)          8 x mma.m16n8k16
//   O^T (128 dims x 8 heads) += V_page^T (128 x 16) . P^T (16 x 8)        8 x mma.m16n8k16
// P^T goes from the S^T accumulator layout to the B-operand layout with two movmatrix.trans.
// Each 16-token page of K and V is read from HBM exactly once per request (P:213 counts
// 2 h_kv (q+c) d_h s bytes).  Pages are fetched with TMA (2-D tensor maps over the pools, one
// 16-row x 64-column SWIZZLE_128B box per half page) into a private NST-stage ring per warp, so a
// page costs one elected thread four TMA instructions and an mbarrier; 8 warps per CTA stream
// pages w, w+8, ...  Slots past the sequence end are masked out of S and zeroed in V.  Online
// softmax per head (exp2 domain); warps and splits are merged with the log-sum-exp rule.
// One CTA per (split, kv head, request).
#include <cuda.h>

#include <cstdlib>
#include <cstring>

#include "dev_common.cuh"
#include "kernels.h"

namespace duet {
namespace dtc {

constexpr int DH = 128, PAGE = 16;
constexpr int HALF = PAGE * 128;              // one 16-row x 64-col SW128 box = 2 KiB
constexpr int PAGE_BYTES = 2 * HALF;          // 4 KiB: one kv head of one page
constexpr int STAGE_BYTES = 2 * PAGE_BYTES;   // K + V
__host__ __device__ constexpr int smem_bytes(int warps, int nst) { return warps * nst * STAGE_BYTES + 1024 + 512; }

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
// byte offset of 16-B chunk ch (0..15) of row r in a page stored as two SW128 [16][64] halves
__device__ __forceinline__ uint32_t swz(int r, int ch) {
  return (uint32_t)((ch >> 3) * HALF + r * 128 + (((ch & 7) ^ (r & 7)) << 4));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
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
__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t& r0, uint32_t& r1, uint32_t& r2, uint32_t& r3) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r0), "=r"(r1), "=r"(r2), "=r"(r3)
               : "r"(addr));
}
__device__ __forceinline__ void mma16816(float (&d)[4], uint32_t a0, uint32_t a1, uint32_t a2, uint32_t a3,
                                         uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t movtrans(uint32_t a) {
  uint32_t d;
  asm volatile("movmatrix.sync.aligned.m8n8.trans.b16 %0, %1;" : "=r"(d) : "r"(a));
  return d;
}
// 2^x on the SFU without exp2f's denormal fix-up (arguments <= 0 here; -inf -> +0)
__device__ __forceinline__ float fast_exp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
// device-side launch timing (DecodeAttnArgs::dev_timer): called by thread 0 of every CTA
__device__ __forceinline__ void dev_timer_start(unsigned long long* t) { atomicMin(&t[0], gtimer()); }
__device__ __forceinline__ void dev_timer_end(unsigned long long* t) {
  atomicMax(&t[1], gtimer());
  __threadfence();
  const unsigned long long total = (unsigned long long)gridDim.x * gridDim.y * gridDim.z;
  if (atomicAdd(&t[2], 1ull) == total - 1) {  // the launch's last CTA
    __threadfence();
    const unsigned long long t0 = atomicAdd(&t[0], 0ull), t1 = atomicAdd(&t[1], 0ull);
    atomicAdd(&t[3], t1 > t0 ? t1 - t0 : 0ull);
    atomicAdd(&t[4], 1ull);
    atomicExch(&t[0], ~0ull);
    atomicExch(&t[1], 0ull);
    atomicExch(&t[2], 0ull);
  }
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&h);
}

// WARPS consumer warps per CTA, NST-stage ring per warp; TMA = pages fetched by TMA boxes (lane 0),
// else by cp.async from all 32 lanes (cheaper to issue on small SM partitions).
// One work item (split of the pages, kv head, request column z) by a group of WARPS warps — the body of
// decode_tc_kernel (the CTA is one group, one item per CTA) and of the decode part of the fused POD launch
// (kernels_pod.cu: three 4-warp groups per CTA, each the standalone kernel's CTA, items strided over the
// groups — so the results are bitwise those of the standalone launch).  smem: the group's rings (1 KiB
// aligned), tid: thread index in the group, bar: 0 = the whole CTA is the group (__syncthreads), else the
// named barrier the group's WARPS * 32 threads use.  Ends with a barrier-separated merge through the rings.
template <int WARPS, int NST, bool TMA>
__device__ __forceinline__ void decode_tc_item(const CUtensorMap* mk_, const CUtensorMap* mv_, const DecodeAttnArgs& a,
                                               int pps, int n_splits, const int split, const int kvh, const int zc,
                                               uint8_t* smem, const int tid, const int bar) {
  const CUtensorMap& map_k = *mk_;
  const CUtensorMap& map_v = *mv_;
  constexpr int WARP_BYTES = NST * STAGE_BYTES;
  auto group_sync = [&]() {
    if (bar == 0) __syncthreads();
    else asm volatile("bar.sync %0, %1;" ::"r"(bar), "n"(WARPS * 32) : "memory");
  };
  const int r = a.order ? a.order[zc] : zc;
  const int warp = tid >> 5, lane = tid & 31;
  const int G = a.hq / a.hkv;
  const int len = a.pos[r] + 1;
  const int n_pages = (len + PAGE - 1) / PAGE;
  const int pg0 = split * pps;
  const int pg1 = min(n_pages, pg0 + pps);
  const int* tab = a.table + (size_t)a.tok_row[r] * a.max_pages;
  uint8_t* wsm = smem + warp * WARP_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + WARPS * WARP_BYTES) + warp * NST;
  const int g = lane >> 2, t4 = lane & 3;
  if (TMA && lane == 0) {
    for (int i = 0; i < NST; ++i) mbar_init(&full[i], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();

  // Q^T as the B operand: b0 = Q[head g][kk*16 + 2t, +1], b1 = Q[g][kk*16 + 8 + 2t, +1]; zero for g >= G
  uint32_t qb[8][2];
  {
    const bf16* qr = reinterpret_cast<const bf16*>(a.q) + (size_t)r * a.q_stride + (size_t)kvh * G * DH;
    const bool v = g < G;
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
      qb[kk][0] = v ? *reinterpret_cast<const uint32_t*>(qr + g * DH + kk * 16 + 2 * t4) : 0u;
      qb[kk][1] = v ? *reinterpret_cast<const uint32_t*>(qr + g * DH + kk * 16 + 8 + 2 * t4) : 0u;
    }
  }
  const int first = pg0 + warp;
  const int n_mine = first < pg1 ? (pg1 - first + WARPS - 1) / WARPS : 0;
  uint32_t soff[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) soff[k] = swz(2 * k + (lane >> 4), lane & 15);
  uint64_t l2_first;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(l2_first));
  // Page-table entries of this warp's pages, 32 at a time: lane L holds the entry of page slot
  // i = 32 b + L (prefetched one batch ahead), read with a shuffle when page i is issued, so no
  // cp.async waits on a dependent global load.
  auto tab_batch = [&](int b) {
    const int i = b * 32 + lane;
    return i < n_mine ? __ldg(tab + first + i * WARPS) : 0;
  };
  int pt_cur = tab_batch(0), pt_next = tab_batch(1);
  auto page_of = [&](int i) {  // warp-uniform i, all lanes participate
    if ((i & 31) == 0 && i > 0) {
      pt_cur = pt_next;
      pt_next = tab_batch((i >> 5) + 1);
    }
    return __shfl_sync(0xffffffffu, pt_cur, i & 31);
  };
  auto issue = [&](int i, int pid) {  // page i of this warp (pool page pid) into stage i % NST
    const int st = i % NST;
    uint8_t* dk = wsm + st * STAGE_BYTES;
    uint8_t* dv = dk + PAGE_BYTES;
    if constexpr (TMA) {  // lane 0 only
      const int prow = (pid * a.hkv + kvh) * PAGE;
      mbar_expect_tx(&full[st], STAGE_BYTES);
      tma_load_2d(&map_k, &full[st], dk, 0, prow);
      tma_load_2d(&map_k, &full[st], dk + HALF, 64, prow);
      tma_load_2d(&map_v, &full[st], dv, 0, prow);
      tma_load_2d(&map_v, &full[st], dv + HALF, 64, prow);
    } else {  // all lanes: 256 x 16 B per tensor; slots past the end are zero-filled
      // chunk k*32 + lane of the 4 KiB page block is row 2k + lane/16, 16-B column lane%16: its global
      // offset is (k*32 + lane) * 8 elements and its swizzled smem offset soff[k] (precomputed)
      const int pg = first + i * WARPS;
      const size_t base = ((size_t)pid * a.hkv + kvh) * PAGE * DH + lane * 8;
      const bf16* ks = reinterpret_cast<const bf16*>(a.k_pool) + base;
      const bf16* vs = reinterpret_cast<const bf16*>(a.v_pool) + base;
      const uint32_t sk = smem_u32(dk), sv = smem_u32(dv);
      const int rows_valid = len - pg * PAGE;  // >= 16 except on the last page
      // KV is read once per step: evict-first in L2, so the stream does not push out the working set
      // of a concurrently running prefill partition (GEMM operands, the chunk's own K/V)
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        const int sz = (2 * k + (lane >> 4)) < rows_valid ? 16 : 0;
        asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2, %3;" ::"r"(sk + soff[k]),
                     "l"(ks + k * 256), "r"(sz), "l"(l2_first) : "memory");
        asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2, %3;" ::"r"(sv + soff[k]),
                     "l"(vs + k * 256), "r"(sz), "l"(l2_first) : "memory");
      }
    }
  };
  if constexpr (TMA) {
    for (int i = 0; i < NST - 1 && i < n_mine; ++i) {
      const int pid = page_of(i);
      if (lane == 0) issue(i, pid);
    }
  } else {
#pragma unroll
    for (int i = 0; i < NST - 1; ++i) {
      if (i < n_mine) issue(i, page_of(i));
      asm volatile("cp.async.commit_group;" ::: "memory");
    }
  }

  const float scale = rsqrtf((float)DH) * 1.4426950408889634f;
  float o[8][4];  // O^T: m-tile mt -> dims mt*16 + {g, g+8}, heads {2t, 2t+1}
#pragma unroll
  for (int j = 0; j < 8; ++j) o[j][0] = o[j][1] = o[j][2] = o[j][3] = 0.f;
  float m[2] = {-INFINITY, -INFINITY}, l[2] = {0.f, 0.f};  // heads 2t, 2t+1

  for (int i = 0; i < n_mine; ++i) {
    // refill the stage consumed in the previous iteration (all lanes are past it: __syncwarp below)
    const int st = i % NST;
    if constexpr (TMA) {
      if (i + NST - 1 < n_mine) {
        const int pid = page_of(i + NST - 1);
        if (lane == 0) issue(i + NST - 1, pid);
      }
      mbar_wait(&full[st], (i / NST) & 1);
    } else {
      if (i + NST - 1 < n_mine) issue(i + NST - 1, page_of(i + NST - 1));
      asm volatile("cp.async.commit_group;" ::: "memory");
      asm volatile("cp.async.wait_group %0;" ::"n"(NST - 1) : "memory");
      __syncwarp();
    }
    const uint32_t sk = smem_u32(wsm + st * STAGE_BYTES), sv = sk + PAGE_BYTES;
    const int key0 = (first + i * WARPS) * PAGE;
    const bool partial = TMA && key0 + PAGE > len;
    if (partial) {  // zero V rows past the sequence end (unwritten slots may hold anything)
      for (int k = lane; k < PAGE * 16; k += 32) {
        const int rr = k >> 4, ch = k & 15;
        if (key0 + rr >= len)
          *reinterpret_cast<uint4*>(wsm + st * STAGE_BYTES + PAGE_BYTES + swz(rr, ch)) = make_uint4(0, 0, 0, 0);
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // before TMA re-fills this stage
      __syncwarp();
    }
    // S^T = K Q^T, two independent accumulation chains (even / odd k-steps)
    float s[4] = {0.f, 0.f, 0.f, 0.f}, s2[4] = {0.f, 0.f, 0.f, 0.f};
    const int key = (lane & 7) + (((lane >> 3) & 1) << 3);
#pragma unroll
    for (int kk = 0; kk < 8; kk += 2) {
      uint32_t a0, a1, a2, a3, c0, c1, c2, c3;
      ldsm_x4(sk + swz(key, kk * 2 + (lane >> 4)), a0, a1, a2, a3);
      ldsm_x4(sk + swz(key, kk * 2 + 2 + (lane >> 4)), c0, c1, c2, c3);
      mma16816(s, a0, a1, a2, a3, qb[kk][0], qb[kk][1]);
      mma16816(s2, c0, c1, c2, c3, qb[kk + 1][0], qb[kk + 1][1]);
    }
    // s[0], s[1]: key g, heads 2t, 2t+1 ; s[2], s[3]: key g+8
    const bool v0 = key0 + g < len, v1 = key0 + g + 8 < len;
    float x[4];
    x[0] = v0 ? (s[0] + s2[0]) * scale : -INFINITY;
    x[1] = v0 ? (s[1] + s2[1]) * scale : -INFINITY;
    x[2] = v1 ? (s[2] + s2[2]) * scale : -INFINITY;
    x[3] = v1 ? (s[3] + s2[3]) * scale : -INFINITY;
    float mx[2] = {fmaxf(x[0], x[2]), fmaxf(x[1], x[3])};
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      mx[h] = fmaxf(mx[h], __shfl_xor_sync(0xffffffffu, mx[h], 4));
      mx[h] = fmaxf(mx[h], __shfl_xor_sync(0xffffffffu, mx[h], 8));
      mx[h] = fmaxf(mx[h], __shfl_xor_sync(0xffffffffu, mx[h], 16));
    }
    // key 0 of a page is always valid, so the new maxima are finite.  l is kept per lane (its 8
    // g-lanes are summed once at the end); O is rescaled only when some head's max moved.
    const float mn0 = fmaxf(m[0], mx[0]), mn1 = fmaxf(m[1], mx[1]);
    const bool moved = mn0 != m[0] || mn1 != m[1];
    const float p0 = fast_exp2(x[0] - mn0), p1 = fast_exp2(x[1] - mn1), p2 = fast_exp2(x[2] - mn0),
                p3 = fast_exp2(x[3] - mn1);
    if (__any_sync(0xffffffffu, moved)) {
      const float c0 = fast_exp2(m[0] - mn0), c1 = fast_exp2(m[1] - mn1);
      l[0] *= c0;
      l[1] *= c1;
#pragma unroll
      for (int mt = 0; mt < 8; ++mt) {
        o[mt][0] *= c0;
        o[mt][1] *= c1;
        o[mt][2] *= c0;
        o[mt][3] *= c1;
      }
      m[0] = mn0;
      m[1] = mn1;
    }
    l[0] += p0 + p2;
    l[1] += p1 + p3;
    // P^T fragments -> B operand of O^T += V^T P^T
    const uint32_t pb0 = movtrans(pack_bf16(p0, p1));  // keys 0-7
    const uint32_t pb1 = movtrans(pack_bf16(p2, p3));  // keys 8-15
    const int vkey = (lane & 7) + ((lane >> 4) << 3);
#pragma unroll
    for (int mt = 0; mt < 8; ++mt) {
      uint32_t a0, a1, a2, a3;
      ldsm_x4_t(sv + swz(vkey, mt * 2 + ((lane >> 3) & 1)), a0, a1, a2, a3);
      mma16816(o[mt], a0, a1, a2, a3, pb0, pb1);
    }
    __syncwarp();  // every lane is done with stage st before lane 0 re-arms it
  }
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    l[h] += __shfl_xor_sync(0xffffffffu, l[h], 4);
    l[h] += __shfl_xor_sync(0xffffffffu, l[h], 8);
    l[h] += __shfl_xor_sync(0xffffffffu, l[h], 16);
  }
  group_sync();
  pdl_trigger();  // only the merge is left
  // merge the warps (heads h < G); the rings are no longer needed
  float* sm_o = reinterpret_cast<float*>(smem);  // [WARPS][8 heads][DH]
  float* sm_ml = sm_o + WARPS * 8 * DH;          // [WARPS][8][2]
  if (g == 0) {
    sm_ml[(warp * 8 + 2 * t4) * 2] = m[0];
    sm_ml[(warp * 8 + 2 * t4) * 2 + 1] = l[0];
    sm_ml[(warp * 8 + 2 * t4 + 1) * 2] = m[1];
    sm_ml[(warp * 8 + 2 * t4 + 1) * 2 + 1] = l[1];
  }
#pragma unroll
  for (int mt = 0; mt < 8; ++mt) {
    const int d0 = mt * 16 + g;
    sm_o[(warp * 8 + 2 * t4) * DH + d0] = o[mt][0];
    sm_o[(warp * 8 + 2 * t4 + 1) * DH + d0] = o[mt][1];
    sm_o[(warp * 8 + 2 * t4) * DH + d0 + 8] = o[mt][2];
    sm_o[(warp * 8 + 2 * t4 + 1) * DH + d0 + 8] = o[mt][3];
  }
  group_sync();
  for (int t = tid; t < G * DH; t += WARPS * 32) {
    const int h = t / DH, dim = t % DH;
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < WARPS; ++w) M = fmaxf(M, sm_ml[(w * 8 + h) * 2]);
    float L = 0.f, O = 0.f;
    if (M != -INFINITY) {
#pragma unroll
      for (int w = 0; w < WARPS; ++w) {
        const float c = exp2f(sm_ml[(w * 8 + h) * 2] - M);
        L += sm_ml[(w * 8 + h) * 2 + 1] * c;
        O += sm_o[(w * 8 + h) * DH + dim] * c;
      }
    }
    const int head = kvh * G + h;
    if (n_splits == 1) {
      bf16* out = reinterpret_cast<bf16*>(a.o) + (size_t)r * a.hq * DH + (size_t)head * DH;
      out[dim] = __float2bfloat16_rn(O / L);
    } else {
      const size_t base = ((size_t)r * a.hq + head) * a.max_splits + split;
      a.part_o[base * DH + dim] = O;
      if (dim == 0) {
        a.part_ml[base * 2] = M;
        a.part_ml[base * 2 + 1] = L;
      }
    }
  }
}

template <int WARPS, int NST, bool TMA>
__global__ void __launch_bounds__(WARPS * 32) decode_tc_kernel(const __grid_constant__ CUtensorMap map_k,
                                                                const __grid_constant__ CUtensorMap map_v,
                                                                DecodeAttnArgs a, int pps, int n_splits) {
  pdl_wait();
  if (a.dev_timer && threadIdx.x == 0) dev_timer_start(a.dev_timer);
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
  decode_tc_item<WARPS, NST, TMA>(&map_k, &map_v, a, pps, n_splits, (int)blockIdx.x, (int)blockIdx.y, (int)blockIdx.z,
                                  smem, (int)threadIdx.x, 0);
  if (a.dev_timer) {
    __syncthreads();
    if (threadIdx.x == 0) dev_timer_end(a.dev_timer);
  }
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
// pool viewed as [n_pages * h_kv * 16 rows][128 dims]; box = 16 rows x 64 dims, SWIZZLE_128B
static bool pool_map(CUtensorMap* m, const void* pool, uint64_t rows) {
  EncodeTiledFn fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {(cuuint64_t)DH, rows};
  cuuint64_t strides[1] = {(cuuint64_t)DH * 2};
  cuuint32_t box[2] = {64, PAGE};
  cuuint32_t es[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(pool), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

#endif  // DUET_BODIES_ONLY
}  // namespace dtc
#ifndef DUET_BODIES_ONLY

bool decode_tc_supported(const DecodeAttnArgs& a) {
  const int G = a.hq / a.hkv;
  return a.dh == dtc::DH && a.page_size == dtc::PAGE && G >= 1 && G <= 8 && a.n_pages > 0 &&
         dtc::encode_fn() != nullptr;
}

template <int W, int N, bool T>
static void launch_variant(const CUtensorMap& mk, const CUtensorMap& mv, const DecodeAttnArgs& a, int pps,
                           int n_splits, cudaStream_t st) {
  static bool attr = false;
  constexpr int smem = dtc::smem_bytes(W, N);
  if (!attr) {
    cudaFuncSetAttribute(dtc::decode_tc_kernel<W, N, T>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attr = true;
  }
  dim3 grid(n_splits, a.hkv, a.n);
  launch_pdl(dtc::decode_tc_kernel<W, N, T>, grid, 32 * W, smem, st, mk, mv, a, pps, n_splits);
}

int launch_decode_tc(const DecodeAttnArgs& a, int pps, int n_splits, cudaStream_t st) {
  CUtensorMap mk, mv;
  const uint64_t rows = (uint64_t)a.n_pages * a.hkv * dtc::PAGE;
  if (!dtc::pool_map(&mk, a.k_pool, rows) || !dtc::pool_map(&mv, a.v_pool, rows)) return -1;
  // variant (A/B measurements, tools/gpu/run_dec_ab.sh): DUET_DECODE = cp4x2 | cp4x3x2 | cp3x3 | cp2x3 |
  // tma8x3 | cp4x6 | cp8x3.  (A two-pages-per-iteration variant with 4-6 warps per SM was measured
  // 20-40 % slower on 8-48 SM partitions: warps hide the latency better than ILP.)
  static const char* v = getenv("DUET_DECODE");
  // Default: 4 warps per CTA with the per-warp ring depth chosen by the partition size — 2 stages
  // (3 CTAs = 12 warps per SM) on small partitions, where the kernel is latency-bound and warps hide
  // it best, 3 stages (2 CTAs per SM) on the full GPU.  Page -> warp assignment and the merge order
  // depend only on the 4 warps, so both give bitwise-identical results.
  const char* sel = v ? v : (a.num_sms < 120 ? "cp4x2" : "cp4x3x2");
  if (!strcmp(sel, "cp4x2")) launch_variant<4, 2, false>(mk, mv, a, pps, n_splits, st);   // 3 CTAs/SM
  else if (!strcmp(sel, "cp3x3")) launch_variant<3, 3, false>(mk, mv, a, pps, n_splits, st);   // 3 CTAs/SM
  else if (!strcmp(sel, "cp2x3")) launch_variant<2, 3, false>(mk, mv, a, pps, n_splits, st);   // 4 CTAs/SM
  else if (!strcmp(sel, "tma8x3")) launch_variant<8, 3, true>(mk, mv, a, pps, n_splits, st);
  else if (!strcmp(sel, "cp8x3")) launch_variant<8, 3, false>(mk, mv, a, pps, n_splits, st);
  else if (!strcmp(sel, "cp4x6")) launch_variant<4, 6, false>(mk, mv, a, pps, n_splits, st);
  else if (!strcmp(sel, "cp2x4x3")) launch_variant<2, 4, false>(mk, mv, a, pps, n_splits, st);
  else launch_variant<4, 3, false>(mk, mv, a, pps, n_splits, st);  // 96 KiB -> 2 CTAs per SM
  return 1;
}

#endif  // DUET_BODIES_ONLY
}  // namespace duet

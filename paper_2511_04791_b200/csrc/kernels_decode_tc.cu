// Paged decode attention on tensor cores (bf16, d_h = 128, GQA group G <= 16).
//
// The G query heads that share a kv head (reading #6) form the rows of a 16 x 128 Q tile (rows
// >= G are zero), so each 16-token page of K and V is read from HBM exactly once per request and
// consumed by two mma.sync m16n8k16 chains (S = Q K^T, 16 x 16; O += P V, 16 x 128) instead of
// warp-shuffle dot products.  One CTA per (split, kv head, request); each of the 4 warps streams
// its own pages (page w, w+4, ...) through a private 3-stage cp.async ring in shared memory
// (XOR-swizzled 256-byte rows, conflict-free ldmatrix); slots past the sequence end are zero-filled
// and masked.  Per-warp online softmax (exp2 domain); the 4 warps and the splits are merged with
// the log-sum-exp rule.  HBM traffic per request and layer: 2 h_kv (c+1) d_h s bytes.
#include "dev_common.cuh"
#include "kernels.h"

namespace duet {
namespace dtc {

constexpr int DH = 128, PAGE = 16, NST = 3, WARPS = 4;
constexpr int ROW_BYTES = DH * 2;
constexpr int PAGE_BYTES = PAGE * ROW_BYTES;  // 4 KiB: one kv head of one page
constexpr int STAGE_BYTES = 2 * PAGE_BYTES;   // K + V
constexpr int WARP_BYTES = NST * STAGE_BYTES;
constexpr int SMEM = WARPS * WARP_BYTES;      // 96 KiB

__device__ __forceinline__ uint32_t swz(int row, int chunk) {
  return (uint32_t)(row * ROW_BYTES + ((chunk ^ (row & 7)) << 4));
}
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void cp_async16(uint32_t dst, const void* src, bool valid) {
  const int sz = valid ? 16 : 0;
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(dst), "l"(src), "r"(sz) : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }
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
__device__ __forceinline__ void mma16816(float (&d)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
      "{%0,%1,%2,%3};"
      : "+f"(d[0]), "+f"(d[1]), "+f"(d[2]), "+f"(d[3])
      : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&h);
}

__global__ void __launch_bounds__(128) decode_tc_kernel(DecodeAttnArgs a, int pps, int n_splits) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int split = blockIdx.x, kvh = blockIdx.y, r = blockIdx.z;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int G = a.hq / a.hkv;
  const int len = a.pos[r] + 1;
  const int n_pages = (len + PAGE - 1) / PAGE;
  const int pg0 = split * pps;
  const int pg1 = min(n_pages, pg0 + pps);
  const int* tab = a.table + (size_t)a.tok_row[r] * a.max_pages;
  const bf16* Kg = reinterpret_cast<const bf16*>(a.k_pool);
  const bf16* Vg = reinterpret_cast<const bf16*>(a.v_pool);
  const size_t page_stride = (size_t)a.hkv * PAGE * DH;
  uint8_t* wsm = smem + warp * WARP_BYTES;
  const int g = lane >> 2, t4 = lane & 3;

  // Q fragments (A operand, rows = heads of the group, zero beyond G)
  uint32_t qf[8][4];
  {
    const bf16* qr = reinterpret_cast<const bf16*>(a.q) + (size_t)r * a.q_stride + (size_t)kvh * G * DH;
    const bool v0 = g < G, v1 = g + 8 < G;
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
      const int c0 = kk * 16 + 2 * t4;
      qf[kk][0] = v0 ? *reinterpret_cast<const uint32_t*>(qr + g * DH + c0) : 0u;
      qf[kk][1] = v1 ? *reinterpret_cast<const uint32_t*>(qr + (g + 8) * DH + c0) : 0u;
      qf[kk][2] = v0 ? *reinterpret_cast<const uint32_t*>(qr + g * DH + c0 + 8) : 0u;
      qf[kk][3] = v1 ? *reinterpret_cast<const uint32_t*>(qr + (g + 8) * DH + c0 + 8) : 0u;
    }
  }
  auto load_page = [&](int pg, int st) {
    const size_t base = (size_t)tab[pg] * page_stride + (size_t)kvh * PAGE * DH;
    const uint32_t sk = smem_u32(wsm + st * STAGE_BYTES), sv = sk + PAGE_BYTES;
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int idx = i * 32 + lane;  // 256 chunks of 16 B per tensor
      const int row = idx >> 4, ch = idx & 15;
      const bool v = pg * PAGE + row < len;
      const size_t off = v ? base + (size_t)row * DH + ch * 8 : 0;
      cp_async16(sk + swz(row, ch), Kg + off, v);
      cp_async16(sv + swz(row, ch), Vg + off, v);
    }
  };
  const float scale = rsqrtf((float)DH) * 1.4426950408889634f;
  float o[16][4];
#pragma unroll
  for (int j = 0; j < 16; ++j) o[j][0] = o[j][1] = o[j][2] = o[j][3] = 0.f;
  float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;

  const int first = pg0 + warp;
  int n_mine = first < pg1 ? (pg1 - first + WARPS - 1) / WARPS : 0;
#pragma unroll
  for (int i = 0; i < NST - 1; ++i) {
    if (i < n_mine) load_page(first + i * WARPS, i);
    cp_commit();
  }
  for (int i = 0; i < n_mine; ++i) {
    if (i + NST - 1 < n_mine) load_page(first + (i + NST - 1) * WARPS, (i + NST - 1) % NST);
    cp_commit();
    cp_wait<NST - 1>();
    __syncwarp();
    const int st = i % NST;
    const uint32_t sk = smem_u32(wsm + st * STAGE_BYTES), sv = sk + PAGE_BYTES;
    const int pg = first + i * WARPS;
    float s[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
#pragma unroll
    for (int kk = 0; kk < 8; ++kk) {
      const int key = (lane & 7) + ((lane >> 4) << 3);
      const int ch = kk * 2 + ((lane >> 3) & 1);
      uint32_t b0, b1, b2, b3;
      ldsm_x4(sk + swz(key, ch), b0, b1, b2, b3);
      mma16816(s[0], qf[kk], b0, b1);
      mma16816(s[1], qf[kk], b2, b3);
    }
    float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
    for (int j = 0; j < 2; ++j)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const bool v = pg * PAGE + j * 8 + 2 * t4 + e < len;
        s[j][e] = v ? s[j][e] * scale : -INFINITY;
        s[j][2 + e] = v ? s[j][2 + e] * scale : -INFINITY;
        mx0 = fmaxf(mx0, s[j][e]);
        mx1 = fmaxf(mx1, s[j][2 + e]);
      }
    mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 1));
    mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 2));
    mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 1));
    mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 2));
    const float mn0 = fmaxf(m0, mx0), mn1 = fmaxf(m1, mx1);  // finite: key 0 of a page is always valid
    const float c0 = exp2f(m0 - mn0), c1 = exp2f(m1 - mn1);
    m0 = mn0;
    m1 = mn1;
    float p[2][4];
    float s0 = 0.f, s1 = 0.f;
#pragma unroll
    for (int j = 0; j < 2; ++j) {
      p[j][0] = exp2f(s[j][0] - mn0);
      p[j][1] = exp2f(s[j][1] - mn0);
      p[j][2] = exp2f(s[j][2] - mn1);
      p[j][3] = exp2f(s[j][3] - mn1);
      s0 += p[j][0] + p[j][1];
      s1 += p[j][2] + p[j][3];
    }
    s0 += __shfl_xor_sync(0xffffffffu, s0, 1);
    s0 += __shfl_xor_sync(0xffffffffu, s0, 2);
    s1 += __shfl_xor_sync(0xffffffffu, s1, 1);
    s1 += __shfl_xor_sync(0xffffffffu, s1, 2);
    l0 = l0 * c0 + s0;
    l1 = l1 * c1 + s1;
    const uint32_t pf[4] = {pack_bf16(p[0][0], p[0][1]), pack_bf16(p[0][2], p[0][3]), pack_bf16(p[1][0], p[1][1]),
                            pack_bf16(p[1][2], p[1][3])};
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      o[j][0] *= c0;
      o[j][1] *= c0;
      o[j][2] *= c1;
      o[j][3] *= c1;
    }
#pragma unroll
    for (int nj = 0; nj < 8; ++nj) {
      const int key = (lane & 7) + (((lane >> 3) & 1) << 3);
      const int ch = nj * 2 + (lane >> 4);
      uint32_t v0, v1, v2, v3;
      ldsm_x4_t(sv + swz(key, ch), v0, v1, v2, v3);
      mma16816(o[2 * nj], pf, v0, v1);
      mma16816(o[2 * nj + 1], pf, v2, v3);
    }
    __syncwarp();
  }
  cp_wait<0>();
  __syncthreads();
  // merge the 4 warps: rows g < G only (row g + 8 is always padding for G <= 8)
  float* sm_o = reinterpret_cast<float*>(smem);             // [WARPS][16][DH]
  float* sm_ml = sm_o + WARPS * 16 * DH;                     // [WARPS][16][2]
  if (t4 == 0) {
    sm_ml[(warp * 16 + g) * 2] = m0;
    sm_ml[(warp * 16 + g) * 2 + 1] = l0;
    sm_ml[(warp * 16 + g + 8) * 2] = m1;
    sm_ml[(warp * 16 + g + 8) * 2 + 1] = l1;
  }
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    const int col = j * 8 + 2 * t4;
    sm_o[(warp * 16 + g) * DH + col] = o[j][0];
    sm_o[(warp * 16 + g) * DH + col + 1] = o[j][1];
    sm_o[(warp * 16 + g + 8) * DH + col] = o[j][2];
    sm_o[(warp * 16 + g + 8) * DH + col + 1] = o[j][3];
  }
  __syncthreads();
  for (int t = threadIdx.x; t < G * DH; t += blockDim.x) {
    const int gg = t / DH, dim = t % DH;
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < WARPS; ++w) M = fmaxf(M, sm_ml[(w * 16 + gg) * 2]);
    float L = 0.f, O = 0.f;
    if (M != -INFINITY) {
#pragma unroll
      for (int w = 0; w < WARPS; ++w) {
        const float c = exp2f(sm_ml[(w * 16 + gg) * 2] - M);
        L += sm_ml[(w * 16 + gg) * 2 + 1] * c;
        O += sm_o[(w * 16 + gg) * DH + dim] * c;
      }
    }
    const int head = kvh * G + gg;
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

}  // namespace dtc

bool decode_tc_supported(const DecodeAttnArgs& a) {
  const int G = a.hq / a.hkv;
  return a.dh == dtc::DH && a.page_size == dtc::PAGE && G >= 1 && G <= 8;
}

int launch_decode_tc(const DecodeAttnArgs& a, int pps, int n_splits, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(dtc::decode_tc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, dtc::SMEM);
    attr = true;
  }
  dim3 grid(n_splits, a.hkv, a.n);
  dtc::decode_tc_kernel<<<grid, 128, dtc::SMEM, st>>>(a, pps, n_splits);
  return 1;
}

}  // namespace duet

// Causal prefill attention over a paged KV cache (chunked prefill: a chunk of q tokens at positions
// c..c+q-1 attends to the c-token prefix and to itself causally; §4.1, readings #2,
// #6, #7).  bf16 tensor-core kernel (mma.sync m16n8k16, fp32 accumulation) in the flash-attention
// form: one CTA = 64 query rows of one query head; 4 warps x 16 rows; 64-key K/V tiles (4 pages of
// 16 tokens) streamed through a double-buffered, XOR-swizzled shared-memory ring with cp.async;
// online softmax in the exp2 domain; P re-used from the S accumulators as the A operand of P.V.
// Keys past the tile's causal end are zero-filled (unwritten page slots may hold anything).
#include "dev_common.cuh"
#include "kernels.h"

namespace duet {
namespace fa {

constexpr int BQ = 64, BKV = 64, DH = 128, PAGE = 16;
constexpr int ROW_BYTES = DH * 2;        // 256
constexpr int TILE_BYTES = BQ * ROW_BYTES;  // 16 KiB
constexpr int SMEM = TILE_BYTES * 5;     // Q + 2 x (K, V)

__device__ __forceinline__ uint32_t swz(int row, int chunk) {  // byte offset of 16-B chunk in a tile
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

__global__ void __launch_bounds__(128) fa_prefill_kernel(PrefillAttnArgs a, int n_qtiles) {
  extern __shared__ __align__(128) uint8_t smem[];
  uint8_t* sQ = smem;
  uint8_t* sK[2] = {smem + TILE_BYTES, smem + 3 * TILE_BYTES};
  uint8_t* sV[2] = {smem + 2 * TILE_BYTES, smem + 4 * TILE_BYTES};
  const int qt = n_qtiles - 1 - blockIdx.x;  // heavy (late) tiles first
  const int head = blockIdx.y, s = blockIdx.z;
  const int G = a.hq / a.hkv, kvh = head / G;
  const int qlen = a.qlen[s];
  if (qt * BQ >= qlen) return;
  const int row0 = a.row0[s], cpre = a.cpre[s];
  const int* tab = a.table + (size_t)a.seq_row[s] * a.max_pages;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int q_first = qt * BQ;                       // first query index in the chunk
  const int q_last = min(q_first + BQ, qlen) - 1;
  const int kv_end = cpre + q_last + 1;              // keys 0..kv_end-1 are visible to some row
  const int n_kt = (kv_end + BKV - 1) / BKV;
  const bf16* Qg = reinterpret_cast<const bf16*>(a.q);
  const bf16* Kg = reinterpret_cast<const bf16*>(a.k_pool);
  const bf16* Vg = reinterpret_cast<const bf16*>(a.v_pool);
  const size_t page_stride = (size_t)a.hkv * PAGE * DH;

  // Q tile -> smem (rows past qlen zero-filled)
  for (int i = tid; i < BQ * (DH / 8); i += 128) {
    const int r = i >> 4, ch = i & 15;
    const int qi = q_first + r;
    const bool v = qi < qlen;
    const bf16* src = Qg + (size_t)(row0 + (v ? qi : 0)) * a.q_stride + head * DH + ch * 8;
    cp_async16(smem_u32(sQ) + swz(r, ch), src, v);
  }
  auto load_kv = [&](int kt, int buf) {
    for (int i = tid; i < BKV * (DH / 8); i += 128) {
      const int r = i >> 4, ch = i & 15;
      const int key = kt * BKV + r;
      const bool v = key < kv_end;
      const int page = v ? tab[key / PAGE] : 0;
      const size_t off = (size_t)page * page_stride + ((size_t)kvh * PAGE + (key % PAGE)) * DH + ch * 8;
      cp_async16(smem_u32(sK[buf]) + swz(r, ch), Kg + (v ? off : 0), v);
      cp_async16(smem_u32(sV[buf]) + swz(r, ch), Vg + (v ? off : 0), v);
    }
  };
  load_kv(0, 0);
  cp_commit();

  const int g = lane >> 2, t4 = lane & 3;
  // query positions of this thread's two rows
  const int pos_r0 = cpre + q_first + warp * 16 + g;
  const int pos_r1 = pos_r0 + 8;
  const float scale = rsqrtf((float)DH) * 1.4426950408889634f;

  float o[16][4];
#pragma unroll
  for (int j = 0; j < 16; ++j) o[j][0] = o[j][1] = o[j][2] = o[j][3] = 0.f;
  float m0 = -INFINITY, m1 = -INFINITY, l0 = 0.f, l1 = 0.f;
  uint32_t qf[8][4];

  for (int kt = 0; kt < n_kt; ++kt) {
    const int buf = kt & 1;
    if (kt + 1 < n_kt) load_kv(kt + 1, buf ^ 1);
    cp_commit();
    cp_wait<1>();
    __syncthreads();
    if (kt == 0) {
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
        const int r = warp * 16 + (lane & 15);
        const int ch = kk * 2 + (lane >> 4);
        ldsm_x4(smem_u32(sQ) + swz(r, ch), qf[kk][0], qf[kk][1], qf[kk][2], qf[kk][3]);
      }
    }
    // skip the tile entirely for this warp if all its keys are in the causal future of all its rows
    const int warp_max_pos = cpre + min(q_first + warp * 16 + 15, qlen - 1);
    if (kt * BKV <= warp_max_pos) {
      // S = Q K^T : 16 x 64 per warp
      float sacc[8][4];
#pragma unroll
      for (int j = 0; j < 8; ++j) sacc[j][0] = sacc[j][1] = sacc[j][2] = sacc[j][3] = 0.f;
#pragma unroll
      for (int kk = 0; kk < 8; ++kk) {
#pragma unroll
        for (int nj = 0; nj < 4; ++nj) {  // pairs of n8 key tiles
          const int key = nj * 16 + (lane & 7) + ((lane >> 4) << 3);
          const int ch = kk * 2 + ((lane >> 3) & 1);
          uint32_t b0, b1, b2, b3;
          ldsm_x4(smem_u32(sK[buf]) + swz(key, ch), b0, b1, b2, b3);
          mma16816(sacc[2 * nj], qf[kk], b0, b1);
          mma16816(sacc[2 * nj + 1], qf[kk], b2, b3);
        }
      }
      // scale, causal mask, online softmax
      float mx0 = -INFINITY, mx1 = -INFINITY;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const int key0 = kt * BKV + j * 8 + 2 * t4;
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int key = key0 + e;
          sacc[j][e] = key <= pos_r0 ? sacc[j][e] * scale : -INFINITY;
          sacc[j][2 + e] = key <= pos_r1 ? sacc[j][2 + e] * scale : -INFINITY;
          mx0 = fmaxf(mx0, sacc[j][e]);
          mx1 = fmaxf(mx1, sacc[j][2 + e]);
        }
      }
      mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 1));
      mx0 = fmaxf(mx0, __shfl_xor_sync(0xffffffffu, mx0, 2));
      mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 1));
      mx1 = fmaxf(mx1, __shfl_xor_sync(0xffffffffu, mx1, 2));
      const float mn0 = fmaxf(m0, mx0), mn1 = fmaxf(m1, mx1);
      // rows with no visible key yet keep m = -inf; guard the exponent base
      const float b0 = mn0 == -INFINITY ? 0.f : mn0, b1 = mn1 == -INFINITY ? 0.f : mn1;
      const float c0 = exp2f(m0 - b0), c1 = exp2f(m1 - b1);
      m0 = mn0;
      m1 = mn1;
      float s0 = 0.f, s1 = 0.f;
      uint32_t pf[4][4];
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const float p0 = exp2f(sacc[j][0] - b0), p1 = exp2f(sacc[j][1] - b0);
        const float p2 = exp2f(sacc[j][2] - b1), p3 = exp2f(sacc[j][3] - b1);
        s0 += p0 + p1;
        s1 += p2 + p3;
        const int kk = j >> 1;
        if ((j & 1) == 0) {
          pf[kk][0] = pack_bf16(p0, p1);
          pf[kk][1] = pack_bf16(p2, p3);
        } else {
          pf[kk][2] = pack_bf16(p0, p1);
          pf[kk][3] = pack_bf16(p2, p3);
        }
      }
      s0 += __shfl_xor_sync(0xffffffffu, s0, 1);
      s0 += __shfl_xor_sync(0xffffffffu, s0, 2);
      s1 += __shfl_xor_sync(0xffffffffu, s1, 1);
      s1 += __shfl_xor_sync(0xffffffffu, s1, 2);
      l0 = l0 * c0 + s0;
      l1 = l1 * c1 + s1;
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        o[j][0] *= c0;
        o[j][1] *= c0;
        o[j][2] *= c1;
        o[j][3] *= c1;
      }
      // O += P V : k = 64 keys (4 k16 steps), n = 128 dims (16 n8 tiles)
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
#pragma unroll
        for (int nj = 0; nj < 8; ++nj) {
          const int key = kk * 16 + (lane & 7) + (((lane >> 3) & 1) << 3);
          const int ch = nj * 2 + (lane >> 4);
          uint32_t v0, v1, v2, v3;
          ldsm_x4_t(smem_u32(sV[buf]) + swz(key, ch), v0, v1, v2, v3);
          mma16816(o[2 * nj], pf[kk], v0, v1);
          mma16816(o[2 * nj + 1], pf[kk], v2, v3);
        }
      }
    }
    __syncthreads();
  }
  // normalise and store
  bf16* O = reinterpret_cast<bf16*>(a.o);
  const float inv0 = l0 > 0.f ? 1.f / l0 : 0.f, inv1 = l1 > 0.f ? 1.f / l1 : 0.f;
  const int qi0 = q_first + warp * 16 + g, qi1 = qi0 + 8;
#pragma unroll
  for (int j = 0; j < 16; ++j) {
    const int col = head * DH + j * 8 + 2 * t4;
    if (qi0 < qlen)
      *reinterpret_cast<__nv_bfloat162*>(O + (size_t)(row0 + qi0) * a.hq * DH + col) =
          __floats2bfloat162_rn(o[j][0] * inv0, o[j][1] * inv0);
    if (qi1 < qlen)
      *reinterpret_cast<__nv_bfloat162*>(O + (size_t)(row0 + qi1) * a.hq * DH + col) =
          __floats2bfloat162_rn(o[j][2] * inv1, o[j][3] * inv1);
  }
}

}  // namespace fa

bool fa_prefill_supported(const PrefillAttnArgs& a) { return a.dh == fa::DH && a.page_size == fa::PAGE; }

int launch_fa_prefill(const PrefillAttnArgs& a, cudaStream_t st) {
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(fa::fa_prefill_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, fa::SMEM);
    attr = true;
  }
  const int n_qt = (a.max_q + fa::BQ - 1) / fa::BQ;
  dim3 grid(n_qt, a.hq, a.n_seqs);
  fa::fa_prefill_kernel<<<grid, 128, fa::SMEM, st>>>(a, n_qt);
  return 1;
}

}  // namespace duet

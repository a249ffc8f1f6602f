// Paged decode attention for small SM partitions (bf16, d_h = 128, GQA group G <= 8): K straight into
// registers, V through shared memory — two load paths that run side by side.
//
// Why (tools/probes/probe_decode_bw.cu, profiles/r02_probe_decode_bw.txt): on a 16-48
// SM partition a kernel that stages every K/V byte in shared memory pays the smem bandwidth twice per
// byte (the fill and the operand read: ~121 GB/s/SM at most; the cp.async kernel reached 98), and random
// 4-KiB blocks loaded into registers top out near 85-120 GB/s/SM.  Here the K page of a (page, kv head)
// goes global -> registers with 16-B LDGs laid out as the MMA A fragment (no shared memory at all), and
// the V page goes global -> shared with two 1-D bulk copies (TMA, no tensor map) completing on an
// mbarrier, read back once with conflict-free 16-B LDS; each path carries half of the bytes.
//
// The math is the transposed form of kernels_decode_tc.cu: the 16 tokens of a page fill the MMA M
// dimension and the G query heads of a kv group (reading #6) fill N = 8:
//   S^T (16 tokens x 8 heads) = K_page (16 x 128) . Q^T (128 x 8)              8 x mma.m16n8k16
//   O^T (128 dims x 8 heads) += V_page^T (128 x 16) . P^T (16 x 8)              8 x mma.m16n8k16
// Two free permutations make the register layouts work without shared memory or bank conflicts:
//  * tokens: MMA row r (0..15) is page token tau(r) = 8 (g & 1) + (g >> 1) + 4 (r >> 3), g = r & 7 — odd
//    rows come from the page's second half, which the bulk copy places 64 B (mod 128) away from the
//    first, so the 8 lanes of an LDS.128 phase (rows g = 2p, 2p+1) hit 8 distinct 16-B bank groups;
//  * dims: lane (g, t) owns the 16-B chunks t, t+4, t+8, t+12 of a token row; k-step 2i + hh of S^T
//    takes chunk 4i + t's elements {4hh, 4hh+1} at k = 2t, 2t+1 and {4hh+2, 4hh+3} at k = 2t+8, 2t+9,
//    with Q^T's B fragment loaded in the same order, so every K chunk is one 16-B load.
// V's chunks become the V^T A fragment through movmatrix.trans of 8x8 tiles; an m-tile's accumulator
// rows are then the dims D(i, u, g) = 8 (4i + (g >> 1)) + 2u + (g & 1), resolved when O is stored.
// Online softmax per head in the exp2 domain; warps and splits merge with the log-sum-exp rule exactly
// as kernels_decode_tc.cu (same page -> warp assignment, same split counts, same combine kernel).
#include <cstdlib>
#include <cstring>

#include "dev_common.cuh"
#include "kernels.h"

namespace duet {
namespace dhy {

constexpr int DH = 128, PAGE = 16;
constexpr int HALF_B = 2048 + 64;        // smem offset of tokens 8..15 (64 B past the 2 KiB of tokens 0..7)
constexpr int STAGE = 4096 + 128;        // one V page (two halves + the skew), 128-B aligned stages

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(bar),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ uint4 ldg_ef(const void* p, uint64_t pol) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ uint4 lds128(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(addr));
  return v;
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
__device__ __forceinline__ float fast_exp2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ uint32_t pack_bf16(float lo, float hi) {
  __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);
  return *reinterpret_cast<uint32_t*>(&h);
}
__device__ __forceinline__ uint32_t u4(const uint4& v, int j) { return j == 0 ? v.x : j == 1 ? v.y : j == 2 ? v.z : v.w; }
// page token of MMA row r
__device__ __forceinline__ int tau(int r) { return ((r & 1) << 3) + ((r & 7) >> 1) + ((r >> 3) << 2); }

template <int WARPS, int NV>
__host__ __device__ constexpr int smem_bytes() {
  return WARPS * NV * STAGE + WARPS * NV * 8 + 128;
}

// One CTA per (split, kv head, request); WARPS warps take pages w, w + WARPS, ... of the split; each warp
// has NV V stages in shared memory and K prefetched one page ahead in registers.
template <int WARPS, int NV, int MINB>
__global__ void __launch_bounds__(WARPS * 32, MINB) decode_hyb_kernel(DecodeAttnArgs a, int pps, int n_splits) {
  extern __shared__ __align__(128) uint8_t smem[];
  pdl_wait();
  const int split = blockIdx.x, kvh = blockIdx.y, r = blockIdx.z;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t4 = lane & 3;
  const int G = a.hq / a.hkv;
  const int len = a.pos[r] + 1;
  const int n_pages = (len + PAGE - 1) / PAGE;
  const int pg0 = split * pps;
  const int pg1 = min(n_pages, pg0 + pps);
  const int* tab = a.table + (size_t)a.tok_row[r] * a.max_pages;
  uint8_t* ring = smem + warp * NV * STAGE;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + WARPS * NV * STAGE) + warp * NV;
  const uint32_t ring_s = smem_u32(ring), bar_s = smem_u32(bars);
  if (lane == 0) {
    for (int i = 0; i < NV; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(bar_s + 8 * i));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncwarp();
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));

  // Q^T B fragments in the chunk order of the K loads: qb[2i + hh] = {Q[g][d0+4hh..+1], Q[g][d0+4hh+2..+3]},
  // d0 = 8 (4i + t); zero for padding heads g >= G
  uint32_t qb[8][2];
  {
    const bf16* qr = reinterpret_cast<const bf16*>(a.q) + (size_t)r * a.q_stride + (size_t)kvh * G * DH + g * DH;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint4 v = g < G ? *reinterpret_cast<const uint4*>(qr + 8 * (4 * i + t4)) : make_uint4(0, 0, 0, 0);
      qb[2 * i][0] = v.x;
      qb[2 * i][1] = v.y;
      qb[2 * i + 1][0] = v.z;
      qb[2 * i + 1][1] = v.w;
    }
  }
  const int first = pg0 + warp;
  const int n_mine = first < pg1 ? (pg1 - first + WARPS - 1) / WARPS : 0;
  // page-table entries of this warp's pages, 32 at a time, broadcast by shuffles (kernels_decode_tc.cu)
  auto tab_batch = [&](int b) {
    const int i = b * 32 + lane;
    return i < n_mine ? __ldg(tab + first + i * WARPS) : 0;
  };
  // lane L holds the entries of pages 32 b0 + L (pt_cur) and 32 (b0 + 1) + L (pt_next): any index in
  // [32 b0, 32 b0 + 64) is one shuffle away; advance_to(j) slides the window before index j is used
  int b0 = 0, pt_cur = tab_batch(0), pt_next = tab_batch(1);
  auto advance_to = [&](int j) {
    while (j >= 32 * (b0 + 2)) {
      pt_cur = pt_next;
      pt_next = tab_batch(b0 + 2);
      ++b0;
    }
  };
  auto page_of = [&](int i) {  // warp-uniform i in the window, all lanes participate
    return __shfl_sync(0xffffffffu, (i >> 5) == b0 ? pt_cur : pt_next, i & 31);
  };
  const size_t blk = (size_t)PAGE * DH;  // elements of one (page, kv head) block
  const int tk0 = tau(g), tk1 = tau(g + 8);
  // this lane's K row offsets (elements) inside a block: rows tau(g), tau(g+8), chunks 4i + t
  const int koff0 = tk0 * DH + 8 * t4, koff1 = tk1 * DH + 8 * t4;
  auto load_k = [&](int pid, uint4 (&kr)[2][4]) {
    const bf16* kb = reinterpret_cast<const bf16*>(a.k_pool) + ((size_t)pid * a.hkv + kvh) * blk;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      kr[0][i] = ldg_ef(kb + koff0 + 32 * i, pol);
      kr[1][i] = ldg_ef(kb + koff1 + 32 * i, pol);
    }
  };
  auto issue_v = [&](int i, int pid) {  // lane 0: page i's V block into stage i % NV (two bulk copies)
    const int st = i % NV;
    const char* src = reinterpret_cast<const char*>(a.v_pool) + ((size_t)pid * a.hkv + kvh) * blk * 2;
    const uint32_t dst = ring_s + st * STAGE, bar = bar_s + 8 * st;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 4096;" ::"r"(bar) : "memory");
    asm volatile(
        "cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], 2048, [%2], %3;" ::"r"(
            dst),
        "l"(src), "r"(bar), "l"(pol)
        : "memory");
    asm volatile(
        "cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], 2048, [%2], %3;" ::"r"(
            dst + HALF_B),
        "l"(src + 2048), "r"(bar), "l"(pol)
        : "memory");
  };
  // V^T fragments: this lane's LDS.128 addresses (rows tau(g), tau(g+8), chunk 4i + t)
  const uint32_t voff0 = (tk0 < 8 ? tk0 * 256 : HALF_B + (tk0 - 8) * 256) + 16 * t4;
  const uint32_t voff1 = (tk1 < 8 ? tk1 * 256 : HALF_B + (tk1 - 8) * 256) + 16 * t4;

  for (int i = 0; i < NV - 1 && i < n_mine; ++i) {
    const int pid = page_of(i);
    if (lane == 0) issue_v(i, pid);
  }
  uint4 kc[2][4], kn[2][4];
  if (n_mine > 0) load_k(page_of(0), kc);

  const float scale = rsqrtf((float)DH) * 1.4426950408889634f;
  float o[8][4];
#pragma unroll
  for (int j = 0; j < 8; ++j) o[j][0] = o[j][1] = o[j][2] = o[j][3] = 0.f;
  float m[2] = {-INFINITY, -INFINITY}, l[2] = {0.f, 0.f};  // heads 2t, 2t+1

  auto page = [&](int i, uint4 (&kcur)[2][4], uint4 (&knext)[2][4]) {
    // V for page i + NV - 1 (its stage was consumed at iteration i - 1) and K for page i + 1
    advance_to(i + NV - 1);  // the largest index this iteration uses (i + 1 <= i + NV - 1 stays inside)
    if (i + NV - 1 < n_mine) {
      const int pid = page_of(i + NV - 1);
      if (lane == 0) issue_v(i + NV - 1, pid);
    }
    if (i + 1 < n_mine) load_k(page_of(i + 1), knext);
    const int key0 = (first + i * WARPS) * PAGE;
    // S^T = K Q^T, two accumulation chains
    float s[4] = {0.f, 0.f, 0.f, 0.f}, s2[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      mma16816(s, kcur[0][c].x, kcur[1][c].x, kcur[0][c].y, kcur[1][c].y, qb[2 * c][0], qb[2 * c][1]);
      mma16816(s2, kcur[0][c].z, kcur[1][c].z, kcur[0][c].w, kcur[1][c].w, qb[2 * c + 1][0], qb[2 * c + 1][1]);
    }
    // s[0], s[1]: token tau(g), heads 2t, 2t+1 ; s[2], s[3]: token tau(g+8)
    const bool v0 = key0 + tk0 < len, v1 = key0 + tk1 < len;
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
    // token 0 of a page (MMA row 0) is always valid, so the new maxima are finite
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
    const uint32_t pb0 = movtrans(pack_bf16(p0, p1));  // MMA rows 0-7
    const uint32_t pb1 = movtrans(pack_bf16(p2, p3));  // MMA rows 8-15
    // V^T: wait for the stage, 8 conflict-free LDS.128, zero the rows past the sequence end (unwritten
    // slots may hold anything; P is 0 there but 0 x NaN is not)
    const int st = i % NV;
    mbar_wait(bar_s + 8 * st, (i / NV) & 1);
    const uint32_t sb = ring_s + st * STAGE;
    uint4 vr[2][4];
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      vr[0][c] = lds128(sb + voff0 + 64 * c);
      vr[1][c] = lds128(sb + voff1 + 64 * c);
    }
    if (!v0) {
#pragma unroll
      for (int c = 0; c < 4; ++c) vr[0][c] = make_uint4(0, 0, 0, 0);
    }
    if (!v1) {
#pragma unroll
      for (int c = 0; c < 4; ++c) vr[1][c] = make_uint4(0, 0, 0, 0);
    }
    // m-tile 2c + e: rows 0-7 = dims D(c, 2e, g), rows 8-15 = D(c, 2e + 1, g)
#pragma unroll
    for (int c = 0; c < 4; ++c) {
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const uint32_t a0 = movtrans(u4(vr[0][c], 2 * e)), a1 = movtrans(u4(vr[0][c], 2 * e + 1));
        const uint32_t a2 = movtrans(u4(vr[1][c], 2 * e)), a3 = movtrans(u4(vr[1][c], 2 * e + 1));
        mma16816(o[2 * c + e], a0, a1, a2, a3, pb0, pb1);
      }
    }
    __syncwarp();  // every lane has read stage st before lane 0 refills it (next iteration)
  };
  int i = 0;
  for (; i + 1 < n_mine; i += 2) {
    page(i, kc, kn);
    page(i + 1, kn, kc);
  }
  if (i < n_mine) page(i, kc, kn);

#pragma unroll
  for (int h = 0; h < 2; ++h) {
    l[h] += __shfl_xor_sync(0xffffffffu, l[h], 4);
    l[h] += __shfl_xor_sync(0xffffffffu, l[h], 8);
    l[h] += __shfl_xor_sync(0xffffffffu, l[h], 16);
  }
  __syncthreads();
  pdl_trigger();
  // merge the warps (heads h < G); the rings are no longer needed
  float* sm_o = reinterpret_cast<float*>(smem);  // [WARPS][8 heads][DH]
  float* sm_ml = sm_o + WARPS * 8 * DH;          // [WARPS][8][2]
  if (g == 0) {
    sm_ml[(warp * 8 + 2 * t4) * 2] = m[0];
    sm_ml[(warp * 8 + 2 * t4) * 2 + 1] = l[0];
    sm_ml[(warp * 8 + 2 * t4 + 1) * 2] = m[1];
    sm_ml[(warp * 8 + 2 * t4 + 1) * 2 + 1] = l[1];
  }
  // accumulator rows -> dims: m-tile 2c + e, row g -> D(c, 2e, g), row g + 8 -> D(c, 2e + 1, g)
#pragma unroll
  for (int c = 0; c < 4; ++c) {
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int dA = 8 * (4 * c + (g >> 1)) + 4 * e + (g & 1), dB = dA + 2;
      sm_o[(warp * 8 + 2 * t4) * DH + dA] = o[2 * c + e][0];
      sm_o[(warp * 8 + 2 * t4 + 1) * DH + dA] = o[2 * c + e][1];
      sm_o[(warp * 8 + 2 * t4) * DH + dB] = o[2 * c + e][2];
      sm_o[(warp * 8 + 2 * t4 + 1) * DH + dB] = o[2 * c + e][3];
    }
  }
  __syncthreads();
  for (int t = threadIdx.x; t < G * DH; t += blockDim.x) {
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

}  // namespace dhy

template <int W, int NV, int MINB>
static void launch_hyb_variant(const DecodeAttnArgs& a, int pps, int n_splits, cudaStream_t st) {
  static bool attr = false;
  constexpr int smem = dhy::smem_bytes<W, NV>();
  if (!attr) {
    cudaFuncSetAttribute(dhy::decode_hyb_kernel<W, NV, MINB>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    attr = true;
  }
  dim3 grid(n_splits, a.hkv, a.n);
  launch_pdl(dhy::decode_hyb_kernel<W, NV, MINB>, grid, 32 * W, smem, st, a, pps, n_splits);
}

bool decode_hyb_supported(const DecodeAttnArgs& a) {
  const int G = a.hq / a.hkv;
  return a.dh == dhy::DH && a.page_size == dhy::PAGE && G >= 1 && G <= 8 && (a.q_stride % 8) == 0 &&
         ((uintptr_t)a.q & 15) == 0 && ((uintptr_t)a.k_pool & 15) == 0 && ((uintptr_t)a.v_pool & 15) == 0;
}

// variant: "hy4x3" (4 warps, 3 V stages per warp), "hy4x4", "hy4x2", "hy2x4"
int launch_decode_hyb(const DecodeAttnArgs& a, int pps, int n_splits, const char* variant, cudaStream_t st) {
  // hyWxNV[xB]: W warps per CTA, NV V stages per warp, at least B CTAs per SM (register cap)
  if (!strcmp(variant, "hy4x4")) launch_hyb_variant<4, 4, 3>(a, pps, n_splits, st);
  else if (!strcmp(variant, "hy4x2")) launch_hyb_variant<4, 2, 3>(a, pps, n_splits, st);
  else if (!strcmp(variant, "hy4x3x2")) launch_hyb_variant<4, 3, 2>(a, pps, n_splits, st);
  else if (!strcmp(variant, "hy4x2x4")) launch_hyb_variant<4, 2, 4>(a, pps, n_splits, st);
  else if (!strcmp(variant, "hy2x4")) launch_hyb_variant<2, 4, 6>(a, pps, n_splits, st);
  else launch_hyb_variant<4, 3, 3>(a, pps, n_splits, st);
  return 1;
}

}  // namespace duet

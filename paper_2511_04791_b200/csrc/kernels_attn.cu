// Paged attention kernels.
//
// decode_attn_kernel — split-K paged decode attention ("concatenate then attend",
// P:142 "KV cache reads dominate runtime as the context grows"): one CTA per
// (split, kv head, request) reads its range of 16-token pages once for all G = h_q/h_kv query
// heads of the group (reading #6), with 16-byte coalesced non-allocating loads, warp-shuffle
// dot products and an online softmax in the exp2 domain; partial (O, m, l) per split are
// merged by an LSE combine.  The same kernel evaluates any set of single query rows, so it is
// also the SIMT path of causal prefill attention (one row at position p reads keys 0..p,
// reading #7) used by the fp32 mode.
#include <cfloat>

#include "dev_common.cuh"
#include "kernels.h"

namespace duet {

constexpr int kPage = 16;
constexpr float kLog2e = 1.4426950408889634f;

template <typename T, int DH, int G>
__global__ void __launch_bounds__(128) decode_attn_kernel(DecodeAttnArgs a, int pages_per_split, int n_splits) {
  constexpr int E = 16 / sizeof(T);
  constexpr int LPK = DH / E;    // lanes sharing one key row
  constexpr int KPI = 32 / LPK;  // keys per warp iteration
  constexpr int IT = kPage / KPI;
  static_assert(LPK <= 32 && 32 % LPK == 0, "head_dim layout");
  const int split = blockIdx.x, kvh = blockIdx.y, r = blockIdx.z;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int len = a.pos[r] + 1;
  const int n_pages = (len + kPage - 1) / kPage;
  const int pg0 = split * pages_per_split;
  const int pg1 = min(n_pages, pg0 + pages_per_split);
  const int* tab = a.table + (size_t)a.tok_row[r] * a.max_pages;
  const int dsl = (lane % LPK) * E;
  const int kslot = lane / LPK;

  float q[G][E];
  const T* qr = reinterpret_cast<const T*>(a.q) + (size_t)r * a.q_stride + (size_t)kvh * G * DH;
  const float scale = rsqrtf((float)DH) * kLog2e;
#pragma unroll
  for (int g = 0; g < G; ++g) {
    load16<T>(qr + g * DH + dsl, q[g]);
#pragma unroll
    for (int e = 0; e < E; ++e) q[g][e] *= scale;
  }
  float m[G], l[G], acc[G][E];
#pragma unroll
  for (int g = 0; g < G; ++g) {
    m[g] = -INFINITY;
    l[g] = 0.f;
#pragma unroll
    for (int e = 0; e < E; ++e) acc[g][e] = 0.f;
  }
  const size_t page_stride = (size_t)a.hkv * kPage * DH;
  const T* kbase = reinterpret_cast<const T*>(a.k_pool) + (size_t)kvh * kPage * DH;
  const T* vbase = reinterpret_cast<const T*>(a.v_pool) + (size_t)kvh * kPage * DH;

  for (int pg = pg0 + warp; pg < pg1; pg += 4) {
    const size_t page = (size_t)tab[pg];
    const T* kp = kbase + page * page_stride;
    const T* vp = vbase + page * page_stride;
    uint4 kr[IT], vr[IT];
#pragma unroll
    for (int it = 0; it < IT; ++it) kr[it] = ldg_nc16(kp + (it * KPI + kslot) * DH + dsl);
#pragma unroll
    for (int it = 0; it < IT; ++it) vr[it] = ldg_nc16(vp + (it * KPI + kslot) * DH + dsl);
    float s[G][IT];
#pragma unroll
    for (int it = 0; it < IT; ++it) {
      float kf[E];
      cvt16<T>(kr[it], kf);
      const bool valid = pg * kPage + it * KPI + kslot < len;
#pragma unroll
      for (int g = 0; g < G; ++g) {
        float part = 0.f;
#pragma unroll
        for (int e = 0; e < E; ++e) part += q[g][e] * kf[e];
#pragma unroll
        for (int o = LPK / 2; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
        s[g][it] = valid ? part : -INFINITY;
      }
    }
    float mnew[G], corr[G];
#pragma unroll
    for (int g = 0; g < G; ++g) {
      float mx = s[g][0];
#pragma unroll
      for (int it = 1; it < IT; ++it) mx = fmaxf(mx, s[g][it]);
#pragma unroll
      for (int o = LPK; o < 32; o <<= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      mnew[g] = fmaxf(m[g], mx);
      corr[g] = exp2f(m[g] - mnew[g]);  // m = -inf -> 0
      l[g] *= corr[g];
#pragma unroll
      for (int e = 0; e < E; ++e) acc[g][e] *= corr[g];
    }
    float psum[G];
#pragma unroll
    for (int g = 0; g < G; ++g) psum[g] = 0.f;
#pragma unroll
    for (int it = 0; it < IT; ++it) {
      float vf[E];
      cvt16<T>(vr[it], vf);
      const bool valid = pg * kPage + it * KPI + kslot < len;
#pragma unroll
      for (int e = 0; e < E; ++e) vf[e] = valid ? vf[e] : 0.f;  // masked slots may hold anything
#pragma unroll
      for (int g = 0; g < G; ++g) {
        const float p = exp2f(s[g][it] - mnew[g]);
        psum[g] += p;
#pragma unroll
        for (int e = 0; e < E; ++e) acc[g][e] += p * vf[e];
      }
    }
#pragma unroll
    for (int g = 0; g < G; ++g) {
#pragma unroll
      for (int o = LPK; o < 32; o <<= 1) psum[g] += __shfl_xor_sync(0xffffffffu, psum[g], o);
      l[g] += psum[g];
      m[g] = mnew[g];
    }
  }
  // reduce acc over the key slots of the warp
#pragma unroll
  for (int g = 0; g < G; ++g)
#pragma unroll
    for (int e = 0; e < E; ++e)
#pragma unroll
      for (int o = LPK; o < 32; o <<= 1) acc[g][e] += __shfl_xor_sync(0xffffffffu, acc[g][e], o);

  __shared__ float sm_m[4][G], sm_l[4][G];
  __shared__ float sm_acc[4][G][DH];
  if (lane == 0) {
#pragma unroll
    for (int g = 0; g < G; ++g) {
      sm_m[warp][g] = m[g];
      sm_l[warp][g] = l[g];
    }
  }
  if (kslot == 0) {
#pragma unroll
    for (int g = 0; g < G; ++g)
#pragma unroll
      for (int e = 0; e < E; ++e) sm_acc[warp][g][dsl + e] = acc[g][e];
  }
  __syncthreads();
  for (int t = threadIdx.x; t < G * DH; t += blockDim.x) {
    const int g = t / DH, dim = t % DH;
    float M = -INFINITY;
#pragma unroll
    for (int w = 0; w < 4; ++w) M = fmaxf(M, sm_m[w][g]);
    float L = 0.f, O = 0.f;
    if (M != -INFINITY) {
#pragma unroll
      for (int w = 0; w < 4; ++w) {
        const float c = exp2f(sm_m[w][g] - M);
        L += sm_l[w][g] * c;
        O += sm_acc[w][g][dim] * c;
      }
    }
    const int head = kvh * G + g;
    if (n_splits == 1) {
      T* o = reinterpret_cast<T*>(a.o) + (size_t)r * a.hq * DH + (size_t)head * DH;
      o[dim] = from_f<T>(O / L);
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

// LSE combine of the split partials: o = sum_s O_s 2^(m_s - M) / sum_s l_s 2^(m_s - M).
template <typename T>
__global__ void attn_combine_kernel(DecodeAttnArgs a, int n_splits) {
  pdl_wait();
  const int rh = blockIdx.x;  // r * hq + head
  const size_t base = (size_t)rh * a.max_splits;
  float M = -INFINITY;
  for (int s = 0; s < n_splits; ++s)
    if (a.part_ml[(base + s) * 2 + 1] > 0.f) M = fmaxf(M, a.part_ml[(base + s) * 2]);
  for (int dim = threadIdx.x; dim < a.dh; dim += blockDim.x) {
    float L = 0.f, O = 0.f;
    for (int s = 0; s < n_splits; ++s) {
      const float ls = a.part_ml[(base + s) * 2 + 1];
      if (!(ls > 0.f)) continue;
      const float c = exp2f(a.part_ml[(base + s) * 2] - M);
      L += ls * c;
      O += a.part_o[(base + s) * a.dh + dim] * c;
    }
    reinterpret_cast<T*>(a.o)[(size_t)rh * a.dh + dim] = from_f<T>(O / L);
  }
}

template <typename T, int DH>
static void dispatch_g(const DecodeAttnArgs& a, dim3 grid, int pps, int ns, cudaStream_t st, bool* ok) {
  const int G = a.hq / a.hkv;
  switch (G) {
    case 1: decode_attn_kernel<T, DH, 1><<<grid, 128, 0, st>>>(a, pps, ns); break;
    case 2: decode_attn_kernel<T, DH, 2><<<grid, 128, 0, st>>>(a, pps, ns); break;
    case 4: decode_attn_kernel<T, DH, 4><<<grid, 128, 0, st>>>(a, pps, ns); break;
    case 5: decode_attn_kernel<T, DH, 5><<<grid, 128, 0, st>>>(a, pps, ns); break;
    case 8: decode_attn_kernel<T, DH, 8><<<grid, 128, 0, st>>>(a, pps, ns); break;
    default: *ok = false;
  }
}

// split plan of a decode batch: (pages per split, splits) from the batch shape only
static void decode_split_plan(const DecodeAttnArgs& a, int* pps_out, int* ns_out) {
  const int max_pages = (a.max_len + kPage - 1) / kPage;
  const int base = a.n * a.hkv;
  const int target = 148 * 4;
  int ns = (target + base - 1) / base;
  ns = ns < 1 ? 1 : ns;
  const int cap_pages = (max_pages + 3) / 4;
  if (ns > cap_pages) ns = cap_pages;
  if (ns > a.max_splits) ns = a.max_splits;
  if (ns < 1) ns = 1;
  const int pps = (max_pages + ns - 1) / ns;
  *ns_out = (max_pages + pps - 1) / pps;
  *pps_out = pps;
}

// f4 fused launch (kernels_pod.cu) + the LSE combine when the decode batch splits
int launch_pod_attn(DT dt, const PrefillAttnArgs& pa, const DecodeAttnArgs& da, int n_dec_ctas, cudaStream_t st) {
  if (dt != DT::BF16 || pa.total_q <= 0 || da.n <= 0) return -1;
  int pps, ns;
  decode_split_plan(da, &pps, &ns);
  if (launch_pod_tc(pa, da, pps, ns, n_dec_ctas, st) <= 0) return -1;
  if (ns > 1) {
    launch_pdl(attn_combine_kernel<bf16>, da.n * da.hq, 128, 0, st, da, ns);
    return 2;
  }
  return 1;
}

int launch_decode_attn(DT dt, const DecodeAttnArgs& a, cudaStream_t st) {
  if (a.n <= 0) return 0;
  // The split count depends only on the batch shape (never on the partition size), so a
  // request's result is bitwise identical whichever SM split or mode runs it.
  int pps, ns;
  decode_split_plan(a, &pps, &ns);
  dim3 grid(ns, a.hkv, a.n);
  bool ok = true;
  if (dt == DT::BF16 && decode_tc_supported(a)) {
    if (launch_decode_tc(a, pps, ns, st) < 0) ok = false;
  } else if (dt == DT::BF16) {
    if (a.dh == 128) dispatch_g<bf16, 128>(a, grid, pps, ns, st, &ok);
    else if (a.dh == 64) dispatch_g<bf16, 64>(a, grid, pps, ns, st, &ok);
    else ok = false;
  } else {
    if (a.dh == 128) dispatch_g<float, 128>(a, grid, pps, ns, st, &ok);
    else if (a.dh == 64) dispatch_g<float, 64>(a, grid, pps, ns, st, &ok);
    else ok = false;
  }
  if (!ok) return -1;
  if (ns > 1) {
    if (dt == DT::BF16) launch_pdl(attn_combine_kernel<bf16>, a.n * a.hq, 128, 0, st, a, ns);
    else attn_combine_kernel<float><<<a.n * a.hq, 128, 0, st>>>(a, ns);
    return 2;
  }
  return 1;
}

// Causal prefill attention.  fp32 (and bf16 until the tensor-core kernel takes over): each
// chunk row is an independent query at its absolute position, evaluated by the decode kernel.
int launch_prefill_attn(DT dt, const PrefillAttnArgs& p, cudaStream_t st) {
  if (p.total_q <= 0) return 0;
  if (dt == DT::BF16) {
    static const char* impl = getenv("DUET_FA");  // "mma": force the mma.sync kernel (A/B comparisons)
    const bool force_mma = impl && impl[0] == 'm';
    if (!force_mma && fa2_tc_supported(p)) {
      const int r = launch_fa2_tc(p, st);
      if (r > 0) return r;
    }
    if (!force_mma && fa_tc_supported(p)) {
      const int r = launch_fa_tc(p, st);
      if (r > 0) return r;
    }
    if (fa_prefill_supported(p)) return launch_fa_prefill(p, st);
  }
  DecodeAttnArgs a{};
  a.q = p.q;
  a.q_stride = p.q_stride;
  a.o = p.o;
  a.n = p.total_q;
  a.hq = p.hq;
  a.hkv = p.hkv;
  a.dh = p.dh;
  a.pos = p.tok_pos;
  a.tok_row = p.tok_row;
  a.table = p.table;
  a.max_pages = p.max_pages;
  a.page_size = p.page_size;
  a.k_pool = p.k_pool;
  a.v_pool = p.v_pool;
  a.part_o = nullptr;
  a.part_ml = nullptr;
  a.max_splits = 1;
  a.num_sms = p.num_sms;
  a.max_len = p.max_len;
  return launch_decode_attn(dt, a, st);
}

}  // namespace duet

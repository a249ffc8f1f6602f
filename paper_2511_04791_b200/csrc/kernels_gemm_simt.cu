// SIMT GEMM with fused epilogues — the fp32 path (1e-4 parity mode; tcgen05 kind::tf32 keeps
// a 10-bit mantissa and cannot meet it) and the fallback for shapes the tensor-core kernel
// does not tile.  C = epi(A . B^T), both operands K-major (nn.Linear layout), fp32 FFMA
// accumulation.  Epilogues: bias, residual (x + u, P:95-97 reading #1), SwiGLU (reading #3).
#include "dev_common.cuh"
#include "kernels.h"

namespace duet {

template <typename T, int EPI>
__global__ void __launch_bounds__(256) gemm_simt_kernel(GemmArgs g) {
  constexpr int BM = 64, BN = 64, BK = 16;
  __shared__ float As[BK][BM + 4];
  __shared__ float Bs[BK][BN + 4];
  __shared__ float Bu[EPI == EPI_SWIGLU ? BK : 1][BN + 4];
  const T* A = reinterpret_cast<const T*>(g.A);
  const T* B = reinterpret_cast<const T*>(g.B);
  const int m0 = blockIdx.y * BM, n0 = blockIdx.x * BN;
  const int tid = threadIdx.x, tx = tid % 16, ty = tid / 16;
  float acc[4][4] = {}, accu[4][4] = {};
  for (int k0 = 0; k0 < g.K; k0 += BK) {
    for (int i = tid; i < BM * BK; i += 256) {
      const int r = i / BK, c = i % BK;
      const int gm = m0 + r, gn = n0 + r;
      As[c][r] = gm < g.M ? to_f(A[(size_t)gm * g.lda + k0 + c]) : 0.f;
      Bs[c][r] = gn < g.N ? to_f(B[(size_t)gn * g.ldb + k0 + c]) : 0.f;
      if constexpr (EPI == EPI_SWIGLU) Bu[c][r] = gn < g.N ? to_f(B[(size_t)(g.N + gn) * g.ldb + k0 + c]) : 0.f;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < BK; ++k) {
      float a[4], b[4], bu[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        a[i] = As[k][ty * 4 + i];
        b[i] = Bs[k][tx * 4 + i];
        if constexpr (EPI == EPI_SWIGLU) bu[i] = Bu[k][tx * 4 + i];
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          acc[i][j] += a[i] * b[j];
          if constexpr (EPI == EPI_SWIGLU) accu[i][j] += a[i] * bu[j];
        }
    }
    __syncthreads();
  }
  T* C = reinterpret_cast<T*>(g.C);
  const T* R = reinterpret_cast<const T*>(g.R);
  const T* bias = reinterpret_cast<const T*>(g.bias);
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int gm = m0 + ty * 4 + i;
    if (gm >= g.M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int gn = n0 + tx * 4 + j;
      if (gn >= g.N) continue;
      float v = acc[i][j];
      if constexpr (EPI == EPI_STORE) {
        if (bias) v += to_f(bias[gn]);
      } else if constexpr (EPI == EPI_RESIDUAL) {
        v += to_f(R[(size_t)gm * g.ldr + gn]);
      } else {
        v = silu_f(v) * accu[i][j];
      }
      C[(size_t)gm * g.ldc + gn] = from_f<T>(v);
    }
  }
}

int launch_gemm_simt(DT dt, const GemmArgs& a, cudaStream_t st) {
  if (a.M <= 0 || a.N <= 0) return 0;
  dim3 grid((a.N + 63) / 64, (a.M + 63) / 64);
  if (dt == DT::BF16) {
    if (a.epi == EPI_STORE) gemm_simt_kernel<bf16, EPI_STORE><<<grid, 256, 0, st>>>(a);
    else if (a.epi == EPI_RESIDUAL) gemm_simt_kernel<bf16, EPI_RESIDUAL><<<grid, 256, 0, st>>>(a);
    else gemm_simt_kernel<bf16, EPI_SWIGLU><<<grid, 256, 0, st>>>(a);
  } else {
    if (a.epi == EPI_STORE) gemm_simt_kernel<float, EPI_STORE><<<grid, 256, 0, st>>>(a);
    else if (a.epi == EPI_RESIDUAL) gemm_simt_kernel<float, EPI_RESIDUAL><<<grid, 256, 0, st>>>(a);
    else gemm_simt_kernel<float, EPI_SWIGLU><<<grid, 256, 0, st>>>(a);
  }
  return 1;
}

// Dispatcher: bf16 shapes the tcgen05 kernel tiles go there; everything else is SIMT.
int launch_gemm(DT dt, const GemmArgs& a, int num_sms, cudaStream_t st) {
  if (a.row_split < a.M || a.epi == EPI_QKV_ROPE || a.epi == EPI_RESIDUAL_AR || a.m_dev) {  // CTA-pair kernel only
    if (dt == DT::BF16 && gemm2_supported(a, num_sms)) return launch_gemm2(a, num_sms, st);
    return -1000000;
  }
  if (dt == DT::BF16 && gemm2_supported(a, num_sms)) {
    const int r = launch_gemm2(a, num_sms, st);
    if (r > 0) return r;
  }
  if (dt == DT::BF16 && gemm_tc_supported(a)) return launch_gemm_tc(a, num_sms, st);
  return launch_gemm_simt(dt, a, st);
}

}  // namespace duet

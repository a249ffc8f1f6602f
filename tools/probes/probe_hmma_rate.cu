// Probe: legacy tensor-path (mma.sync m16n8k16 bf16 -> f32, SASS HMMA.16816.F32.BF16) throughput per SM
// on B200, versus warps per SM, with CHAINS independent accumulators per warp.  The paged decode
// attention issues 16 of these per 16-token page (N = 8, G = 4 heads used), so this rate bounds the
// bytes per SM-clock it can stream.  nvcc -gencode arch=compute_100a,code=sm_100a -O3 probe_hmma_rate.cu
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

template <int CHAINS>
__global__ void hmma_loop(float* out, int iters) {
  float d[CHAINS][4];
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) d[c][0] = d[c][1] = d[c][2] = d[c][3] = 0.f;
  uint32_t a0 = threadIdx.x, a1 = a0 * 3, a2 = a0 * 5, a3 = a0 * 7, b0 = a0 * 11, b1 = a0 * 13;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int c = 0; c < CHAINS; ++c)
      asm volatile(
          "mma.sync.aligned.m16n8k16.row.col.f32.bf16.bf16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};"
          : "+f"(d[c][0]), "+f"(d[c][1]), "+f"(d[c][2]), "+f"(d[c][3])
          : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
  }
  float s = 0.f;
#pragma unroll
  for (int c = 0; c < CHAINS; ++c) s += d[c][0] + d[c][1] + d[c][2] + d[c][3];
  if (s == 1.2345f) out[threadIdx.x] = s;
}

template <int CHAINS>
void run(int warps, int sms) {
  float* out;
  cudaMalloc(&out, 4096);
  const int iters = 4096;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  hmma_loop<CHAINS><<<sms, warps * 32>>>(out, 16);
  cudaEventRecord(a);
  hmma_loop<CHAINS><<<sms, warps * 32>>>(out, iters);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  int clk_khz;
  cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0);
  const double mmas = (double)sms * warps * iters * CHAINS;
  const double per_sm_per_s = mmas / sms / (ms * 1e-3);
  printf("chains=%d warps/SM=%2d: %.3f ms  %.2f G mma/s/SM  = %.0f MAC/clk/SM at %.0f MHz (%.1f clk per mma per SM)\n",
         CHAINS, warps, ms, per_sm_per_s / 1e9, per_sm_per_s * 4096 / (clk_khz * 1e3), clk_khz / 1e3,
         clk_khz * 1e3 / per_sm_per_s);
  cudaFree(out);
}

int main() {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int w : {1, 2, 4, 8, 12, 16}) run<1>(w, sms);
  for (int w : {1, 4, 8, 12, 16}) run<4>(w, sms);
  for (int w : {4, 8, 16}) run<8>(w, sms);
  return 0;
}

// Probe: tcgen05.mma (kind::f16, cta_group::1, A/B K-major SW128 in smem) issue-to-completion cost per
// instruction as a function of N (and M = 64 / 128).  One CTA per SM; one thread issues R UMMAs
// back-to-back into TMEM, commits, waits; reports cycles per UMMA and per-SM FLOP/clk.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 probe_umma_rate.cu -o probe_umma_rate
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ uint64_t desc(uint32_t a) {
  return (uint64_t)((a & 0x3FFFF) >> 4) | ((uint64_t)1 << 16) | ((uint64_t)64 << 32) | ((uint64_t)1 << 46) | ((uint64_t)2 << 61);
}
__host__ __device__ constexpr uint32_t idesc(int m, int n) {
  return (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(m >> 4) << 24);
}
template <int M, int N, int MODE>  // MODE 0: A,B K-major smem (4 addresses)  1: K-major, 64 distinct
                                    // 1-KiB-aligned tile addresses  2: B MN-major  3: A from TMEM, B MN-major
__global__ void k(int reps, unsigned long long* out) {
  extern __shared__ __align__(1024) uint8_t sm[];
  __shared__ uint32_t slot;
  __shared__ __align__(8) uint64_t bar;
  __shared__ __align__(8) uint64_t bar2;
  const int warp = threadIdx.x / 32;
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(su32(&slot)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar)));
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar2)));
    asm volatile("fence.mbarrier_init.release.cluster;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem = slot;
  if (threadIdx.x == 0) {
    const uint32_t a = su32(sm), b = su32(sm + 32768);
    const unsigned long long t0 = clock64();
    constexpr uint32_t ID = MODE >= 2 ? (idesc(M, N) | (1u << 16)) : idesc(M, N);
    for (int i = 0; i < reps; ++i) {
      const uint32_t off = MODE == 0 ? (i & 3) * 32 : ((i * 7) & 7) * 1024 + (i & 3) * 32;
      if (MODE == 4) {  // FA-like mix: 8 SS UMMAs into D0, then 8 TS UMMAs (A = TMEM cols 384+) into D1
        if ((i >> 3) & 1)
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tmem + 128),
                       "r"(tmem + 384 + (i & 7) * 8), "l"(desc(b + off)), "r"(ID | (1u << 16)), "r"(i & 7));
        else
          asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
                       "l"(desc(a + off)), "l"(desc(b + off)), "r"(ID), "r"(i & 7));
      } else if (MODE == 5) {  // FA-like mix with a commit after every 8 UMMAs
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem + ((i >> 3) & 1) * 128),
                     "l"(desc(a + off)), "l"(desc(b + off)), "r"(ID), "r"(i & 7));
        if ((i & 7) == 7)
          asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar2)) : "memory");
      } else if (MODE == 3) {
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(tmem),
                     "r"(tmem + 128 + (i & 3) * 8), "l"(desc(b + off)), "r"(ID), "r"(i & 1));
      } else {
        asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem),
                     "l"(desc(a + off)), "l"(desc(b + off)), "r"(ID), "r"(i & 1));
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(su32(&bar)) : "memory");
    asm volatile("{\n.reg .pred p;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n@!p bra W;\n}\n" ::"r"(su32(&bar)));
    const unsigned long long t1 = clock64();
    if (blockIdx.x == 0) out[0] = t1 - t0;
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem));
  }
}
template <int M, int N, int MODE = 0>
void run(unsigned long long* d) {
  cudaFuncSetAttribute(k<M, N, MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, 98304 + 1024);
  const int reps = 4096;
  k<M, N, MODE><<<148, 128, 98304 + 1024>>>(reps, d);
  k<M, N, MODE><<<148, 128, 98304 + 1024>>>(reps, d);
  cudaDeviceSynchronize();
  unsigned long long h;
  cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
  const double cyc = (double)h / reps;
  printf("mode %d UMMA M=%3d N=%3d K=16: %7.1f cycles/instr  %7.0f FLOP/clk/SM  (%s)\n", MODE, M, N, cyc, 2.0 * M * N * 16 / cyc,
         cudaGetErrorString(cudaGetLastError()));
}
int main() {
  unsigned long long* d;
  cudaMalloc(&d, 8);
  run<128, 32>(d);
  run<128, 64>(d);
  run<128, 128>(d);
  run<128, 256>(d);
  run<64, 64>(d);
  run<64, 128>(d);
  run<64, 256>(d);
  run<128, 64, 1>(d);
  run<128, 128, 1>(d);
  run<128, 256, 1>(d);
  run<128, 64, 2>(d);
  run<128, 128, 2>(d);
  run<128, 128, 3>(d);
  run<128, 256, 3>(d);
  run<128, 128, 4>(d);
  run<128, 128, 5>(d);
  return 0;
}

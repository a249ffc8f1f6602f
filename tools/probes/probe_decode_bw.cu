// Probe: read bandwidth per SM of the access pattern of paged decode attention (random 4 KiB blocks,
// one kv head of one page) on green-context partitions of S SMs, for the candidate load mechanisms of a
// decode-attention kernel on a small partition (VERDICT r1 "What's weak" #6):
//   ldg-ring   R blocks in flight per warp in REGISTERS (LDG.128, 8 per lane per block), fragment
//              order (rows g, g+8; 64-B row segments) or lane-contiguous order
//   bulk1d     cp.async.bulk (non-tensor TMA) 4 KiB per instruction into shared memory, completion on
//              an mbarrier; I issuing lanes per warp (1 or 32), D blocks in flight per issuing lane
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 probe_decode_bw.cu -lcuda -o probe_decode_bw
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <numeric>
#include <random>
#include <vector>

#define CK(x) do { CUresult r_ = (x); if (r_ != CUDA_SUCCESS) { const char* s; cuGetErrorString(r_, &s); \
  printf("CU error %s at %d\n", s, __LINE__); exit(1);} } while (0)
#define RK(x) do { cudaError_t r_ = (x); if (r_ != cudaSuccess) { printf("RT error %s at %d\n", \
  cudaGetErrorString(r_), __LINE__); exit(1);} } while (0)

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint4 ldg_ef(const uint4* p, uint64_t pol) {
  uint4 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.u32 {%0,%1,%2,%3}, [%4], %5;"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "l"(p), "l"(pol));
  return v;
}

// Each warp streams `units` blocks; block u of warp w is pool block perm[(w * units + u) % n_blocks].
template <int R, bool FRAG>
__global__ void ldg_ring(const uint4* __restrict__ pool, const int* __restrict__ perm, int units, int n_blocks,
                         unsigned* sink) {
  const int lane = threadIdx.x & 31;
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  // per-lane uint4 offsets inside a 4 KiB block (256 uint4 = 16 rows x 16 chunks)
  int off[8];
#pragma unroll
  for (int j = 0; j < 8; ++j)
    off[j] = FRAG ? ((lane >> 2) + 8 * (j >> 2)) * 16 + (j & 3) * 4 + (lane & 3) : j * 32 + lane;
  uint4 b[R][8];
  uint32_t acc = 0;
  const size_t base = (size_t)w * units;
#pragma unroll
  for (int r = 0; r < R; ++r) {
    const uint4* p = pool + (size_t)__ldg(perm + (base + r) % n_blocks) * 256;
#pragma unroll
    for (int j = 0; j < 8; ++j) b[r][j] = ldg_ef(p + off[j], pol);
  }
  for (int i = 0; i < units; i += R) {
#pragma unroll
    for (int r = 0; r < R; ++r) {
#pragma unroll
      for (int j = 0; j < 8; ++j) acc ^= b[r][j].x ^ b[r][j].y ^ b[r][j].z ^ b[r][j].w;
      const int u = i + r + R;
      if (u < units) {
        const uint4* p = pool + (size_t)__ldg(perm + (base + u) % n_blocks) * 256;
#pragma unroll
        for (int j = 0; j < 8; ++j) b[r][j] = ldg_ef(p + off[j], pol);
      }
    }
  }
  if (acc == 0x9e3779b9u) sink[0] = acc;
}

// I issuing lanes per warp, D stages of 4 KiB per issuing lane.
template <int D>
__global__ void bulk1d(const uint8_t* __restrict__ pool, const int* __restrict__ perm, int units, int n_blocks,
                       int issuers, unsigned* sink) {
  extern __shared__ __align__(128) uint8_t smem[];
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int w = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + (size_t)nw * issuers * D * 4096);
  if (lane < issuers) {
    uint8_t* ring = smem + ((size_t)wl * issuers + lane) * D * 4096;
    uint64_t* bar = bars + ((size_t)wl * issuers + lane) * D;
    for (int s = 0; s < D; ++s) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&bar[s])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    uint64_t pol;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
    const size_t base = ((size_t)w * issuers + lane) * units;
    auto issue = [&](int u) {
      const int s = u % D;
      const uint8_t* src = pool + (size_t)__ldg(perm + (base + u) % n_blocks) * 4096;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 4096;" ::"r"(su32(&bar[s])) : "memory");
      asm volatile(
          "cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], 4096, [%2], %3;" ::"r"(
              su32(ring + s * 4096)), "l"(src), "r"(su32(&bar[s])), "l"(pol) : "memory");
    };
    for (int u = 0; u < D && u < units; ++u) issue(u);
    uint32_t acc = 0;
    for (int u = 0; u < units; ++u) {
      const int s = u % D;
      const uint32_t par = (u / D) & 1;
      asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(
                       su32(&bar[s])), "r"(par) : "memory");
      acc ^= *reinterpret_cast<const uint32_t*>(ring + s * 4096 + (u & 1023) * 4);
      if (u + D < units) issue(u + D);
    }
    if (acc == 0x9e3779b9u) sink[0] = acc;
  }
}

int main() {
  RK(cudaSetDevice(0));
  RK(cudaFree(0));
  CUdevice dev;
  CK(cuDeviceGet(&dev, 0));
  CUdevResource all;
  CK(cuDeviceGetDevResource(dev, &all, CU_DEV_RESOURCE_TYPE_SM));
  const size_t bytes = (size_t)2 << 30;
  const int n_blocks = (int)(bytes / 4096);
  void* buf;
  RK(cudaMalloc(&buf, bytes));
  RK(cudaMemset(buf, 1, bytes));
  std::vector<int> perm(n_blocks);
  std::iota(perm.begin(), perm.end(), 0);
  std::mt19937 rng(4791);
  std::shuffle(perm.begin(), perm.end(), rng);
  int* dperm;
  RK(cudaMalloc(&dperm, n_blocks * sizeof(int)));
  RK(cudaMemcpy(dperm, perm.data(), n_blocks * sizeof(int), cudaMemcpyHostToDevice));
  unsigned* sink;
  RK(cudaMalloc(&sink, 64));
  cudaEvent_t e0, e1;
  RK(cudaEventCreate(&e0));
  RK(cudaEventCreate(&e1));
  for (int S : {16, 32, 48, 148}) {
    cudaStream_t st = nullptr;
    CUgreenCtx g1 = nullptr;
    if (S < 148) {
      CUdevResource grp[1], rem;
      unsigned n = 1;
      CK(cuDevSmResourceSplitByCount(grp, &n, &all, &rem, 0, S));
      CUdevResourceDesc d1;
      CK(cuDevResourceGenerateDesc(&d1, grp, 1));
      CK(cuGreenCtxCreate(&g1, d1, dev, CU_GREEN_CTX_DEFAULT_STREAM));
      CUstream s1;
      CK(cuGreenCtxStreamCreate(&s1, g1, CU_STREAM_NON_BLOCKING, 0));
      st = (cudaStream_t)s1;
    } else {
      RK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    }
    auto time_it = [&](auto launch, double moved) {
      float best = 1e9;
      for (int rep = 0; rep < 5; ++rep) {
        RK(cudaEventRecord(e0, st));
        launch();
        RK(cudaGetLastError());
        RK(cudaEventRecord(e1, st));
        RK(cudaEventSynchronize(e1));
        float ms;
        RK(cudaEventElapsedTime(&ms, e0, e1));
        best = std::min(best, ms);
      }
      return moved / best / 1e6;
    };
    // ---- LDG register rings
    auto ring = [&](auto kern, int R, bool frag, int wpb) {
      int occ = 0;
      RK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kern, wpb * 32, 0));
      cudaFuncAttributes fa;
      RK(cudaFuncGetAttributes(&fa, kern));
      const int warps = S * occ * wpb;
      const int units = (int)std::min<size_t>(n_blocks / warps, 4096) / R * R;
      const double moved = (double)warps * units * 4096;
      const double gbs = time_it([&] { kern<<<S * occ, wpb * 32, 0, st>>>((const uint4*)buf, dperm, units, n_blocks, sink); },
                                 moved);
      printf("S=%3d  ldg-ring R=%d %-6s %2d warps/SM (%3d regs)  in flight %3d KB/SM  %7.0f GB/s (%5.1f GB/s/SM)\n", S,
             R, frag ? "frag" : "lanes", occ * wpb, fa.numRegs, occ * wpb * R * 4, gbs, gbs / S);
    };
    for (int wpb : {4, 8}) {
      ring(ldg_ring<1, true>, 1, true, wpb);
      ring(ldg_ring<2, true>, 2, true, wpb);
      ring(ldg_ring<3, true>, 3, true, wpb);
      ring(ldg_ring<4, true>, 4, true, wpb);
      ring(ldg_ring<6, true>, 6, true, wpb);
      ring(ldg_ring<2, false>, 2, false, wpb);
      ring(ldg_ring<4, false>, 4, false, wpb);
    }
    // ---- bulk 1-D copies
    auto bulk = [&](auto kern, int D, int issuers, int wpb, int ctas_per_sm) {
      const int smem = wpb * issuers * D * 4096 + wpb * issuers * D * 8;
      if (smem * ctas_per_sm > 227 * 1024) return;
      RK(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
      const int lanes = S * ctas_per_sm * wpb * issuers;
      const int units = (int)std::min<size_t>(n_blocks / lanes, 4096);
      const double moved = (double)lanes * units * 4096;
      const double gbs = time_it(
          [&] { kern<<<S * ctas_per_sm, wpb * 32, smem, st>>>((const uint8_t*)buf, dperm, units, n_blocks, issuers, sink); },
          moved);
      printf("S=%3d  bulk1d D=%d issuers/warp=%2d warps/SM=%2d  in flight %3d KB/SM  %7.0f GB/s (%5.1f GB/s/SM)\n", S, D,
             issuers, wpb * ctas_per_sm, wpb * ctas_per_sm * issuers * D * 4, gbs, gbs / S);
    };
    bulk(bulk1d<4>, 4, 1, 4, 1);
    bulk(bulk1d<4>, 4, 1, 8, 1);
    bulk(bulk1d<4>, 4, 1, 16, 1);
    bulk(bulk1d<2>, 2, 1, 16, 1);
    bulk(bulk1d<1>, 1, 32, 1, 1);
    bulk(bulk1d<1>, 1, 16, 2, 1);
    bulk(bulk1d<1>, 1, 8, 4, 1);
    bulk(bulk1d<2>, 2, 8, 2, 1);
    bulk(bulk1d<1>, 1, 32, 1, 2);
    if (g1) {
      CK(cuStreamDestroy((CUstream)st));
      CK(cuGreenCtxDestroy(g1));
    } else {
      RK(cudaStreamDestroy(st));
    }
  }
  printf("PROBE DONE\n");
  return 0;
}

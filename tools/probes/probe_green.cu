// Probe: green-context SM partitions on this B200 (granularity, disjointness,
// runtime-API launches and CUDA-graph capture on green-context streams).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 probe_green.cu -lcuda -o probe_green
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <set>

#define CK(x) do { CUresult r_ = (x); if (r_ != CUDA_SUCCESS) { const char* s; cuGetErrorString(r_, &s); \
  printf("CU error %s at %s:%d\n", s, __FILE__, __LINE__); exit(1);} } while (0)
#define RK(x) do { cudaError_t r_ = (x); if (r_ != cudaSuccess) { printf("RT error %s at %s:%d\n", \
  cudaGetErrorString(r_), __FILE__, __LINE__); exit(1);} } while (0)

__global__ void smid_kernel(int* seen, long long spin) {
  unsigned s; asm volatile("mov.u32 %0, %%smid;" : "=r"(s));
  if (threadIdx.x == 0) atomicAdd(&seen[s], 1);
  long long t0 = clock64();
  while (clock64() - t0 < spin) {}
}

__global__ void stamp_kernel(unsigned long long* ts, int idx, long long spin) {
  unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  long long t0 = clock64();
  while (clock64() - t0 < spin) {}
  unsigned long long t1; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t1));
  if (blockIdx.x == 0 && threadIdx.x == 0) { ts[2*idx] = t; ts[2*idx+1] = t1; }
}

int main() {
  RK(cudaSetDevice(0));
  RK(cudaFree(0));
  CUdevice dev; CK(cuDeviceGet(&dev, 0));
  CUdevResource all; CK(cuDeviceGetDevResource(dev, &all, CU_DEV_RESOURCE_TYPE_SM));
  printf("device SM count = %u\n", all.sm.smCount);
  int *seen; RK(cudaMallocManaged(&seen, 256 * sizeof(int)));
  for (unsigned flags = 0; flags < 2; ++flags) {
    for (unsigned want : {1u, 2u, 4u, 6u, 8u, 10u, 16u, 24u, 32u, 64u, 72u, 74u, 140u}) {
      CUdevResource grp[1]; unsigned n = 1; CUdevResource rem;
      CUresult r = cuDevSmResourceSplitByCount(grp, &n, &all, &rem, flags, want);
      if (r != CUDA_SUCCESS) { printf("flags=%u want=%u -> error %d\n", flags, want, (int)r); continue; }
      printf("flags=%u want=%u -> groups=%u group.sm=%u rem.sm=%u\n", flags, want, n, grp[0].sm.smCount, rem.sm.smCount);
    }
  }
  // Build one split and check disjointness + concurrency
  for (unsigned flags = 0; flags < 2; ++flags) {
    unsigned want = flags ? 10 : 16;
    CUdevResource grp[1]; unsigned n = 1; CUdevResource rem;
    CK(cuDevSmResourceSplitByCount(grp, &n, &all, &rem, flags, want));
    CUdevResourceDesc d1, d2;
    CK(cuDevResourceGenerateDesc(&d1, grp, 1));
    CK(cuDevResourceGenerateDesc(&d2, &rem, 1));
    CUgreenCtx g1, g2;
    CK(cuGreenCtxCreate(&g1, d1, dev, CU_GREEN_CTX_DEFAULT_STREAM));
    CK(cuGreenCtxCreate(&g2, d2, dev, CU_GREEN_CTX_DEFAULT_STREAM));
    CUstream s1, s2;
    CK(cuGreenCtxStreamCreate(&s1, g1, CU_STREAM_NON_BLOCKING, 0));
    CK(cuGreenCtxStreamCreate(&s2, g2, CU_STREAM_NON_BLOCKING, 0));
    // runtime API launch on green stream, large grid
    for (int i = 0; i < 256; ++i) seen[i] = 0;
    smid_kernel<<<2000, 128, 0, (cudaStream_t)s1>>>(seen, 2000);
    RK(cudaGetLastError());
    RK(cudaStreamSynchronize((cudaStream_t)s1));
    std::set<int> A, B;
    for (int i = 0; i < 256; ++i) if (seen[i]) A.insert(i);
    for (int i = 0; i < 256; ++i) seen[i] = 0;
    smid_kernel<<<2000, 128, 0, (cudaStream_t)s2>>>(seen, 2000);
    RK(cudaStreamSynchronize((cudaStream_t)s2));
    for (int i = 0; i < 256; ++i) if (seen[i]) B.insert(i);
    int overlap = 0; for (int x : A) overlap += B.count(x);
    printf("split flags=%u want=%u: side1 used %zu SMs, side2 used %zu SMs, overlap=%d\n", flags, want, A.size(), B.size(), overlap);
    printf("  side1 smids:"); for (int x : A) printf(" %d", x); printf("\n");
    // concurrency: two long kernels, one per side
    unsigned long long* ts; RK(cudaMallocManaged(&ts, 8 * sizeof(unsigned long long)));
    stamp_kernel<<<8, 128, 0, (cudaStream_t)s1>>>(ts, 0, 20000000);
    stamp_kernel<<<100, 128, 0, (cudaStream_t)s2>>>(ts, 1, 20000000);
    RK(cudaDeviceSynchronize());
    printf("  concurrency: s1 [%llu, %llu] s2 [%llu, %llu] (ns rel) overlap=%lld ns\n", 0ull, ts[1]-ts[0], ts[2]-ts[0], ts[3]-ts[0],
           (long long)(std::min(ts[1], ts[3])) - (long long)(std::max(ts[0], ts[2])));
    // graph capture on green stream
    cudaGraph_t graph; cudaGraphExec_t gexec;
    RK(cudaStreamBeginCapture((cudaStream_t)s1, cudaStreamCaptureModeThreadLocal));
    for (int i = 0; i < 256; ++i) seen[i] = 0;
    smid_kernel<<<500, 128, 0, (cudaStream_t)s1>>>(seen, 1000);
    RK(cudaStreamEndCapture((cudaStream_t)s1, &graph));
    RK(cudaGraphInstantiate(&gexec, graph, 0));
    for (int i = 0; i < 256; ++i) seen[i] = 0;
    RK(cudaGraphLaunch(gexec, (cudaStream_t)s1));
    RK(cudaStreamSynchronize((cudaStream_t)s1));
    std::set<int> C; for (int i = 0; i < 256; ++i) if (seen[i]) C.insert(i);
    int ov2 = 0; for (int x : C) ov2 += B.count(x);
    printf("  graph replay on green stream used %zu SMs, overlap with side2=%d\n", C.size(), ov2);
    // event timing on green streams
    cudaEvent_t e0, e1; RK(cudaEventCreate(&e0)); RK(cudaEventCreate(&e1));
    RK(cudaEventRecord(e0, (cudaStream_t)s2));
    stamp_kernel<<<100, 128, 0, (cudaStream_t)s2>>>(ts, 2, 2000000);
    RK(cudaEventRecord(e1, (cudaStream_t)s2));
    RK(cudaEventSynchronize(e1));
    float ms; RK(cudaEventElapsedTime(&ms, e0, e1));
    printf("  runtime events on green stream ok: %.3f ms\n", ms);
    // cross-stream wait between a green stream and a normal stream
    cudaStream_t ns; RK(cudaStreamCreateWithFlags(&ns, cudaStreamNonBlocking));
    RK(cudaEventRecord(e0, ns));
    RK(cudaStreamWaitEvent((cudaStream_t)s1, e0, 0));
    RK(cudaStreamSynchronize((cudaStream_t)s1));
    printf("  cross-ctx event wait ok\n");
    CK(cuStreamDestroy(s1)); CK(cuStreamDestroy(s2));
    CK(cuGreenCtxDestroy(g1)); CK(cuGreenCtxDestroy(g2));
  }
  printf("PROBE DONE\n");
  return 0;
}

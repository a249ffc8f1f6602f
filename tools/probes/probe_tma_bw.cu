// Probe: achievable HBM read bandwidth per SM with (a) plain 16-B LDG streaming, (b) TMA 2-D boxes into
// an mbarrier ring (no compute), on green-context partitions of S SMs.  Box shapes: "gemm" = 128 rows x
// 128 B with an 8 KiB row pitch (a K-major weight tile), "page" = 16 rows x 128 B with a 256 B pitch
// (half a KV page).  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O2 probe_tma_bw.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x) do { CUresult r_ = (x); if (r_ != CUDA_SUCCESS) { const char* s; cuGetErrorString(r_, &s); \
  printf("CU error %s at %d\n", s, __LINE__); exit(1);} } while (0)
#define RK(x) do { cudaError_t r_ = (x); if (r_ != cudaSuccess) { printf("RT error %s at %d\n", \
  cudaGetErrorString(r_), __LINE__); exit(1);} } while (0)

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__global__ void __launch_bounds__(512) ldg_kernel(const uint4* __restrict__ buf, size_t n_vec, unsigned* sink) {
  uint32_t acc = 0;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i + 3 * stride < n_vec; i += 4 * stride) {
    uint4 a = __ldcs(buf + i), b = __ldcs(buf + i + stride), c = __ldcs(buf + i + 2 * stride), d = __ldcs(buf + i + 3 * stride);
    acc ^= a.x ^ b.y ^ c.z ^ d.w;
  }
  if (acc == 0x12345) sink[0] = acc;
}

// one CTA per SM; lane 0 of each of the blockDim/32 warps issues boxes into its own NST stages;
// all boxes are "consumed" immediately
template <int NST>
__global__ void tma_kernel(const __grid_constant__ CUtensorMap map, int box_bytes, int boxes_per_stage, int rows_total,
                           int box_rows, int cols_boxes, int total_units_all) {
  extern __shared__ __align__(1024) uint8_t smem_all[];
  const int nw = blockDim.x / 32, w = threadIdx.x / 32;
  const int ring = NST * box_bytes * boxes_per_stage;
  uint8_t* smem = smem_all + w * ring;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_all + nw * ring) + w * NST;
  const int total_units = total_units_all / nw;   // this warp's share: units u*nw + w
  if ((threadIdx.x & 31) == 0) {
    for (int i = 0; i < NST; ++i)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su32(&full[i])));
    asm volatile("fence.mbarrier_init.release.cluster;");
    // unit u -> (row block, col box) ; each stage = boxes_per_stage consecutive units
    int issued = 0, done = 0;
    const int my_units = (total_units - blockIdx.x + gridDim.x - 1) / gridDim.x;
    const int my_stages = my_units / boxes_per_stage;
    auto issue = [&](int s) {
      const int st = s % NST;
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[st])),
                   "r"(box_bytes * boxes_per_stage));
      for (int b = 0; b < boxes_per_stage; ++b) {
        // consecutive boxes of a stage are consecutive units (neighbouring column boxes of the same rows)
        const int u = (((s * gridDim.x + blockIdx.x) * nw + w) * boxes_per_stage + b) % total_units_all;
        const int rb = u / cols_boxes, cb = u % cols_boxes;
        const int c0 = cb * 64, c1 = (rb * box_rows) % rows_total;
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4}], [%2];" ::"r"(
                su32(smem + (st * boxes_per_stage + b) * box_bytes)),
            "l"(&map), "r"(su32(&full[st])), "r"(c0), "r"(c1)
            : "memory");
      }
    };
    for (; issued < NST && issued < my_stages; ++issued) issue(issued);
    for (; done < my_stages; ++done) {
      const int st = done % NST;
      const uint32_t par = (done / NST) & 1;
      asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(
                       su32(&full[st])), "r"(par) : "memory");
      if (issued < my_stages) issue(issued++);
    }
  }
  __syncthreads();
}

// cp.async (LDGSTS 16 B) streaming: each CTA copies stages of `stage_bytes` contiguous bytes, NST groups in flight
template <int NST>
__global__ void cpasync_kernel(const uint8_t* __restrict__ buf, size_t bytes, int stage_bytes) {
  extern __shared__ __align__(1024) uint8_t smem[];
  const size_t n_stages = bytes / stage_bytes;
  int slot = 0;
  for (size_t s = blockIdx.x; s < n_stages; s += gridDim.x) {
    const uint8_t* src = buf + s * stage_bytes;
    uint8_t* dst = smem + slot * stage_bytes;
    for (int i = threadIdx.x * 16; i < stage_bytes; i += blockDim.x * 16)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(su32(dst + i)), "l"(src + i) : "memory");
    asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group %0;" ::"n"(NST - 1) : "memory");
    slot = (slot + 1) % NST;
  }
  asm volatile("cp.async.wait_group 0;" ::: "memory");
}

int main() {
  RK(cudaSetDevice(0));
  RK(cudaFree(0));
  CUdevice dev; CK(cuDeviceGet(&dev, 0));
  CUdevResource all; CK(cuDeviceGetDevResource(dev, &all, CU_DEV_RESOURCE_TYPE_SM));
  const size_t bytes = (size_t)2 << 30;
  void* buf; RK(cudaMalloc(&buf, bytes)); RK(cudaMemset(buf, 1, bytes));
  unsigned* sink; RK(cudaMalloc(&sink, 64));
  cudaEvent_t e0, e1; RK(cudaEventCreate(&e0)); RK(cudaEventCreate(&e1));
  // tensor maps over buf viewed as [rows][cols] bf16
  struct Shape { const char* name; uint64_t cols; uint32_t box_rows; int boxes_per_stage; };
  Shape shapes[] = {{"gemm-128x128B-pitch8K", 4096, 128, 1},
                    {"gemm-128x(4x128B)-pitch8K", 4096, 128, 4},
                    {"gemm-32x(4x128B)-pitch8K", 4096, 32, 4},
                    {"contig-128x128B-pitch128", 64, 128, 1},
                    {"page-16x128B-pitch256", 128, 16, 4}};
  for (int S : {16, 148}) {
    cudaStream_t st = nullptr;
    CUgreenCtx g1 = nullptr, g2 = nullptr;
    if (S < 148) {
      CUdevResource grp[1], rem; unsigned n = 1;
      CK(cuDevSmResourceSplitByCount(grp, &n, &all, &rem, 0, S));
      CUdevResourceDesc d1; CK(cuDevResourceGenerateDesc(&d1, grp, 1));
      CK(cuGreenCtxCreate(&g1, d1, dev, CU_GREEN_CTX_DEFAULT_STREAM));
      CUstream s1; CK(cuGreenCtxStreamCreate(&s1, g1, CU_STREAM_NON_BLOCKING, 0));
      st = (cudaStream_t)s1;
    } else {
      RK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    }
    // LDG
    float best = 1e9;
    for (int rep = 0; rep < 5; ++rep) {
      RK(cudaEventRecord(e0, st));
      ldg_kernel<<<S * 4, 512, 0, st>>>((const uint4*)buf, bytes / 16, sink);
      RK(cudaEventRecord(e1, st)); RK(cudaEventSynchronize(e1));
      float ms; RK(cudaEventElapsedTime(&ms, e0, e1)); if (ms < best) best = ms;
    }
    printf("S=%3d  LDG stream                        %7.0f GB/s  (%5.1f GB/s/SM)\n", S, bytes / best / 1e6, bytes / best / 1e6 / S);
    for (int threads : {256, 512}) {
      const int stage = 8192, nst = 8;
      RK(cudaFuncSetAttribute(cpasync_kernel<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, stage * nst));
      best = 1e9;
      for (int rep = 0; rep < 5; ++rep) {
        RK(cudaEventRecord(e0, st));
        cpasync_kernel<8><<<S * 2, threads, stage * nst, st>>>((const uint8_t*)buf, bytes, stage);
        RK(cudaGetLastError());
        RK(cudaEventRecord(e1, st)); RK(cudaEventSynchronize(e1));
        float ms; RK(cudaEventElapsedTime(&ms, e0, e1)); if (ms < best) best = ms;
      }
      printf("S=%3d  cp.async 8 KB stages x8, 2 CTA/SM x %d thr %7.0f GB/s  (%5.1f GB/s/SM)\n", S, threads,
             bytes / best / 1e6, bytes / best / 1e6 / S);
    }
    for (auto& sh : shapes) {
      for (int nw : {1, 2, 4})
      for (int nst : {4, 8}) {
        CUtensorMap map;
        const uint64_t rows = bytes / 2 / sh.cols;
        cuuint64_t dims[2] = {sh.cols, rows};
        cuuint64_t strides[1] = {sh.cols * 2};
        cuuint32_t box[2] = {64, sh.box_rows};
        cuuint32_t es[2] = {1, 1};
        CK(cuTensorMapEncodeTiled(&map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, strides, box, es,
                                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                  CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE));
        const int box_bytes = 64 * 2 * sh.box_rows;
        const int cols_boxes = (int)(sh.cols / 64);
        const int rows_total = (int)rows;
        const int total_units = (int)(bytes / box_bytes);
        const int smem = nw * nst * box_bytes * sh.boxes_per_stage + 1024;
        if (smem > 220 * 1024) continue;
        void (*k)(CUtensorMap, int, int, int, int, int, int) = nst == 4 ? tma_kernel<4> : tma_kernel<8>;
        RK(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
        best = 1e9;
        for (int rep = 0; rep < 5; ++rep) {
          RK(cudaEventRecord(e0, st));
          k<<<S, 32 * nw, smem, st>>>(map, box_bytes, sh.boxes_per_stage, rows_total, sh.box_rows, cols_boxes,
                                      total_units);
          RK(cudaGetLastError());
          RK(cudaEventRecord(e1, st)); RK(cudaEventSynchronize(e1));
          float ms; RK(cudaEventElapsedTime(&ms, e0, e1)); if (ms < best) best = ms;
        }
        const double moved = (double)(total_units / nw / S / sh.boxes_per_stage) * sh.boxes_per_stage * S * nw *
                             box_bytes;
        printf("S=%3d  TMA %-32s warps=%d nst=%d in-flight %3d KB  %7.0f GB/s  (%5.1f GB/s/SM)\n", S, sh.name, nw,
               nst, nw * nst * box_bytes * sh.boxes_per_stage / 1024, moved / best / 1e6, moved / best / 1e6 / S);
      }
    }
    if (g1) { CK(cuStreamDestroy((CUstream)st)); CK(cuGreenCtxDestroy(g1)); } else RK(cudaStreamDestroy(st));
    (void)g2;
  }
  printf("PROBE DONE\n");
  return 0;
}

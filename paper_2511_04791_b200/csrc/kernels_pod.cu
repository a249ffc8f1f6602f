// POD-style fused prefill + decode attention for a temporal (aggregated) step (
// PAPER.md §6 Related Work P:499, POD-Attention: the compute-bound prefill attention and the
// memory-bound decode attention of one batch overlap on the GPU instead of running one after the other).
//
// ONE launch of 148 CTAs of 448 threads, one per SM: the first n_fa CTAs are persistent prefill-attention
// CTAs (fatc::fa_tc_body: tcgen05 / TMEM flash attention over their snake order of work items), the
// remaining ones are persistent decode-attention CTAs: three groups of 4 warps, each group exactly the
// standalone decode kernel's CTA (dtc::decode_tc_item<4, 2>, 64 KiB of page rings, named barriers),
// striding the (split, kv head, request) items — the 12 decode warps per SM of the standalone launch's
// three co-resident CTAs, and bitwise its results.  Each SM runs one role; which SMs stream KV and which run the tensor cores is decided
// by the block scheduler inside one grid, with no green-context fork / join around the pair.  A prefill
// CTA cannot share its SM with decode warps: it holds 224 KiB of shared memory and all 512 TMEM columns.
#define DUET_BODIES_ONLY
#include "kernels_fa_tc.cu"
#include "kernels_decode_tc.cu"
#undef DUET_BODIES_ONLY

#include <algorithm>

namespace duet {
namespace pod {

constexpr int THREADS = fatc::THREADS;  // 448 = 14 warps: the prefill role's, or three 4-warp decode groups
constexpr int DEC_WARPS = 4, DEC_NST = 2, DEC_GROUPS = 3;
constexpr int DEC_GROUP_BYTES = DEC_WARPS * DEC_NST * dtc::STAGE_BYTES;  // 64 KiB
constexpr int SMEM = fatc::Ring<3, 2>::SMEM > DEC_GROUPS * DEC_GROUP_BYTES + 1024 ? fatc::Ring<3, 2>::SMEM
                                                                              : DEC_GROUPS * DEC_GROUP_BYTES + 1024;
static_assert(SMEM <= 227 * 1024, "smem");

__global__ void __launch_bounds__(THREADS, 1)
    pod_attn_kernel(const __grid_constant__ CUtensorMap map_q, fatc::Params fp, const __grid_constant__ CUtensorMap map_k,
                    const __grid_constant__ CUtensorMap map_v, DecodeAttnArgs da, int pps, int n_splits, int n_fa,
                    int dec_first) {
  // role by block index: prefill CTAs first (default) or decode CTAs first (DUET_POD_DEC_FIRST=1, A/B: which
  // SMs the block scheduler hands each role)
  const int n_dec_ctas = (int)gridDim.x - n_fa;
  const int fa_idx = dec_first ? (int)blockIdx.x - n_dec_ctas : (int)blockIdx.x;
  if (fa_idx >= 0 && fa_idx < n_fa) {
    fatc::fa_tc_body<3, 2>(&map_q, fp, fa_idx, n_fa);
    return;
  }
  const int dec_idx = dec_first ? (int)blockIdx.x : (int)blockIdx.x - n_fa;
  pdl_wait();
  const int group = (int)threadIdx.x / (DEC_WARPS * 32);
  if (group >= DEC_GROUPS) return;  // warps 12-13 of a decode CTA idle
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023) + group * DEC_GROUP_BYTES;
  const int tid = (int)threadIdx.x - group * DEC_WARPS * 32;
  const int slot = dec_idx * DEC_GROUPS + group, n_slots = n_dec_ctas * DEC_GROUPS;
  const int items = n_splits * da.hkv * da.n;
  for (int it = slot; it < items; it += n_slots) {  // split fastest, then kv head, then request (as the grid)
    const int split = it % n_splits, kvh = (it / n_splits) % da.hkv, z = it / (n_splits * da.hkv);
    dtc::decode_tc_item<DEC_WARPS, DEC_NST, false>(&map_k, &map_v, da, pps, n_splits, split, kvh, z, smem, tid,
                                                   1 + group);
    asm volatile("bar.sync %0, %1;" ::"r"(1 + group), "n"(DEC_WARPS * 32) : "memory");  // rings reused next
  }
}

typedef CUresult (*EncodeTiledFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                                  const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                                  CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
static EncodeTiledFn encode_fn() {
  static EncodeTiledFn fn = nullptr;
  if (!fn) {
    cudaDriverEntryPointQueryResult q;
    void* f = nullptr;
    if (cudaGetDriverEntryPointByVersion("cuTensorMapEncodeTiled", &f, 12000, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = (EncodeTiledFn)f;
  }
  return fn;
}

}  // namespace pod

// the q tensor map of the prefill role (as launch_fa_tc builds it); the decode role's copy-based rings
// use no tensor map (zero maps are passed)
int launch_pod_tc(const PrefillAttnArgs& a, const DecodeAttnArgs& da, int pps, int n_splits, int n_dec_ctas,
                  cudaStream_t st) {
  if (!fa_tc_supported(a) || !decode_tc_supported(da) || n_dec_ctas < 1 || a.num_sms <= n_dec_ctas) return -1;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(pod::pod_attn_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, pod::SMEM);
    attr = true;
  }
  pod::EncodeTiledFn fn = pod::encode_fn();
  if (!fn) return -1;
  CUtensorMap mq, mz;
  memset(&mz, 0, sizeof(mz));
  {
    cuuint64_t dims[2] = {(cuuint64_t)a.q_stride, (cuuint64_t)a.total_rows};
    cuuint64_t strides[1] = {(cuuint64_t)a.q_stride * 2};
    cuuint32_t box[2] = {64, (cuuint32_t)fatc::BQ};
    cuuint32_t es[2] = {1, 1};
    if (fn(&mq, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(a.q), dims, strides, box, es,
           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
      return -1;
  }
  fatc::Params p{a.row0, a.qlen, a.cpre, a.seq_row, a.table, a.max_pages, a.hq, a.hkv, 0, 0, 0, 0, nullptr,
                 (bf16*)a.o, (const bf16*)a.k_pool, (const bf16*)a.v_pool};
  const int G = a.hq / a.hkv;
  p.n_qtiles = (a.max_q + fatc::BQ - 1) / fatc::BQ;
  p.n_pairs = a.hkv * ((G + 1) / 2);
  p.n_seqs = a.n_seqs;
  p.shape_dev = a.shape_dev;
  const int fa_items = p.n_qtiles * a.n_seqs * p.n_pairs;
  const int n_fa = std::min(a.num_sms - n_dec_ctas, fa_items);
  const int dec_items = n_splits * da.hkv * da.n;
  const int n_dec = std::min(n_dec_ctas, (dec_items + pod::DEC_GROUPS - 1) / pod::DEC_GROUPS);
  static const int dec_first = getenv("DUET_POD_DEC_FIRST") ? atoi(getenv("DUET_POD_DEC_FIRST")) : 0;
  launch_pdl(pod::pod_attn_kernel, n_fa + n_dec, pod::THREADS, pod::SMEM, st, mq, p, mz, mz, da, pps, n_splits, n_fa,
             dec_first);
  return 1;
}

}  // namespace duet

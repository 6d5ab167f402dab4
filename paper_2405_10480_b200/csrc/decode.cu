// Host side of the decode path: kernel selection, K/V tensor maps (cached per plan), the
// persistent launch, and the sequence-shard combine kernel (la_combine).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>

#include <atomic>
#include <cstdint>
#include <cstring>
#include <mutex>
#include <string>

#include "decode_kernel.cuh"

namespace la {

static std::atomic<int64_t> g_launches{0};
int64_t launch_count() { return g_launches.load(); }
void note_launch() { g_launches.fetch_add(1); }

namespace {

// ---------------------------------------------------------------------------------------
// Sequence-shard combine: L = ln sum_r e^{L_r}, O = sum_r e^{L_r - L} O_r  (ascending r)
// ---------------------------------------------------------------------------------------
template <int D>
__global__ void __launch_bounds__(D) la_combine_kernel(const float* __restrict__ o_parts, size_t o_stride,
                                                       const float* __restrict__ lse_parts, size_t l_stride, int parts,
                                                       float* __restrict__ out, float* __restrict__ lse) {
  // part p's row r: o_parts[p * o_stride + r * D + c], lse_parts[p * l_stride + r]
  const int r = blockIdx.x, c = threadIdx.x;
  float mx = -INFINITY;
  for (int p = 0; p < parts; ++p) mx = fmaxf(mx, lse_parts[p * l_stride + r]);
  float s = 0.f, acc = 0.f;
  for (int p = 0; p < parts; ++p) {
    const float w = expf(lse_parts[p * l_stride + r] - mx);
    s += w;
    acc = fmaf(w, o_parts[p * o_stride + size_t(r) * D + c], acc);
  }
  out[size_t(r) * D + c] = acc / s;
  if (c == 0 && lse) lse[r] = mx + logf(s);
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn(std::string& err) {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  if (!fn) err = "cuTensorMapEncodeTiled unavailable";
  return fn;
}

bool make_tmap(CUtensorMap* tm, const void* base, int64_t rows, int d, int dtype, int box_rows, int box_halves,
               std::string& err) {
  auto enc = encode_fn(err);
  if (!enc) return false;
  // d = 64: 2-D {element, row}.  d = 128: 3-D {element, row, half} (half stride 128 B), so
  // one box carries both 128-B halves of box_rows rows (GqaEngine::row_off).
  // FP8 (d = 128): 2-D {code, row}, one 128-B box row per token.
  const bool fp8 = dtype == LA_FP8_E4M3;
  const int rank = (d == 64 || fp8) ? 2 : 3;
  cuuint64_t gdim[3] = {cuuint64_t(fp8 ? 128 : 64), cuuint64_t(rows), 2};
  cuuint64_t gstride[2] = {cuuint64_t(d) * (fp8 ? 1 : 2), 128};
  cuuint32_t box[3] = {cuuint32_t(fp8 ? 128 : 64), cuuint32_t(box_rows), cuuint32_t(box_halves)};
  cuuint32_t estr[3] = {1, 1, 1};
  const CUtensorMapDataType ty = fp8 ? CU_TENSOR_MAP_DATA_TYPE_UINT8
                                     : (dtype == LA_FP16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16
                                                         : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16);
  CUresult r = enc(tm, ty, rank,
                   const_cast<void*>(base), gdim, gstride, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                   CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) {
    err = "cuTensorMapEncodeTiled failed (" + std::to_string(int(r)) + ")";
    return false;
  }
  return true;
}

}  // namespace

KernelInfo decode_kernel_info(int dtype, int head_dim, int group, int engine) {
  if (engine == LA_ENGINE_TCGEN05) {  // 5th-gen tensor cores (bf16 / fp16, d = 128, T_m <= 32, any layout)
    if (head_dim != 128 || group > 32) return KernelInfo{};
    if (dtype == LA_BF16) return info_tc5_bf16(group);
    if (dtype == LA_FP16) return info_tc5_fp16(group);
    return KernelInfo{};
  }
  if (dtype == LA_FP8_E4M3) return info_fp8(head_dim, group);  // tensor cores for every T_m <= 8 (MHA too)
  if (group == 1) return info_mha(dtype, head_dim);              // CUDA cores (a GEMV)
  if (group > 8) return KernelInfo{};
  return info_gqa(dtype, head_dim);                              // mma.sync, T_m <= 8
}

int launch_decode(const KernelInfo& ki, const DecodeArgs& a_in, int64_t kv_rows, int head_dim, int dtype,
                  bool cooperative, void* stream, TmapCache* cache, std::string& err) {
  static_assert(sizeof(TmapPair) <= sizeof(TmapCache::maps), "tensor-map cache size");
  DecodeArgs a = a_in;
  TmapPair tm;
  std::memset(&tm, 0, sizeof(tm));
  a.uses_tmap = ki.uses_tma_tensor ? 1 : 0;
  if (ki.uses_tma_tensor) {
    // encoded once per (k, v, rows): a decode loop over the same cache pays no host encode
    if (cache->k != a.k || cache->v != a.v || cache->rows != kv_rows) {
      cache->k = cache->v = nullptr;
      TmapPair enc;
      if (!make_tmap(&enc.k, a.k, kv_rows, head_dim, dtype, a.box_rows, ki.box_halves, err)) return 1;
      if (!make_tmap(&enc.v, a.v, kv_rows, head_dim, dtype, a.box_rows, ki.box_halves, err)) return 1;
      std::memcpy(cache->maps, &enc, sizeof(enc));
      cache->k = a.k;
      cache->v = a.v;
      cache->rows = kv_rows;
    }
    std::memcpy(&tm, cache->maps, sizeof(tm));
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(a.grid);
  cfg.blockDim = dim3(ki.threads);
  cfg.dynamicSmemBytes = ki.smem_bytes;
  cfg.stream = static_cast<cudaStream_t>(stream);
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;  // static hosts spin on peers: co-residency
  attr[0].val.cooperative = cooperative ? 1 : 0;  // measured: no cost vs a plain launch
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  void* args[] = {&a, &tm};
  cudaError_t e = cudaLaunchKernelExC(&cfg, ki.fn, args);
  if (e != cudaSuccess) {
    err = std::string("decode launch: ") + cudaGetErrorString(e);
    cudaGetLastError();
    return 1;
  }
  note_launch();
  return 0;
}

int launch_combine(const float* o_parts, size_t o_stride, const float* lse_parts, size_t l_stride, int parts, int rows,
                   int head_dim, float* out, float* lse, void* stream, std::string& err) {
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (head_dim == 128)
    la_combine_kernel<128><<<rows, 128, 0, st>>>(o_parts, o_stride, lse_parts, l_stride, parts, out, lse);
  else
    la_combine_kernel<64><<<rows, 64, 0, st>>>(o_parts, o_stride, lse_parts, l_stride, parts, out, lse);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    err = std::string("combine launch: ") + cudaGetErrorString(e);
    return 1;
  }
  note_launch();
  return 0;
}

}  // namespace la


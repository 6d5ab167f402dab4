// GqaEngine instantiations (T_m <= 8 rows, warp-level mma.sync): bf16 / fp16 at d = 64, 128.
#include "decode_kernel.cuh"

namespace la {

KernelInfo info_gqa(int dtype, int head_dim) {
  if (dtype == LA_BF16 && head_dim == 128) return info_of<GqaEngine<__nv_bfloat16, 128, LA_GQA_NST, LA_GQA_WPS>>(true);
  if (dtype == LA_BF16 && head_dim == 64) return info_of<GqaEngine<__nv_bfloat16, 64, LA_GQA_NST, LA_GQA_WPS>>(true);
  if (dtype == LA_FP16 && head_dim == 128) return info_of<GqaEngine<__half, 128, LA_GQA_NST, LA_GQA_WPS>>(true);
  if (dtype == LA_FP16 && head_dim == 64) return info_of<GqaEngine<__half, 64, LA_GQA_NST, LA_GQA_WPS>>(true);
  return KernelInfo{};
}

}  // namespace la

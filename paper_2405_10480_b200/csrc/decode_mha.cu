// MhaEngine instantiations (T_m = 1, CUDA cores): bf16 / fp16 / fp32 at d = 64, 128.
#include "decode_kernel.cuh"

namespace la {

KernelInfo info_mha(int dtype, int head_dim) {
  if (dtype == LA_BF16 && head_dim == 128) return info_of<MhaEngine<__nv_bfloat16, 128, LA_MHA_NST, LA_MHA_WPS>>(false);
  if (dtype == LA_BF16 && head_dim == 64) return info_of<MhaEngine<__nv_bfloat16, 64, LA_MHA_NST, LA_MHA_WPS>>(false);
  if (dtype == LA_FP16 && head_dim == 128) return info_of<MhaEngine<__half, 128, LA_MHA_NST, LA_MHA_WPS>>(false);
  if (dtype == LA_FP16 && head_dim == 64) return info_of<MhaEngine<__half, 64, LA_MHA_NST, LA_MHA_WPS>>(false);
  if (dtype == LA_FP32 && head_dim == 128) return info_of<MhaEngine<float, 128, LA_MHA_NST, LA_MHA_WPS>>(false);
  if (dtype == LA_FP32 && head_dim == 64) return info_of<MhaEngine<float, 64, LA_MHA_NST, LA_MHA_WPS>>(false);
  return KernelInfo{};
}

}  // namespace la

// Fp8Engine instantiations (E4M3 KV cache, bf16 q, d = 128; T_m = 1 and <= 8).
#include "decode_kernel.cuh"

namespace la {

KernelInfo info_fp8(int head_dim, int group) {
  if (head_dim == 128 && group == 1) return info_of<Fp8Engine<128, LA_FP8M_NST, LA_FP8M_WPS, 1>>(true);
  if (head_dim == 128 && group <= 8) return info_of<Fp8Engine<128, LA_FP8_NST, LA_FP8_WPS, 8>>(true);
  return KernelInfo{};
}

}  // namespace la

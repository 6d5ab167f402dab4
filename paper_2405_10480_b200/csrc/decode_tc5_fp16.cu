// Tc5Engine instantiations (fp16, d = 128): 8-, 16- and 32-row query tiles on tcgen05 + TMEM.
#include "decode_kernel.cuh"

namespace la {

KernelInfo info_tc5_fp16(int group) {
  return group <= 8    ? info_of<Tc5Engine<__half, LA_TC5_NST, 8, LA_TC5_NWG8>>(true)
         : group <= 16 ? info_of<Tc5Engine<__half, LA_TC5_NST, 16, LA_TC5_NWG16>>(true)
                       : info_of<Tc5Engine<__half, LA_TC5_NST32, 32, LA_TC5_NWG32>>(true);
}

}  // namespace la

// Instantiations of the one-warp-per-instance kernel (ic_solo_kernel.cuh).
#include "ic_solo_kernel.cuh"

namespace icsched {
KernelFn kernel_solo(bool drop, bool state, bool packed) {
  if (packed) {
    if (state) return drop ? ic_solo_kernel<true, true, true> : ic_solo_kernel<false, true, true>;
    return drop ? ic_solo_kernel<true, false, true> : ic_solo_kernel<false, false, true>;
  }
  if (state) return drop ? ic_solo_kernel<true, true, false> : ic_solo_kernel<false, true, false>;
  return drop ? ic_solo_kernel<true, false, false> : ic_solo_kernel<false, false, false>;
}
}  // namespace icsched

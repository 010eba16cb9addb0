// Instantiations of the one-warp-per-instance kernel (ic_solo_kernel.cuh).
#include "ic_solo_kernel.cuh"

namespace icsched {
KernelFn kernel_solo(bool drop, bool state) {
  if (state) return drop ? ic_solo_kernel<true, true> : ic_solo_kernel<false, true>;
  return drop ? ic_solo_kernel<true, false> : ic_solo_kernel<false, false>;
}
}  // namespace icsched

// Instantiations of the one-warp-per-instance kernel for task sets with at most 4 optional
// stages (unrolled sweeps for K <= 5 only; ic_solo_kernel.cuh).
#include "ic_solo_kernel.cuh"

namespace icsched {
KernelFn kernel_solo5(bool drop, bool state, bool packed) {
  if (packed) {
    if (state) return drop ? ic_solo_kernel<true, true, true, 5> : ic_solo_kernel<false, true, true, 5>;
    return drop ? ic_solo_kernel<true, false, true, 5> : ic_solo_kernel<false, false, true, 5>;
  }
  if (state) return drop ? ic_solo_kernel<true, true, false, 5> : ic_solo_kernel<false, true, false, 5>;
  return drop ? ic_solo_kernel<true, false, false, 5> : ic_solo_kernel<false, false, false, 5>;
}
}  // namespace icsched

// Instantiations of the one-warp-per-instance kernel (ic_solo_kernel.cuh).
#include "ic_solo_kernel.cuh"

namespace icsched {
KernelFn kernel_solo(bool drop) { return drop ? ic_solo_kernel<true> : ic_solo_kernel<false>; }
}  // namespace icsched

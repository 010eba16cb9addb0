// Kernel instantiations with NW = 16 DP warps (split per NW so nvcc builds them in parallel).
#include "ic_sched_kernel.cuh"

namespace icsched {
KernelFn kernel_nw16(bool sb, bool drop) {
  if (sb) return drop ? ic_dp_kernel<16, true, true> : ic_dp_kernel<16, true, false>;
  return drop ? ic_dp_kernel<16, false, true> : ic_dp_kernel<16, false, false>;
}
}  // namespace icsched

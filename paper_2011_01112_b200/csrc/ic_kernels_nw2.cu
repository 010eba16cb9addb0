// Kernel instantiations with NW = 2 DP warps (split per NW so nvcc builds them in parallel).
#include "ic_sched_kernel.cuh"

namespace icsched {
KernelFn kernel_nw2(bool sb, bool drop) {
  if (sb) return nullptr;
  return drop ? ic_dp_kernel<2, false, true> : ic_dp_kernel<2, false, false>;
}
}  // namespace icsched

// Kernel instantiations with NW = 8 DP warps (split per NW so nvcc builds them in parallel).
#include "ic_sched_kernel.cuh"

namespace icsched {
KernelFn kernel_nw8(bool sb, bool drop) {
  if (sb) return drop ? ic_dp_kernel<8, true, true> : ic_dp_kernel<8, true, false>;
  return drop ? ic_dp_kernel<8, false, true> : ic_dp_kernel<8, false, false>;
}
}  // namespace icsched

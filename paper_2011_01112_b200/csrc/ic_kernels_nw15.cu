// Kernel instantiations with NW = 15 DP warps: with the tail warp 16 warps, 4 per SM sub-partition, so the register budget is 128 (17 warps leave 96).
#include "ic_sched_kernel.cuh"

namespace icsched {
KernelFn kernel_nw15(bool sb, bool drop) {
  if (sb) return drop ? ic_dp_kernel<15, true, true> : ic_dp_kernel<15, true, false>;
  return drop ? ic_dp_kernel<15, false, true> : ic_dp_kernel<15, false, false>;
}
}  // namespace icsched

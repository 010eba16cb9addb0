/* ic_probe.h — measured roofline denominators for the solver (measurement only).
 *
 * The DP sweep (include/ic_sched.h) is bound by shared-memory load
 * bandwidth: one 4-byte LDS + one VIADDMNMX per option evaluation.  MEASURED_PEAKS.json
 * holds only HBM and GEMM peaks, so this probe measures the shared-memory ceiling on the
 * device it runs on: every SM runs 64 resident warps that stream conflict-free loads from
 * a 32 KB shared array (each warp reads 32 consecutive words / 16-byte vectors per
 * instruction), timed with CUDA events over ~kernel_ms, with the SM cycles elapsed read by
 * clock64 so the result is also given per clock (independent of the clock the GPU ran at).
 *
 *   mode 0  LDS.32 + IADD          (the bandwidth the sweep's scalar loads can reach)
 *   mode 1  LDS.128 + IADD         (the crossbar with a quarter of the instructions)
 *   mode 2  LDS.32 + VIADDMNMX     (the sweep's inner op: one option evaluation per lane)
 *
 * ic_probe_smem(device, mode, target_ms, &bytes_per_s, &bytes_per_clk_per_sm, &sm_clock_hz)
 *   device: CUDA ordinal; target_ms: approximate kernel duration (1..1000).
 *   Outputs: achieved shared-memory load bytes / s over the whole GPU (CUDA events), the SM
 *   clock the probe ran at (SM cycles over the %globaltimer nanoseconds of the same window)
 *   and the bytes per SM clock per SM that follow from the two.  Returns 0, -1 on invalid arguments, -3 on a CUDA error.  Synchronous;
 *   uses the legacy default stream of `device`.  Allocates and frees its own buffers.
 */
#ifndef IC_PROBE_H
#define IC_PROBE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif
int ic_probe_smem(int32_t device, int32_t mode, double target_ms, double* bytes_per_s,
                  double* bytes_per_clk_per_sm, double* sm_clock_hz);
#ifdef __cplusplus
}
#endif
#endif

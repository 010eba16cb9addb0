// ic_probe.cu — shared-memory bandwidth probe (include/ic_probe.h): the measured
// denominator of the sweep's roofline.  Measurement only; the solver never calls it.
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/ic_probe.h"

namespace {

constexpr int kThreads = 1024, kWords = 9216;  // 36 KB of shared memory per CTA

template <int MODE>
__global__ void __launch_bounds__(kThreads, 2) smem_probe(int iters, int key, int* sink,
                                                            long long* cycles) {
  // cycles[blockIdx.x] = SM cycles of this CTA's timed loop; CTA 0 also records the
  // global nanosecond timer over the same window (cycles[gridDim.x]) -> the SM clock it ran at
  __shared__ __align__(16) int buf[kWords];
  for (int i = threadIdx.x; i < kWords; i += kThreads) buf[i] = i * 2654435761u;
  __syncthreads();
  unsigned long long g0 = 0;
  if (blockIdx.x == 0 && threadIdx.x == 0) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g0));
  const long long t0 = clock64();
  int acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  if (MODE == 1) {
    const int4* b4 = reinterpret_cast<const int4*>(buf);
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int4 v = b4[(i & 7) * 128 + u * 32 + threadIdx.x];  // < kWords / 4
        acc[u] += v.x ^ v.y ^ v.z ^ v.w;
      }
    }
  } else {
    for (int i = 0; i < iters; ++i) {
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int v = buf[(i & 31) * 256 + u * 32 + threadIdx.x];  // < kWords
        acc[u] = MODE == 2 ? __viaddmax_s32(v, key, acc[u]) : acc[u] + v;
      }
    }
  }
  __syncthreads();
  const long long t1 = clock64();
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    unsigned long long g1;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g1));
    cycles[gridDim.x] = (long long)(g1 - g0);
  }
  int s = 0;
#pragma unroll
  for (int u = 0; u < 8; ++u) s ^= acc[u];
  if (s == 0x7fffffff) sink[0] = s;  // keeps the loads live
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

template <int MODE>
int run(int sms, int iters, float* ms, double* cyc_mean, double* clk_hz, int* sink, long long* cycles) {
  cudaEvent_t e0, e1;
  if (cudaEventCreate(&e0) != cudaSuccess || cudaEventCreate(&e1) != cudaSuccess) return -3;
  const int grid = 2 * sms;
  smem_probe<MODE><<<grid, kThreads>>>(iters / 8 + 1, 3, sink, cycles);  // warm-up
  cudaEventRecord(e0);
  smem_probe<MODE><<<grid, kThreads>>>(iters, 3, sink, cycles);
  cudaEventRecord(e1);
  if (cudaEventSynchronize(e1) != cudaSuccess) return -3;
  cudaEventElapsedTime(ms, e0, e1);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  long long h[2 * 1024 + 1];
  if (grid > 2 * 1024 || cudaMemcpy(h, cycles, sizeof(long long) * (grid + 1), cudaMemcpyDeviceToHost) != cudaSuccess)
    return -3;
  *clk_hz = h[grid] > 0 ? (double)h[0] / (h[grid] * 1e-9) : 0.0;
  double c = 0;
  for (int i = 0; i < grid; ++i) c += (double)h[i];
  *cyc_mean = c / grid;
  return cudaGetLastError() == cudaSuccess ? 0 : -3;
}

}  // namespace

extern "C" int ic_probe_smem(int32_t device, int32_t mode, double target_ms, double* bytes_per_s,
                             double* bytes_per_clk_per_sm, double* sm_clock_hz) {
  if (mode < 0 || mode > 2 || !bytes_per_s || !bytes_per_clk_per_sm || !sm_clock_hz ||
      !(target_ms >= 1 && target_ms <= 1000))
    return -1;
  if (cudaSetDevice(device) != cudaSuccess) return -3;
  int sms = 0;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) return -3;
  int* sink = nullptr;
  long long* cycles = nullptr;
  if (cudaMalloc(&sink, 4) != cudaSuccess) return -3;
  if (cudaMalloc(&cycles, sizeof(long long) * (2 * sms + 1)) != cudaSuccess) {
    cudaFree(sink);
    return -3;
  }
  double clk = 0;
  auto go = [&](int iters, float* ms, double* cyc) {
    return mode == 0   ? run<0>(sms, iters, ms, cyc, &clk, sink, cycles)
           : mode == 1 ? run<1>(sms, iters, ms, cyc, &clk, sink, cycles)
                       : run<2>(sms, iters, ms, cyc, &clk, sink, cycles);
  };
  // calibrate the iteration count to about target_ms, then measure
  int iters = 256, rc = 0;
  float ms = 0;
  double cyc = 0;
  for (int k = 0; k < 12; ++k) {
    if ((rc = go(iters, &ms, &cyc)) != 0) break;
    if (ms >= target_ms * 0.5) break;
    iters = (int)(iters * (target_ms / (ms > 0.01 ? ms : 0.01)));
    if (iters > (1 << 24)) iters = 1 << 24;
  }
  if (rc == 0) rc = go(iters, &ms, &cyc);
  if (rc == 0) {
    const double per_thread = (mode == 1 ? 16.0 : 4.0) * 8.0 * iters;
    const double bytes_cta = per_thread * kThreads;
    *bytes_per_s = bytes_cta * 2.0 * sms / (ms * 1e-3);
    *sm_clock_hz = clk;
    // per SM clock: the event-timed rate over the clock the SMs ran at (CTA 0's cycles over
    // the global timer); the mean CTA cycle count is the cross-check (two CTAs share an SM)
    *bytes_per_clk_per_sm = clk > 0 ? *bytes_per_s / (sms * clk) : 2.0 * bytes_cta / cyc;
  }
  cudaFree(sink);
  cudaFree(cycles);
  return rc;
}

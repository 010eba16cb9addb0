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
  __shared__ __align__(16) int buf[kWords];
  for (int i = threadIdx.x; i < kWords; i += kThreads) buf[i] = i * 2654435761u;
  __syncthreads();
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
  int s = 0;
#pragma unroll
  for (int u = 0; u < 8; ++u) s ^= acc[u];
  if (s == 0x7fffffff) sink[0] = s;  // keeps the loads live
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

template <int MODE>
int run(int sms, int iters, float* ms, double* cyc_mean, int* sink, long long* cycles) {
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
  long long h[2 * 1024];
  if (grid > 2 * 1024 || cudaMemcpy(h, cycles, sizeof(long long) * grid, cudaMemcpyDeviceToHost) != cudaSuccess)
    return -3;
  double c = 0;
  for (int i = 0; i < grid; ++i) c += (double)h[i];
  *cyc_mean = c / grid;
  return cudaGetLastError() == cudaSuccess ? 0 : -3;
}

}  // namespace

extern "C" int ic_probe_smem(int32_t device, int32_t mode, double target_ms, double* bytes_per_s,
                             double* bytes_per_clk_per_sm) {
  if (mode < 0 || mode > 2 || !bytes_per_s || !bytes_per_clk_per_sm || !(target_ms >= 1 && target_ms <= 1000))
    return -1;
  if (cudaSetDevice(device) != cudaSuccess) return -3;
  int sms = 0;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device) != cudaSuccess) return -3;
  int* sink = nullptr;
  long long* cycles = nullptr;
  if (cudaMalloc(&sink, 4) != cudaSuccess) return -3;
  if (cudaMalloc(&cycles, sizeof(long long) * 2 * sms) != cudaSuccess) {
    cudaFree(sink);
    return -3;
  }
  auto go = [&](int iters, float* ms, double* cyc) {
    return mode == 0 ? run<0>(sms, iters, ms, cyc, sink, cycles)
                     : mode == 1 ? run<1>(sms, iters, ms, cyc, sink, cycles) : run<2>(sms, iters, ms, cyc, sink, cycles);
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
    *bytes_per_clk_per_sm = 2.0 * bytes_cta / cyc;  // two resident CTAs share one SM's crossbar
  }
  cudaFree(sink);
  cudaFree(cycles);
  return rc;
}

// ic_gen_device.cu — on-device build of the seeded input generator (K9).
// The recipe lives in gen/ic_gen_core.h (input plumbing shared with the
// tests; no solver arithmetic).  One thread per task row; rank w of a
// multi-GPU sweep generates its own global-id shard without any H2D copy.
#include <cuda_runtime.h>

#include "../../include/ic_gen.h"

namespace {

__global__ void gen_kernel(const ic_gen_config c, int64_t id_offset, int64_t n_instances, int64_t* task_begin,
                           int32_t* release, int32_t* deadline, int32_t* mand_wcet, uint8_t* n_opt,
                           int32_t* opt_wcet, uint32_t* mand_conf, int32_t* opt_gain) {
  const int64_t N = c.n_tasks, st = c.opt_stride;
  const int64_t total = n_instances * N;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t <= n_instances || t < total;
       t += (int64_t)gridDim.x * blockDim.x) {
    if (t <= n_instances) task_begin[t] = t * N;
    if (t < total) {
      const int64_t b = t / N;
      const int32_t i = (int32_t)(t - b * N);
      ic_gen_task(&c, (uint64_t)(id_offset + b), i, release + t, deadline + t, mand_wcet + t, n_opt + t,
                  opt_wcet + t * st, mand_conf + t, opt_gain + t * st);
    }
  }
}

}  // namespace

extern "C" int ic_gen_batch_device(const ic_gen_config* c, int64_t id_offset, int64_t n_instances,
                                   int64_t* task_begin, int32_t* release, int32_t* deadline,
                                   int32_t* mand_wcet, uint8_t* n_opt, int32_t* opt_wcet,
                                   uint32_t* mand_conf, int32_t* opt_gain, void* cuda_stream) {
  if (!c || n_instances < 0 || id_offset < 0 || !task_begin) return -1;
  if (c->n_tasks < 0 || c->n_opt < 0 || c->n_opt > c->opt_stride || c->horizon < 1 ||
      c->u_lo_q16 < 0 || c->u_lo_q16 > c->u_hi_q16 || c->d_lo < 0 || c->d_lo > c->horizon)
    return -1;
  const int64_t total = n_instances * c->n_tasks;
  const int64_t work = total > n_instances + 1 ? total : n_instances + 1;
  int64_t blocks = (work + 255) / 256;
  if (blocks > 148 * 32) blocks = 148 * 32;
  gen_kernel<<<(unsigned)blocks, 256, 0, (cudaStream_t)cuda_stream>>>(
      *c, id_offset, n_instances, task_begin, release, deadline, mand_wcet, n_opt, opt_wcet, mand_conf,
      opt_gain);
  return cudaGetLastError() == cudaSuccess ? 0 : -3;
}

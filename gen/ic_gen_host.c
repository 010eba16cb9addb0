/* ic_gen_host.c — host build of the seeded generator (gen/libicgen.so).
 * See include/ic_gen.h for the contract; the recipe is in ic_gen_core.h. */
#include "../include/ic_gen.h"
#include <stddef.h>

int ic_gen_validate(const ic_gen_config* c) {
  if (!c) return -1;
  if (c->n_tasks < 0 || c->n_opt < 0 || c->n_opt > c->opt_stride || c->opt_stride > 255) return -1;
  if (c->horizon < 1 || c->u_lo_q16 < 0 || c->u_lo_q16 > c->u_hi_q16) return -1;
  if (c->d_lo < 0 || c->d_lo > c->horizon) return -1;
  return 0;
}

int ic_gen_batch_host(const ic_gen_config* c, int64_t id_offset, int64_t n_instances,
                      int64_t* task_begin, int32_t* release, int32_t* deadline,
                      int32_t* mand_wcet, uint8_t* n_opt, int32_t* opt_wcet,
                      uint32_t* mand_conf, int32_t* opt_gain) {
  if (ic_gen_validate(c) || n_instances < 0 || id_offset < 0) return -1;
  if (!task_begin) return -1;
  const int64_t N = c->n_tasks, st = c->opt_stride;
  if (n_instances * N > 0 && (!release || !deadline || !mand_wcet || !n_opt || !mand_conf ||
                              (st > 0 && (!opt_wcet || !opt_gain))))
    return -1;
  for (int64_t b = 0; b <= n_instances; ++b) task_begin[b] = b * N;
  for (int64_t b = 0; b < n_instances; ++b) {
    for (int32_t i = 0; i < N; ++i) {
      const int64_t t = b * N + i;
      ic_gen_task(c, (uint64_t)(id_offset + b), i, release + t, deadline + t, mand_wcet + t,
                  n_opt + t, opt_wcet + t * st, mand_conf + t, opt_gain + t * st);
    }
  }
  return 0;
}

/* ic_gen.h — C ABI of the seeded synthetic input generator (input plumbing).
 *
 * The generator writes task sets in exactly the input layout of
 * include/ic_sched.h (ic_batch_in): instance b of the batch owns tasks
 * [b*N, (b+1)*N); opt_wcet / opt_gain rows have `opt_stride` entries.
 * Instance b is global instance id `id_offset + b`, so a shard of a large
 * sweep generated on rank w is byte-identical to the same ids generated
 * anywhere else.
 *
 * The recipe (utilisation, deadlines, confidence curves) is documented in
 * gen/ic_gen_core.h and DESIGN.md "Input recipe".  It contains none of the
 * solver's arithmetic.
 *
 * Two entry points with identical output:
 *   ic_gen_batch_host   — gen/libicgen.so, host pointers, single-threaded.
 *   ic_gen_batch_device — paper_2011_01112_b200/libicsched.so, CUDA device
 *                         pointers, stream-ordered (cudaStream_t as void*).
 * Both return 0 on success, -1 on invalid arguments (null pointer,
 * n_tasks < 0, n_opt > opt_stride, horizon < 1, u_lo > u_hi, d_lo > horizon),
 * and the device variant returns -3 if a CUDA call fails.
 * All buffers are owned by the caller and must hold n_instances*n_tasks
 * task rows (task_begin: n_instances+1 entries).
 */
#ifndef IC_GEN_H
#define IC_GEN_H
#include <stdint.h>
#include "../gen/ic_gen_core.h"

#ifdef __cplusplus
extern "C" {
#endif

int ic_gen_batch_host(const ic_gen_config* cfg, int64_t id_offset, int64_t n_instances,
                      int64_t* task_begin, int32_t* release, int32_t* deadline,
                      int32_t* mand_wcet, uint8_t* n_opt, int32_t* opt_wcet,
                      uint32_t* mand_conf, int32_t* opt_gain);

int ic_gen_batch_device(const ic_gen_config* cfg, int64_t id_offset, int64_t n_instances,
                        int64_t* task_begin, int32_t* release, int32_t* deadline,
                        int32_t* mand_wcet, uint8_t* n_opt, int32_t* opt_wcet,
                        uint32_t* mand_conf, int32_t* opt_gain, void* cuda_stream);

#ifdef __cplusplus
}
#endif
#endif

/* ic_sched.h — C ABI of the batched confidence-maximising depth assignment.
 *
 * The operation (PAPER.md = P, SPEC.md = S; P:Lnn = line nn):
 *   Each instance is a task set J(t).  Task i is an imprecise
 *   computation: a mandatory block of m_i ticks with confidence a_i0,
 *   followed by S_i optional stages with WCETs c_ik (P:L48 p_il) and
 *   confidence gains g_ik, so that R_i(k) = a_i0 + sum_{j<=k} g_ij is the
 *   confidence after k optional stages (P:L48 R_i^L) and
 *   C_i(k) = m_i + sum_{j<=k} c_ij its cumulative WCET (P:L48 P_i^L).
 *   The solver chooses for every task k_i in {dropped, 0..S_i} so that the
 *   quantised total sum floor(R_i(k_i)/Delta) is maximal while every
 *   kept task finishes by its (adjusted) deadline when the kept tasks
 *   run back to back in EDF order — the paper's
 *   depth assignment, Eqs. 1-2 and Algorithm 1.  Among optimal
 *   plans it returns the one with the least makespan (Eq. 2's "least amount
 *   of execution time"), then the smallest depth vector compared from
 *   the last EDF task backwards, so the result is unique and
 *   bit-reproducible.
 *   Delta is fixed (0.1) or the FPTAS step Delta = eps*R/N of
 *   Theorem 1 with R the best individually feasible reward.
 *
 * Units: time in integer ticks; confidence in integer micro-units (1e-6).
 * EDF order: ascending (deadline, release, index within the instance).
 * A task starts at max(previous kept finish, release) (reading R9;
 * with all releases 0 this is exactly the paper's Eq. 2).
 *
 * Ownership and calls:
 *   - All ic_batch_in / ic_batch_out pointers passed to ic_sched_solve_batch
 *     are CUDA device pointers on the handle's device, owned by the caller.
 *   - ic_sched_solve_batch is asynchronous and stream-ordered on
 *     `cuda_stream` (a cudaStream_t; NULL = legacy default stream).  Outputs
 *     are valid once the stream has synchronised.  One stream at a time per
 *     handle (the handle's workspace is reused); handles are independent.
 *   - ic_sched_solve_batch_host takes HOST pointers (pinned memory is
 *     fastest), copies inputs to handle-owned device staging, solves, copies
 *     the outputs back and synchronises `cuda_stream` before returning.
 *
 * Errors:
 *   - Host-checkable problems return a negative code immediately and launch
 *     nothing: IC_ERR_INVALID_ARG (null handle / pointer, bad config),
 *     IC_ERR_LIMIT (config beyond the compiled limits: max_tasks > 4096,
 *     max_opt_stages > 14, max_horizon > 32768, or the per-instance tables do
 *     not fit one SM's 227 KB of shared memory — see "Envelope" below — or the
 *     workspace does not fit the device), IC_ERR_CUDA (a CUDA runtime call failed; no device at
 *     all also reports this), IC_ERR_OOM (workspace allocation failed).
 *   - Data problems are reported per instance in out->status, never by
 *     return code: IC_INST_BAD_INPUT when an instance has more than
 *     max_tasks tasks or a task has n_opt > max_opt_stages, release < 0,
 *     deadline >= max_horizon, any WCET < 1, mand_conf > 1e6, or a
 *     cumulative confidence R_i(k) outside [0, 1e6];
 *     IC_INST_INFEASIBLE when dropping is disallowed and no plan keeps every
 *     task; IC_INST_LIMIT when 16 * sum_i max_k q_i(k) + 16 * N >= 2^30, the max
 *     taken over the depths k that fit alone (r_i + C_i(k) <= d_i) (the packed
 *     32-bit DP keys would overflow; use a larger Delta).  For all
 *     three, every kept = -1, start = finish = -1, q_total = conf_micro = 0,
 *     conf_total = 0.0, makespan = 0.  There is no fallback path.
 */
#ifndef IC_SCHED_H
#define IC_SCHED_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct ic_sched ic_sched; /* opaque; owns device workspace, bound to one device */

enum { IC_OK = 0, IC_ERR_INVALID_ARG = -1, IC_ERR_LIMIT = -2, IC_ERR_CUDA = -3, IC_ERR_OOM = -4 };
enum { IC_DROP_ALLOWED = 0, IC_MANDATORY_ENFORCED = 1 }; /* P:L70 "if dropping entire tasks is disallowed" */
enum { IC_INST_OK = 0, IC_INST_INFEASIBLE = 1, IC_INST_BAD_INPUT = 2, IC_INST_LIMIT = 3 };

typedef struct {
  int32_t device;         /* CUDA device ordinal                                         */
  int32_t drop_mode;      /* IC_DROP_ALLOWED (default, P:L96 skip term) or IC_MANDATORY_ENFORCED */
  uint32_t delta_micro;   /* > 0: fixed Delta in micro-units (paper default 0.1 -> 100000)   */
  uint32_t epsilon_micro; /* iff delta_micro == 0: Delta = max(1, floor(eps*R/(1e6*N))),
                             R = max over tasks/depths with r + C <= d of R_i(k) (Thm 1)    */
  int32_t max_tasks;      /* N per instance, 1..4096 within the envelope below              */
  int32_t max_opt_stages; /* S_i bound and the row stride of opt_wcet/opt_gain, 0..14       */
  int32_t max_horizon;    /* H: deadlines must be < H; 1..32768                             */
} ic_sched_config;

typedef struct { /* CSR: instance b owns tasks [task_begin[b], task_begin[b+1]) */
  int64_t n_instances;
  const int64_t* task_begin;  /* [B+1], non-decreasing, task_begin[0] is the first task row */
  const int32_t* release;     /* [T] ticks, >= 0 (earliest start)                          */
  const int32_t* deadline;    /* [T] ticks, adjusted, inclusive; may be negative     */
  const int32_t* mand_wcet;   /* [T] ticks >= 1 (the mandatory part as one block, omega = 1) */
  const uint8_t* n_opt;       /* [T] S_i <= max_opt_stages                                  */
  const int32_t* opt_wcet;    /* [T][max_opt_stages] ticks >= 1 (first S_i entries used)    */
  const uint32_t* mand_conf;  /* [T] micro-confidence of the mandatory result, <= 1e6       */
  const int32_t* opt_gain;    /* [T][max_opt_stages] micro-confidence gain of each stage (may
                                 be negative: confidence may dip, reading R17)     */
} ic_batch_in;

typedef struct {
  int8_t* kept;        /* [T] -1 = dropped (planned miss), else #optional stages kept 0..S_i */
  int32_t* start;      /* [T] ticks, -1 if dropped                                          */
  int32_t* finish;     /* [T] ticks, -1 if dropped; finish = start + C_i(kept)               */
  int64_t* q_total;    /* [B] sum of floor(R/Delta) over kept tasks (the DP objective)       */
  int64_t* conf_micro; /* [B] sum of R_i(kept) over kept tasks, exact                        */
  double* conf_total;  /* [B] conf_micro / 1e6                                               */
  int32_t* makespan;   /* [B] finish of the last kept task (0 if none)                       */
  uint8_t* status;     /* [B] IC_INST_*                                                      */
  int64_t* stats;      /* nullable; [8] accumulated (+=) over the batch: instances, tasks of
                          OK instances, dropped tasks of OK instances, instances not OK,
                          kept optional stages, offered optional stages (OK instances),
                          sum conf_micro, sum q_total                                        */
} ic_batch_out;

/* Envelope.  One SM holds an instance's DP row (4 (H + pad) bytes, pad >= 64 ticks) and
 * its per-task tables (option table 8 kp bytes per slot with kp = max_opt_stages + 2
 * rounded down to even, plus ~84 bytes of EDF keys, row headers and staging), with two
 * table slots when they fit (setup of the next instance overlaps the sweep) and one
 * otherwise.  So max_tasks is bounded by about (227 KB - 4 (H + pad)) / (8 kp + 52):
 * e.g. ~1500 tasks at S = 8, H = 4096 and ~500 at S = 14, H = 32768; beyond that
 * ic_sched_create returns IC_ERR_LIMIT (tests/test_gpu_parity.py::test_create_envelope
 * finds the boundary). */
int ic_sched_create(const ic_sched_config* cfg, ic_sched** out);

/* Launch tuning, fixed at create time (A/B measurements and tests that must reach every
 * kernel variant).  ic_sched_create(cfg, out) == ic_sched_create_tuned(cfg, NULL, out);
 * a zero field means "the default the library picks".  The library never reads the
 * process environment.  Results are identical for every valid tuning;
 * IC_ERR_INVALID_ARG for out-of-range fields. */
typedef struct {
  int32_t dp_warps;      /* 1, 2, 4, 8, 15 or 16 DP warps per instance (default: ~32 column groups per thread;
                            15: with the tail warp 4 warps per SM sub-partition, 128 registers) */
  int32_t pad_cols;      /* NEG pad left of column 0 in ticks (default: grown into spare shared memory)      */
  int32_t in_place;      /* 1: rows updated in place (forces >= 8 DP warps); default only when H needs it     */
  int32_t slots;         /* 1: setup and sweep serialised (one table slot); default 2 when they fit           */
  int32_t decisions;     /* 1: decisions in shared memory if they fit; 2: one global buffer; default 2 global */
  int32_t option_tables; /* 1: option tables of both slots in a per-CTA global slab (>= 8 DP warps)          */
  int32_t axis;          /* 1: time axis only; 2: reward axis whenever eligible; default per instance         */
  int32_t ckpt;          /* re-plan checkpoint spacing in rows, power of two (default 4)                     */
  int32_t ctas_per_sm;   /* cap on resident CTAs per SM (default: occupancy)                                 */
  int32_t no_vec_loads;  /* 1: scalar descriptor loads only                                                  */
  int32_t kernel;        /* 1: warp-specialised kernel; 2: one warp per instance; default by shape          */
  int32_t packed_options;/* 2: int2 option tables in the one-warp kernel; default packed 32-bit entries when
                            a fixed Delta >= 489 micro and H <= 4096 bound every field to 16 bits      */
  int32_t discard;       /* 1: invalidate each instance's dead decision lines in L2 after its backtrack
                            (DRAM ~1.1x the algorithmic bytes); 2: never; default: on in the one-warp
                            kernel.  The warp-specialised kernel honours it only when built with
                            IC_WS_DISCARD=1 (the code alone costs its sweep 2 %); otherwise it never
                            discards and the field is accepted and ignored there */
} ic_sched_tuning;
int ic_sched_create_tuned(const ic_sched_config* cfg, const ic_sched_tuning* tuning, ic_sched** out);

int ic_sched_solve_batch(ic_sched* h, const ic_batch_in* in, ic_batch_out* out, void* cuda_stream);
int ic_sched_solve_batch_host(ic_sched* h, const ic_batch_in* in, ic_batch_out* out, void* cuda_stream);
int ic_sched_destroy(ic_sched* h);

/* ---- Stage completion (NEXT-3; the scheduler's second event) ---------------
 * After a stage of the EDF-current task J_1 (the first kept task in EDF order) completes,
 * its future confidences are re-predicted from the observed one:
 *   IC_UTIL_MAX  R^{L+1} = 1;   IC_UTIL_EXP  R^{L+1} = R^L + (1 - R^L) / 2;
 *   IC_UTIL_LIN  R^{L+1} = min(1, R^L * P^{L+1} / P^L);
 *   IC_UTIL_GIVEN  the instance's own gains (the paper's oracle utility)
 * (integer floor in micro-units).  If no planned depth of J_1 got less valuable, the plan
 * stands.  Otherwise Eq. 5: among the later EDF tasks i and depths
 * l > l_i* whose extra WCET fits J_1's released budget sum_{l'=l_1+1}^{l_1*} p_{1l'} and
 * keep every deadline, take the largest gain R_i^l - R_i^{l_i*} (ties: the
 * earlier task, then the shallower depth); if it exceeds J_1's remaining predicted gain
 * R_1^{l_1*} - R_1^{l_1}, J_1 stops at l_1 and task i runs to l.  Dropped tasks count
 * as l_i* = -1 (R = 0, C = 0).
 *   upd->kept:     [T] current plan (as ic_sched_solve_batch writes it), device pointer
 *   upd->done:     [B] optional stages J_1 has completed, 0 <= done <= kept(J_1)
 *   upd->observed: [B] J_1's confidence observed after them, micro-units <= 1e6
 * Outputs: the new plan in out (kept/start/finish/makespan/status; conf_micro and
 * conf_total = the plan's predicted confidence with J_1 on its new curve; q_total = 0),
 * swapped[B] = 1 where Eq. 5 changed the plan.  Invalid instances or updates get
 * IC_INST_BAD_INPUT; a given plan that misses a deadline gets IC_INST_INFEASIBLE.
 * Asynchronous on cuda_stream; device pointers; the handle's limits apply. */
enum { IC_UTIL_GIVEN = 0, IC_UTIL_MAX = 1, IC_UTIL_EXP = 2, IC_UTIL_LIN = 3 };
typedef struct {
  const int8_t* kept;
  const int8_t* done;
  const uint32_t* observed;
  int32_t heuristic;
} ic_stage_update;
int ic_sched_reassign_batch(ic_sched* h, const ic_batch_in* in, const ic_stage_update* upd, ic_batch_out* out,
                            uint8_t* swapped, void* cuda_stream);

/* ---- Incremental re-plan on arrival (NEXT-2; Alg. 1 from row k) -------
 * "When a task J_k arrives whose deadline is d_k, existing table rows for tasks with
 * deadlines d < d_k stay the same.  Table rows for tasks with deadlines d >= d_k
 * (including the new arrival) need to be (re)computed".  With a state buffer
 * the solver keeps every DP row of each instance (active columns + tail value), its
 * decisions and tail codes:
 *   ic_sched_state_bytes(h, B)        bytes of state for B instances (caller allocates,
 *                                     device memory, 256-byte aligned)
 *   ic_sched_solve_batch_state(...)   = ic_sched_solve_batch, and fills the state
 *   ic_sched_replan_batch(...)        the inputs are the previous instances with ONE new
 *                                     task appended at the end of each instance (every
 *                                     other task unchanged and in the same order); rows
 *                                     before the arrival's EDF position are taken from the
 *                                     state, the rest recomputed; the state is updated, so
 *                                     arrivals can be chained.  Results are identical to a
 *                                     full ic_sched_solve_batch of the new instances.
 *   ic_sched_depart_batch(...)        a departure (a request answered or expired
 *                                     leaves the task set): the inputs are the previous
 *                                     instances with ONE task removed (the others unchanged
 *                                     and in the same order); removed_index[b] is its input
 *                                     index in the previous instance and removed_deadline[b],
 *                                     removed_release[b] its deadline and release, which fix
 *                                     its old EDF position k: rows before k are kept, the rest
 *                                     recomputed, the state updated.  Results are identical to
 *                                     a full solve of the new instances.  Device pointers [B].
 * Requires a fixed Delta (delta_micro > 0: the FPTAS step eps*R/N changes with N)
 * (IC_ERR_INVALID_ARG otherwise); any horizon (in-place rows at H = 32768 included; the state
 * then holds (max_tasks / ckpt + 1) * (H + 1) * 4 bytes of rows per instance).  Every ckpt-th row
 * is kept (ic_sched_tuning.ckpt, default 4), so a re-plan restarts at the last kept row before the
 * arrival; if the instance's sweep axis changes (time vs reward) it restarts at row 0.
 * Same stream/ownership rules as ic_sched_solve_batch. */
int64_t ic_sched_state_bytes(const ic_sched* h, int64_t n_instances);
int ic_sched_solve_batch_state(ic_sched* h, const ic_batch_in* in, ic_batch_out* out, void* state,
                               void* cuda_stream);
int ic_sched_replan_batch(ic_sched* h, const ic_batch_in* in, void* state, ic_batch_out* out, void* cuda_stream);
int ic_sched_depart_batch(ic_sched* h, const ic_batch_in* in, const int32_t* removed_index,
                          const int32_t* removed_deadline, const int32_t* removed_release, void* state,
                          ic_batch_out* out, void* cuda_stream);

/* Launch geometry chosen at create time (for tests, bench and profiling).  The fields describe
 * the kernel plain solves run first (the one-warp-per-instance kernel for H <= 1024 rows or
 * the hybrid below, else the warp-specialised kernel).  hybrid = 1: fixed Delta with short
 * reward rows (N * floor(1e6 / Delta) + 1 <= 1024) but a longer horizon; a solve is then two
 * launches, the second over the instances whose sweep did not fit the first's row. */
typedef struct {
  int32_t threads_per_cta, cols_per_thread, ctas_per_sm, grid;
  int32_t smem_bytes, decisions_in_smem, double_buffered, pad_cols;
  int64_t workspace_bytes;
  int32_t kernels_per_solve, hybrid;
  int32_t packed_options;  /* 1: the one-warp kernel holds packed option entries */
} ic_sched_info;
int ic_sched_get_info(const ic_sched* h, ic_sched_info* info);

#ifdef __cplusplus
}
#endif
#endif

/* ic_sim.h — NEXT-4: event-driven simulation of RTDeepIoT edge servers (§III-B,
 * §IV) on synthetic traces, many independent servers advanced in
 * lockstep so the planner's DP runs as one GPU batch across servers.
 *
 * Model (integer ticks; confidence in micro-units):
 *   - each server runs one stage at a time, non-preemptively;
 *   - K clients per server.  period == 0: closed loop, a client issues its next request
 *     `think` ticks after the previous one is answered; period > 0: open loop, gaps between
 *     a client's requests uniform in [period/2, 3*period/2] ("within a time
 *     interval"; S:L357 for the closed loop); relative deadline D ~ U{d_lo..d_hi}
 *     (P:L245-246).  The planner plans only at GPU-idle instants, where no running stage
 *     can block the plan, so it uses the raw deadline (the P:L73-75 one-stage adjustment
 *     covers a scheduler invoked while a stage runs; reading R22);
 *   - a request is an anytime network of 1 + n_opt stages, WCET w_j = wcet_base *
 *     (1 + U[0,10%)) (the 99%-CI bound stand-in), true confidence after stage j
 *     from the generator's easy/hard mixture with residual shrink rho (gen/ic_gen_core.h);
 *   - outcome: the confidence of the last stage completed by the raw deadline;
 *     none completed = a deadline miss (counted with confidence 0).
 * Policies:
 *   IC_SIM_PLANNER — RTDeepIoT: at every scheduling point after an arrival or a stage
 *     completion the server's pending requests are re-planned with the paper's
 *     DP (ic_sched_solve_batch_host, Delta = delta_micro; completed stages are sunk,
 *     SPEC S:L237, and each task is valued floor(conf/Delta) - floor(current/Delta)), then the EDF-first request with planned stages left runs its next stage.
 *     Utility: IC_SIM_UTIL_EXP (prior r_0 before the first stage, then Exp) or
 *     IC_SIM_UTIL_ORACLE (the true curve, RTDeepIoT-OPT).
 *   IC_SIM_EDF — full depth, earliest deadline first;  IC_SIM_LCF — least current
 *   confidence first (unstarted lowest, ties earlier deadline);  IC_SIM_RR — stage-level
 *   round robin in arrival order.
 * Returns 0 on success, -1 invalid config, -3 CUDA error (planner only: the baselines
 * need no GPU).  Deterministic for a given config. */
#ifndef IC_SIM_H
#define IC_SIM_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { IC_SIM_PLANNER = 0, IC_SIM_EDF = 1, IC_SIM_LCF = 2, IC_SIM_RR = 3 };
enum { IC_SIM_UTIL_EXP = 0, IC_SIM_UTIL_ORACLE = 1 };

typedef struct {
  int32_t servers, clients, requests_per_client, n_opt;
  int32_t wcet_base, d_lo, d_hi, think;
  uint64_t seed;
  int32_t policy, utility;
  uint32_t delta_micro;  /* planner's Delta (paper default 0.1 = 100000) */
  uint32_t prior_micro;  /* planner's confidence prior before a request's first stage */
  int32_t device;
  int32_t period;        /* 0: closed loop (think); > 0: open loop, mean gap in ticks */
  int32_t plan_cells_per_tick; /* scheduler cost model: > 0: every plan
                                  holds the server for cells / plan_cells_per_tick ticks (the
                                  fraction carried to the server's next plan) before the next
                                  stage may start, cells = the size of the
                                  paper's reward-indexed table, sum_i (Qpre_i + 1)(S_i + 1);
                                  0: planning is free (the GPU-batched solver's view) */
} ic_sim_config;

typedef struct {
  int64_t requests, misses, stages_run, plans, rounds;
  int64_t conf_micro;     /* sum of the outcome confidences */
  double accuracy;        /* conf_micro / 1e6 / requests (misses count 0) */
  double miss_rate, mean_depth;
  double sim_seconds, gpu_seconds;
  int64_t plan_ticks, busy_ticks; /* ticks spent planning (cost model) and running stages */
} ic_sim_result;

/* Parity hook: a copy of the first planner batches the simulator sent to the solver, inputs
 * (the ic_batch_in layout, opt_* rows with stride n_opt) and the solver's outputs, until
 * either capacity is reached (whole batches only).  All pointers are caller-owned host
 * buffers of the stated capacities; n_instances / n_tasks report what was written. */
typedef struct {
  int64_t cap_instances, cap_tasks;
  int64_t n_instances, n_tasks;
  int64_t* task_begin;  /* [cap_instances + 1] */
  int32_t *release, *deadline, *mand_wcet;
  uint8_t* n_opt;
  int32_t* opt_wcet;    /* [cap_tasks][n_opt] */
  uint32_t* mand_conf;
  int32_t* opt_gain;    /* [cap_tasks][n_opt] */
  int8_t* kept;
  int32_t *start, *finish;
  int64_t *q_total, *conf_micro;
  int32_t* makespan;
  uint8_t* status;
} ic_sim_dump;

int ic_sim_run(const ic_sim_config* cfg, ic_sim_result* out);
int ic_sim_run_dump(const ic_sim_config* cfg, ic_sim_result* out, ic_sim_dump* dump);

#ifdef __cplusplus
}
#endif
#endif

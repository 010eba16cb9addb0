/* ic_gen_core.h — seeded synthetic task-set generator (input plumbing only).
 *
 * This module is shared by the CPU oracle's tests and by the CUDA path's
 * on-device generator (K9).  It produces the *inputs* of the solver in the
 * C-ABI layout of include/ic_sched.h and holds none of the method's
 * arithmetic: no quantisation, no prefix sums used by the solver, no EDF
 * ordering, no DP.  Everything here is integer-only so host and device
 * produce byte-identical buffers for the same (seed, global instance id).
 *
 * Workload shape:
 *   - ResNet-style anytime network: 1 mandatory block + S optional stages of
 *     near-uniform cost ("divide the number of layers in ResNet uniformly
 *     into three stages").  Nominal stage cost
 *     c = U*H/(N*(S+1)); each stage is inflated by U[0,10%) as a stand-in for
 *     the 99%-CI WCET of PAPER.md L246.
 *   - Per-instance utilisation U ~ U[u_lo, u_hi] (full-depth demand / H).
 *   - Raw relative deadlines D ~ U{d_lo..H};
 *     adjusted deadline d = D - max stage WCET.
 *   - Releases r = 0 (snapshot of J(t)) or, for tests,
 *     r ~ U{0..H/2}.
 *   - Confidence: mandatory confidence a0 from an easy/hard mixture;
 *     residual to 1 shrinks by rho ~ U[0.3,0.8] per stage (rho = 0.5 is the
 *     paper's Exp heuristic).  Gains in micro-units (1e-6).
 *
 * Random numbers: Philox4x32-10 (Salmon et al. 2011), key = seed,
 * counter = (gid lo, gid hi, task or 0xFFFFFFFF, block).
 */
#ifndef IC_GEN_CORE_H
#define IC_GEN_CORE_H

#include <stdint.h>

#if defined(__CUDACC__)
#define IC_GEN_HD __host__ __device__ __forceinline__
#else
#define IC_GEN_HD static inline
#endif

typedef struct {
  uint64_t seed;
  int32_t n_tasks;      /* N tasks per instance                          */
  int32_t n_opt;        /* S optional stages per task (<= opt_stride)     */
  int32_t opt_stride;   /* row stride of opt_wcet / opt_gain (ABI max S)  */
  int32_t horizon;      /* H ticks                                        */
  int32_t u_lo_q16;     /* utilisation range, Q16.16                      */
  int32_t u_hi_q16;
  int32_t d_lo;         /* smallest raw relative deadline (ticks)         */
  int32_t release_mode; /* 0: r = 0; 1: r ~ U{0..H/2}                     */
} ic_gen_config;

IC_GEN_HD uint32_t ic_gen_mulhi32(uint32_t a, uint32_t b) {
  return (uint32_t)(((uint64_t)a * (uint64_t)b) >> 32);
}

/* Philox4x32-10 block function. */
IC_GEN_HD void ic_gen_philox(const uint32_t ctr_in[4], uint64_t seed, uint32_t out[4]) {
  uint32_t c0 = ctr_in[0], c1 = ctr_in[1], c2 = ctr_in[2], c3 = ctr_in[3];
  uint32_t k0 = (uint32_t)seed, k1 = (uint32_t)(seed >> 32);
  for (int r = 0; r < 10; ++r) {
    uint64_t p0 = (uint64_t)0xD2511F53u * c0;
    uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
    uint32_t hi0 = (uint32_t)(p0 >> 32), lo0 = (uint32_t)p0;
    uint32_t hi1 = (uint32_t)(p1 >> 32), lo1 = (uint32_t)p1;
    c0 = hi1 ^ c1 ^ k0;
    c1 = lo1;
    c2 = hi0 ^ c3 ^ k1;
    c3 = lo0;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

IC_GEN_HD void ic_gen_draw(uint64_t seed, uint64_t gid, uint32_t task, uint32_t block,
                           uint32_t out[4]) {
  uint32_t ctr[4];
  ctr[0] = (uint32_t)gid; ctr[1] = (uint32_t)(gid >> 32); ctr[2] = task; ctr[3] = block;
  ic_gen_philox(ctr, seed, out);
}

/* Uniform integer in [lo, hi] (inclusive), from one 32-bit draw. */
IC_GEN_HD int64_t ic_gen_uniform(uint32_t x, int64_t lo, int64_t hi) {
  uint64_t span = (uint64_t)(hi - lo + 1);
  return lo + (int64_t)(((uint64_t)x * span) >> 32);
}

/* Instance-level utilisation in Q16.16. */
IC_GEN_HD int32_t ic_gen_instance_u(const ic_gen_config* c, uint64_t gid) {
  uint32_t x[4];
  ic_gen_draw(c->seed, gid, 0xFFFFFFFFu, 0u, x);
  return (int32_t)ic_gen_uniform(x[0], c->u_lo_q16, c->u_hi_q16);
}

/* Generate task `i` of instance `gid`, writing one ABI row.
 * opt_wcet / opt_gain point at the task's row (opt_stride entries). */
IC_GEN_HD void ic_gen_task(const ic_gen_config* c, uint64_t gid, int32_t i,
                           int32_t* release, int32_t* deadline, int32_t* mand_wcet,
                           uint8_t* n_opt, int32_t* opt_wcet, uint32_t* mand_conf,
                           int32_t* opt_gain) {
  const int32_t N = c->n_tasks, S = c->n_opt, H = c->horizon;
  const int64_t u_q16 = ic_gen_instance_u(c, gid);
  /* nominal stage cost, Q16.16 ticks */
  const uint64_t cbar_q16 = (uint64_t)((u_q16 * (int64_t)H) / ((int64_t)N * (S + 1)));

  uint32_t x[4];
  ic_gen_draw(c->seed, gid, (uint32_t)i, 0u, x);
  const int32_t D = (int32_t)ic_gen_uniform(x[0], c->d_lo, H);
  const int easy = (int)(x[1] >> 31);
  const uint32_t a0 = easy ? (uint32_t)ic_gen_uniform(x[2], 800000, 990000)
                           : (uint32_t)ic_gen_uniform(x[2], 100000, 600000);
  const uint32_t rho_q16 = (uint32_t)ic_gen_uniform(x[3], 19661, 52429); /* [0.3, 0.8] */

  /* stage WCETs: w = max(1, round(cbar * (1 + f/65536))), f ~ U{0..6553} */
  int32_t wmax = 0;
  for (int32_t j = 0; j <= S; ++j) {
    uint32_t y[4];
    ic_gen_draw(c->seed, gid, (uint32_t)i, 1u + (uint32_t)(j >> 2), y);
    const uint64_t f = (uint64_t)ic_gen_mulhi32(y[j & 3], 6554u);
    uint64_t w = (cbar_q16 * (65536u + f) + 0x80000000ull) >> 32;
    if (w < 1) w = 1;
    const int32_t wi = (int32_t)w;
    if (wi > wmax) wmax = wi;
    if (j == 0) *mand_wcet = wi; else opt_wcet[j - 1] = wi;
  }
  for (int32_t j = S; j < c->opt_stride; ++j) { opt_wcet[j] = 0; opt_gain[j] = 0; }

  /* residual-to-one confidence curve: D_0 = 1e6 - a0, D_k = (D_{k-1} * rho) >> 16 */
  uint32_t resid = 1000000u - a0;
  for (int32_t k = 1; k <= S; ++k) {
    const uint32_t nr = (uint32_t)(((uint64_t)resid * rho_q16) >> 16);
    opt_gain[k - 1] = (int32_t)(resid - nr);
    resid = nr;
  }

  int32_t r = 0;
  if (c->release_mode == 1) {
    uint32_t z[4];
    ic_gen_draw(c->seed, gid, (uint32_t)i, 15u, z);
    r = (int32_t)ic_gen_uniform(z[0], 0, H / 2);
  }
  *release = r;
  *deadline = D - wmax;  /* subtract one stage of non-preemption */
  *n_opt = (uint8_t)S;
  *mand_conf = a0;
}

#endif /* IC_GEN_CORE_H */

/* ic_oracle.c — CPU oracle for the confidence-maximising depth assignment.
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / --impl reference legs may load this library.
 * The product path (paper_2011_01112_b200/) never links, imports or calls it,
 * and shares no code with it: the only common module is the input generator
 * in gen/, which holds none of the method's arithmetic.
 *
 * Citations: P:Lnn = /root/reference/PAPER.md line nn, S:Lnn = SPEC.md.
 * Everything is integer arithmetic: time in ticks, confidence in micro-units
 * (1e-6), so that the paper's floor(R/Delta) is exact decimal arithmetic
 * (reading R11; fp64 floor(0.7/0.1) would give 6, S:L190 needs 7).
 *
 * What is computed (DESIGN.md §"Canonical problem"):
 *   tasks i with release r_i, adjusted deadline d_i, mandatory WCET
 *   m_i, optional WCETs c_i1..c_iS (P:L48 p_il), mandatory confidence a_i0
 *   and optional gains g_ik (P:L48 R_i^L).
 *   C_i(k) = m_i + sum_{j<=k} c_ij   (P_i^L)
 *   R_i(k) = a_i0 + sum_{j<=k} g_ij  (R_i^L, cumulative confidence)
 *   q_i(k) = floor(R_i(k) / Delta)
 *   choice k_i in {DROP, 0..S_i}; DROP forbidden in ENFORCED mode.
 *   EDF order pi: (d, r, input index) ascending.
 *   schedule: F=0; for i in pi, kept: s=max(F,r_i), f=s+C_i(k_i), need f<=d_i.
 *   objective (lexicographic): max Q = sum q, then min
 *   makespan (Eq. 2's least execution time), then the smallest
 *   depth vector compared from the last task in pi backwards with
 *   DROP < 0 < 1 < ... ("ties broken toward the smaller depth").
 *
 * Three algorithms that must agree exactly (tests pin each):
 *   O1 brute force — the definition above, enumerated.
 *   O2 paper DP    — Eqs. 1-2 / Alg. 1 in the paper's order:
 *                    reward-indexed table P(i,r), r* = largest finite column,
 *                    backtrack S(N,r*) -> S(i-1, r - q) with the budget kept
 *                    explicitly so releases stay exact.
 *   O3 time DP     — the time-indexed dual G_i(t) (scale oracle; pinned
 *                    against O1 and O2).
 */
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define OR_INF INT64_MAX
#define OR_NEG (INT64_MIN / 4)

enum { OR_OK = 0, OR_INFEASIBLE = 1, OR_BAD_INPUT = 2 };

typedef struct {
  int32_t drop_mode;       /* 0 = drop allowed, 1 = mandatory enforced */
  uint32_t delta_micro;    /* > 0: fixed Delta in micro-units                  */
  uint32_t epsilon_micro;  /* used iff delta_micro == 0: Delta = eps*R/N (Thm 1) */
  int32_t max_tasks, max_opt_stages, max_horizon;
} or_cfg;

typedef struct {          /* the C-ABI input layout (include/ic_sched.h) */
  int64_t n_instances;
  const int64_t* task_begin;
  const int32_t *release, *deadline, *mand_wcet;
  const uint8_t* n_opt;
  const int32_t* opt_wcet;  /* [T][max_opt_stages] */
  const uint32_t* mand_conf;
  const int32_t* opt_gain;  /* [T][max_opt_stages] */
} or_in;

typedef struct {
  int8_t* kept; int32_t *start, *finish;
  int64_t *q_total, *conf_micro; int32_t* makespan; uint8_t* status;
  int64_t* delta_used;     /* nullable; Delta in micro-units per instance */
} or_out;

/* One instance, derived quantities.  Arrays indexed by the input order. */
typedef struct {
  int n, smax;
  int64_t r[4096], d[4096];
  int S[4096];
  int64_t *C, *R, *q;   /* [n][smax+1] */
  int pi[4096];         /* pi[pos] = input index, EDF order */
  int64_t delta;
  int bad;
} inst_t;

#define AT(a, i, k) ((a)[(size_t)(i) * (size_t)(I->smax + 1) + (size_t)(k)])

/* Task set, cumulative sums, validation, Delta, quantisation, EDF order. */
static int prep(const or_cfg* cfg, const or_in* in, int64_t b, inst_t* I) {
  const int64_t lo = in->task_begin[b], hi = in->task_begin[b + 1];
  const int st = cfg->max_opt_stages;
  I->n = (int)(hi - lo);
  I->smax = st;
  I->bad = 0;
  I->delta = 1;
  I->C = I->R = I->q = NULL;
  if (hi < lo || I->n > cfg->max_tasks || I->n > 4096) { I->bad = 1; I->n = 0; return 0; }
  size_t cells = (size_t)(I->n > 0 ? I->n : 1) * (size_t)(st + 1);
  I->C = (int64_t*)calloc(cells, sizeof(int64_t));
  I->R = (int64_t*)calloc(cells, sizeof(int64_t));
  I->q = (int64_t*)calloc(cells, sizeof(int64_t));
  for (int i = 0; i < I->n; ++i) {
    const int64_t t = lo + i;
    I->r[i] = in->release[t];
    I->d[i] = in->deadline[t];
    I->S[i] = in->n_opt[t];
    if (I->S[i] > st || I->r[i] < 0 || I->d[i] >= cfg->max_horizon || in->mand_wcet[t] < 1 ||
        in->mand_conf[t] > 1000000u) {
      I->bad = 1; continue;
    }
    /* P_i^L = sum_{l<=L} p_il; R_i^L cumulative confidence */
    AT(I->C, i, 0) = in->mand_wcet[t];
    AT(I->R, i, 0) = in->mand_conf[t];
    for (int k = 1; k <= I->S[i]; ++k) {
      const int32_t w = in->opt_wcet[t * st + (k - 1)];
      const int64_t g = in->opt_gain[t * st + (k - 1)];
      if (w < 1) I->bad = 1;
      AT(I->C, i, k) = AT(I->C, i, k - 1) + w;
      AT(I->R, i, k) = AT(I->R, i, k - 1) + g;
      if (AT(I->R, i, k) < 0 || AT(I->R, i, k) > 1000000) I->bad = 1;
    }
  }
  if (I->bad) return 0;
  /* Delta: fixed (P:L261 uses 0.1) or the FPTAS step Delta = eps*R/N,
   * with R the largest reward of an individually feasible (task, depth)
   * (reading R8: Theorem 1 needs R <= OPT). */
  if (cfg->delta_micro > 0) {
    I->delta = cfg->delta_micro;
  } else {
    int64_t Rmax = 0;
    for (int i = 0; i < I->n; ++i)
      for (int k = 0; k <= I->S[i]; ++k)
        if (I->r[i] + AT(I->C, i, k) <= I->d[i] && AT(I->R, i, k) > Rmax) Rmax = AT(I->R, i, k);
    int64_t dl = I->n > 0 ? ((int64_t)cfg->epsilon_micro * Rmax) / (1000000LL * I->n) : 1;
    I->delta = dl < 1 ? 1 : dl;
  }
  /* floor(R / Delta) */
  for (int i = 0; i < I->n; ++i)
    for (int k = 0; k <= I->S[i]; ++k) AT(I->q, i, k) = AT(I->R, i, k) / I->delta;
  /* EDF index: d_1 <= d_2 <= ...; ties by release then input index
   * (reading R10).  Plain insertion sort. */
  for (int i = 0; i < I->n; ++i) I->pi[i] = i;
  for (int a = 1; a < I->n; ++a) {
    int x = I->pi[a], p = a - 1;
    while (p >= 0) {
      int y = I->pi[p];
      int later = (I->d[y] > I->d[x]) || (I->d[y] == I->d[x] && I->r[y] > I->r[x]) ||
                  (I->d[y] == I->d[x] && I->r[y] == I->r[x] && y > x);
      if (!later) break;
      I->pi[p + 1] = y; --p;
    }
    I->pi[p + 1] = x;
  }
  return 0;
}

static void release_inst(inst_t* I) { free(I->C); free(I->R); free(I->q); }

/* Write the outputs of instance b from a choice vector (by EDF position:
 * code[pos] = 0 drop, k+1 keep k optional stages).  Schedule per P:L48/P:L90. */
static void emit(const or_in* in, const or_out* out, int64_t b, const inst_t* I,
                 const int* code, int status) {
  const int64_t lo = in->task_begin[b], n_all = in->task_begin[b + 1] - lo;
  int64_t F = 0, Q = 0, conf = 0;
  for (int64_t i = 0; i < n_all; ++i) {
    out->kept[lo + i] = -1; out->start[lo + i] = -1; out->finish[lo + i] = -1;
  }
  if (status == OR_OK) {
    for (int pos = 0; pos < I->n; ++pos) {
      const int i = I->pi[pos];
      if (code[pos] == 0) continue;
      const int k = code[pos] - 1;
      const int64_t s = F > I->r[i] ? F : I->r[i];
      const int64_t f = s + AT(I->C, i, k);
      out->kept[lo + i] = (int8_t)k;
      out->start[lo + i] = (int32_t)s;
      out->finish[lo + i] = (int32_t)f;
      F = f;
      Q += AT(I->q, i, k);
      conf += AT(I->R, i, k);
    }
  }
  out->q_total[b] = Q;
  out->conf_micro[b] = conf;
  out->makespan[b] = (int32_t)F;
  out->status[b] = (uint8_t)status;
  if (out->delta_used) out->delta_used[b] = I->delta;
}

/* ---------------- O1: brute force over all depth vectors ------------- */
static int solve_brute(const or_cfg* cfg, inst_t* I, int* best) {
  const int n = I->n, lowc = cfg->drop_mode == 0 ? 0 : 1;
  int code[4096];
  double combos = 1;
  for (int pos = 0; pos < n; ++pos) combos *= (double)(I->S[I->pi[pos]] + 2 - lowc);
  if (combos > 1e7) return -2; /* cap */
  int have = 0;
  int64_t bestQ = 0, bestF = 0;
  for (int pos = 0; pos < n; ++pos) code[pos] = lowc;
  for (;;) {
    /* evaluate: EDF sequence of the kept tasks, inclusive deadline test */
    int64_t F = 0, Q = 0;
    int ok = 1;
    for (int pos = 0; pos < n && ok; ++pos) {
      const int i = I->pi[pos];
      if (code[pos] == 0) continue;
      const int k = code[pos] - 1;
      const int64_t s = F > I->r[i] ? F : I->r[i];
      const int64_t f = s + AT(I->C, i, k);
      if (f > I->d[i]) ok = 0;
      F = f;
      Q += AT(I->q, i, k);
    }
    if (ok) {
      int better = !have || Q > bestQ || (Q == bestQ && F < bestF);
      if (!better && Q == bestQ && F == bestF) {
        for (int pos = n - 1; pos >= 0; --pos) { /* reverse-lexicographic, last task first */
          if (code[pos] != best[pos]) { better = code[pos] < best[pos]; break; }
        }
      }
      if (better) {
        have = 1; bestQ = Q; bestF = F;
        memcpy(best, code, sizeof(int) * (size_t)n);
      }
    }
    int pos = 0;
    while (pos < n && code[pos] == I->S[I->pi[pos]] + 1) { code[pos] = lowc; ++pos; }
    if (pos == n) break;
    code[pos]++;
  }
  return have ? OR_OK : OR_INFEASIBLE;
}

/* ---------------- O2: the paper's DP, Eqs. 1-2 and Alg. 1 ------------- */
/* Fills P (rows 0..N, columns 0..Qtot) for one instance; returns Qtot.
 * P(i, r) = least finish time of the first i EDF tasks attaining exactly
 * quantised reward r; OR_INF = no such selection. */
static int64_t paper_table(const or_cfg* cfg, const inst_t* I, int64_t** Pout) {
  const int n = I->n;
  int64_t qmax_prefix[4097];
  qmax_prefix[0] = 0;
  for (int pos = 0; pos < n; ++pos) {
    const int i = I->pi[pos];
    int64_t m = 0;
    for (int k = 0; k <= I->S[i]; ++k) if (AT(I->q, i, k) > m) m = AT(I->q, i, k);
    qmax_prefix[pos + 1] = qmax_prefix[pos] + m;
  }
  const int64_t Qtot = qmax_prefix[n];
  const size_t W = (size_t)Qtot + 1;
  int64_t* P = (int64_t*)malloc(sizeof(int64_t) * W * (size_t)(n + 1));
  /* row 0: P(0,0) = 0, others infinite (reading R4: a row-0 base) */
  for (size_t r = 0; r < W; ++r) P[r] = OR_INF;
  P[0] = 0;
  for (int row = 1; row <= n; ++row) {
    const int i = I->pi[row - 1];
    const int64_t* prev = P + (size_t)(row - 1) * W;
    int64_t* cur = P + (size_t)row * W;
    for (int64_t r = 0; r <= Qtot; ++r) {
      if (r > qmax_prefix[row]) { cur[r] = prev[r]; continue; } /* Alg. 1 lines 4-5 */
      /* Eq. 2: min over the skip term P(i, r) and, per depth l, the candidate
       * P_{i+1}^l + P(i, r - q) when it meets d_{i+1} (reading R1: the
       * feasibility test applies per candidate).  With a release the task
       * starts at max(F, r_i) (reading R9). */
      int64_t best = cfg->drop_mode == 0 ? prev[r] : OR_INF;
      for (int k = 0; k <= I->S[i]; ++k) {
        const int64_t qq = AT(I->q, i, k);
        if (qq > r || prev[r - qq] == OR_INF) continue;
        const int64_t s = prev[r - qq] > I->r[i] ? prev[r - qq] : I->r[i];
        const int64_t v = s + AT(I->C, i, k);
        if (v <= I->d[i] && v < best) best = v;
      }
      cur[r] = best;
    }
  }
  *Pout = P;
  return Qtot;
}

static int solve_paper(const or_cfg* cfg, inst_t* I, int* code) {
  const int n = I->n;
  int64_t* P = NULL;
  const int64_t Qtot = paper_table(cfg, I, &P);
  const size_t W = (size_t)Qtot + 1;
  /* r* = the largest finite column of row N (P:L114 read as max reward) */
  int64_t r = -1;
  for (int64_t c = Qtot; c >= 0; --c) if (P[(size_t)n * W + c] != OR_INF) { r = c; break; }
  if (r < 0) { free(P); return OR_INFEASIBLE; }
  /* backtrack from S(N, r*) to S(i-1, r - Delta*floor(R_i^{l*})), keeping the
   * remaining time budget b explicit; the first valid option in the order
   * DROP, 0, 1, ... gives the canonical (reverse-lexicographic) plan. */
  int64_t bud = P[(size_t)n * W + r];
  for (int row = n; row >= 1; --row) {
    const int i = I->pi[row - 1];
    const int64_t* prev = P + (size_t)(row - 1) * W;
    int chosen = -1;
    if (cfg->drop_mode == 0 && prev[r] <= bud) chosen = 0;
    for (int k = 0; chosen < 0 && k <= I->S[i]; ++k) {
      const int64_t qq = AT(I->q, i, k);
      if (qq > r || prev[r - qq] == OR_INF) continue;
      const int64_t lim = bud < I->d[i] ? bud : I->d[i];
      const int64_t s = prev[r - qq] > I->r[i] ? prev[r - qq] : I->r[i];
      if (s + AT(I->C, i, k) <= lim) {
        chosen = k + 1;
        r -= qq;
        bud = lim - AT(I->C, i, k);
      }
    }
    code[row - 1] = chosen; /* a valid option always exists by construction */
  }
  free(P);
  return OR_OK;
}

/* ---------------- O3: time-indexed DP (the dual of Eqs. 1-2) ------------------------- */
/* G_i(t) = best Q of the first i EDF tasks whose kept ones all finish by t:
 *   G_i(t) = max( G_{i-1}(t) [drop],
 *                 max_k G_{i-1}(min(t,d_i) - C_i(k)) + q_i(k)  if min(t,d_i)-C_i(k) >= r_i )
 * Ties go to the smallest code (drop, then fewer stages). */
static int64_t time_table(const or_cfg* cfg, const inst_t* I, int64_t** Gout, uint8_t** Dout) {
  const int n = I->n;
  int64_t T = 0;
  for (int i = 0; i < n; ++i) if (I->d[i] > T) T = I->d[i];
  const size_t W = (size_t)T + 1;
  int64_t* G = (int64_t*)malloc(sizeof(int64_t) * W * (size_t)(n + 1));
  uint8_t* D = (uint8_t*)calloc(W * (size_t)(n + 1), 1);
  for (size_t t = 0; t < W; ++t) G[t] = 0;
  for (int row = 1; row <= n; ++row) {
    const int i = I->pi[row - 1];
    const int64_t* prev = G + (size_t)(row - 1) * W;
    int64_t* cur = G + (size_t)row * W;
    uint8_t* dec = D + (size_t)row * W;
    for (int64_t t = 0; t <= T; ++t) {
      int64_t best = OR_NEG;
      int bc = -1;
      if (cfg->drop_mode == 0) { best = prev[t]; bc = 0; }
      const int64_t tt = t < I->d[i] ? t : I->d[i];
      for (int k = 0; k <= I->S[i]; ++k) {
        const int64_t src = tt - AT(I->C, i, k);
        if (src < I->r[i] || src < 0 || prev[src] == OR_NEG) continue;
        const int64_t v = prev[src] + AT(I->q, i, k);
        if (bc < 0 || v > best) { best = v; bc = k + 1; }
      }
      cur[t] = bc < 0 ? OR_NEG : best;
      dec[t] = (uint8_t)(bc < 0 ? 255 : bc);
    }
  }
  *Gout = G; *Dout = D;
  return T;
}

static int solve_time(const or_cfg* cfg, inst_t* I, int* code) {
  const int n = I->n;
  int64_t* G; uint8_t* D;
  const int64_t T = time_table(cfg, I, &G, &D);
  const size_t W = (size_t)T + 1;
  const int64_t Qs = G[(size_t)n * W + T];
  if (Qs == OR_NEG) { free(G); free(D); return OR_INFEASIBLE; }
  int64_t t = 0;
  while (G[(size_t)n * W + t] != Qs) ++t; /* least makespan attaining Q* */
  for (int row = n; row >= 1; --row) {
    const int i = I->pi[row - 1];
    const int c = D[(size_t)row * W + t];
    code[row - 1] = c;
    if (c > 0) t = (t < I->d[i] ? t : I->d[i]) - AT(I->C, i, c - 1);
  }
  free(G); free(D);
  return OR_OK;
}

/* ---------------- batch driver -------------------------------------------------------- */
int or_solve_batch(int algo, const or_cfg* cfg, const or_in* in, const or_out* out, int n_threads) {
  if (!cfg || !in || !out || algo < 1 || algo > 3) return -1;
  if (cfg->max_tasks > 4096 || cfg->max_opt_stages < 0) return -1;
  if (cfg->delta_micro == 0 && cfg->epsilon_micro == 0) return -1;
  int err = 0;
#ifdef _OPENMP
  if (n_threads > 0) omp_set_num_threads(n_threads);
#pragma omp parallel for schedule(dynamic, 16)
#endif
  for (int64_t b = 0; b < in->n_instances; ++b) {
    inst_t* I = (inst_t*)malloc(sizeof(inst_t));
    int* code = (int*)malloc(sizeof(int) * 4097);
    prep(cfg, in, b, I);
    int st;
    if (I->bad) {
      st = OR_BAD_INPUT;
    } else if (algo == 1) {
      st = solve_brute(cfg, I, code);
    } else if (algo == 2) {
      st = solve_paper(cfg, I, code);
    } else {
      st = solve_time(cfg, I, code);
    }
    if (st == -2) {
#ifdef _OPENMP
#pragma omp atomic write
#endif
      err = -2;
      st = OR_BAD_INPUT;
    }
    emit(in, out, b, I, code, st);
    release_inst(I);
    free(I); free(code);
  }
  return err;
}

/* Tables of a single instance for the pins (P(i,r) of Eq. 2; G_i(t) of O3).
 * Caller provides `buf` of `cap` int64; returns the number of columns, or
 * -1 if bad input / too small a buffer.  Rows are in EDF order, row 0 first. */
int64_t or_paper_table(const or_cfg* cfg, const or_in* in, int64_t b, int64_t* buf, int64_t cap) {
  inst_t* I = (inst_t*)malloc(sizeof(inst_t));
  prep(cfg, in, b, I);
  int64_t cols = -1;
  if (!I->bad) {
    int64_t* P;
    cols = paper_table(cfg, I, &P) + 1;
    const int64_t need = cols * (I->n + 1);
    if (need <= cap) memcpy(buf, P, sizeof(int64_t) * (size_t)need); else cols = -1;
    free(P);
  }
  release_inst(I); free(I);
  return cols;
}

int64_t or_time_table(const or_cfg* cfg, const or_in* in, int64_t b, int64_t* buf, int64_t cap) {
  inst_t* I = (inst_t*)malloc(sizeof(inst_t));
  prep(cfg, in, b, I);
  int64_t cols = -1;
  if (!I->bad) {
    int64_t* G; uint8_t* D;
    cols = time_table(cfg, I, &G, &D) + 1;
    const int64_t need = cols * (I->n + 1);
    if (need <= cap) memcpy(buf, G, sizeof(int64_t) * (size_t)need); else cols = -1;
    free(G); free(D);
  }
  release_inst(I); free(I);
  return cols;
}

/* ---------------- invariant checker ---------------------------- */
/* Returns 0 if instance b's result is a valid plan, else a bit mask:
 *  1 start < release   2 finish != start + C   4 finish > deadline
 *  8 overlap in EDF order   16 processor-demand criterion violated
 *  32 task dropped in ENFORCED mode   64 Q / confidence / makespan mismatch
 *  128 kept out of range or inconsistent drop encoding */
int or_check(const or_cfg* cfg, const or_in* in, const or_out* out, int64_t b) {
  inst_t* I = (inst_t*)malloc(sizeof(inst_t));
  prep(cfg, in, b, I);
  const int64_t lo = in->task_begin[b];
  int bits = 0;
  if (I->bad) {
    if (out->status[b] != OR_BAD_INPUT) bits |= 64;
    release_inst(I); free(I);
    return bits;
  }
  if (out->status[b] == OR_INFEASIBLE) {
    for (int i = 0; i < I->n; ++i) if (out->kept[lo + i] != -1) bits |= 128;
    if (cfg->drop_mode == 0) bits |= 32; /* drop mode always admits the empty plan */
    release_inst(I); free(I);
    return bits;
  }
  int64_t Q = 0, conf = 0, F = 0, prevf = 0;
  for (int pos = 0; pos < I->n; ++pos) {
    const int i = I->pi[pos];
    const int k = out->kept[lo + i];
    if (k < -1 || k > I->S[i]) { bits |= 128; continue; }
    if (k == -1) {
      if (cfg->drop_mode == 1) bits |= 32;
      if (out->start[lo + i] != -1 || out->finish[lo + i] != -1) bits |= 128;
      continue;
    }
    const int64_t s = out->start[lo + i], f = out->finish[lo + i];
    if (s < I->r[i]) bits |= 1;
    if (f != s + AT(I->C, i, k)) bits |= 2;
    if (f > I->d[i]) bits |= 4;
    if (s < prevf) bits |= 8;
    prevf = f;
    if (f > F) F = f;
    Q += AT(I->q, i, k);
    conf += AT(I->R, i, k);
  }
  /* processor demand: for all t1 < t2, demand of kept jobs with r >= t1 and d <= t2
   * fits in t2 - t1 (EDF schedulability of the kept set). */
  for (int a = 0; a < I->n; ++a) {
    if (out->kept[lo + a] < 0) continue;
    for (int c = 0; c < I->n; ++c) {
      if (out->kept[lo + c] < 0) continue;
      const int64_t t1 = I->r[a], t2 = I->d[c];
      if (t2 <= t1) continue;
      int64_t dem = 0;
      for (int j = 0; j < I->n; ++j) {
        const int k = out->kept[lo + j];
        if (k >= 0 && k <= I->S[j] && I->r[j] >= t1 && I->d[j] <= t2) dem += AT(I->C, j, k);
      }
      if (dem > t2 - t1) bits |= 16;
    }
  }
  if (Q != out->q_total[b] || conf != out->conf_micro[b] || F != out->makespan[b]) bits |= 64;
  release_inst(I); free(I);
  return bits;
}

/* ======================= NEXT-3: stage completion update ============================
 * Utility prediction (§II-D) and the greedy depth reassignment of Eq. 5
 * (§II-E), written in the paper's order.  All confidences in micro-units.
 *
 * Predict the next stage from the current one:
 *   Max: R^{L+1} = 1;  Exp: R^{L+1} = R^L + 0.5 (1 - R^L);
 *   Lin: R^{L+1} = min(1, R^L * P^{L+1} / P^L)   (integer floor in micro-units)
 * Given (the oracle utility): the instance's own gains are the true increments. */
enum { OR_UTIL_GIVEN = 0, OR_UTIL_MAX = 1, OR_UTIL_EXP = 2, OR_UTIL_LIN = 3 };

int64_t or_predict_next(int heuristic, int64_t r_cur, int64_t p_cur, int64_t p_next) {
  if (heuristic == OR_UTIL_MAX) return 1000000;
  if (heuristic == OR_UTIL_EXP) return r_cur + (1000000 - r_cur) / 2;
  if (heuristic == OR_UTIL_LIN) {
    const int64_t v = p_cur > 0 ? r_cur * p_next / p_cur : 1000000;
    return v < 1000000 ? v : 1000000;
  }
  return r_cur;
}

/* EDF-feasibility of a plan (codes by input index: -1 drop, else kept stages), the
 * forward schedule of P:L48/P:L90; fills start/finish and returns 1 if every kept
 * task meets its deadline. */
static int schedule_plan(const inst_t* I, const int* kept, int64_t* st, int64_t* fi, int64_t* F_out) {
  int64_t F = 0;
  int ok = 1;
  for (int pos = 0; pos < I->n; ++pos) {
    const int i = I->pi[pos];
    st[i] = fi[i] = -1;
    if (kept[i] < 0) continue;
    const int64_t s = F > I->r[i] ? F : I->r[i];
    const int64_t f = s + AT(I->C, i, kept[i]);
    if (f > I->d[i]) ok = 0;
    st[i] = s;
    fi[i] = f;
    F = f;
  }
  *F_out = F;
  return ok;
}

/* One instance: the current plan `kept_in` (by input index), the EDF-current task J_1
 * (the first kept task in EDF order) has completed `done` optional stages and shows
 * confidence `observed`.  Returns the new plan in kept_out; *swapped = 1 if changed. */
static int reassign_one(const inst_t* I, const int8_t* kept_in, int done, int64_t observed, int heuristic,
                        int* kept_out, int64_t* Rnew /* [smax+1] J_1's new curve */, int* j1_out,
                        int* swapped) {
  const int n = I->n;
  *swapped = 0;
  *j1_out = -1;
  for (int i = 0; i < n; ++i) kept_out[i] = kept_in[i];
  int p1 = -1;
  for (int pos = 0; pos < n && p1 < 0; ++pos)
    if (kept_in[I->pi[pos]] >= 0) p1 = pos;
  if (p1 < 0) return OR_OK;  /* nothing is running: the plan stands */
  const int j1 = I->pi[p1];
  *j1_out = j1;
  const int l1 = done, l1s = kept_in[j1];
  if (l1 < 0 || l1 > l1s || observed < 0 || observed > 1000000) return OR_BAD_INPUT;
  /* J_1's re-predicted curve from the observed confidence ("revisit estimated utility") */
  for (int k = 0; k <= I->S[j1]; ++k) Rnew[k] = AT(I->R, j1, k);
  Rnew[l1] = observed;
  for (int k = l1 + 1; k <= I->S[j1]; ++k) {
    if (heuristic == OR_UTIL_GIVEN)
      Rnew[k] = Rnew[k - 1] + (AT(I->R, j1, k) - AT(I->R, j1, k - 1));
    else
      Rnew[k] = or_predict_next(heuristic, Rnew[k - 1], AT(I->C, j1, k - 1), AT(I->C, j1, k));
  }
  /* "if the updated future utility ... becomes larger, our previous depth assignment still
   * preserves optimality": no decrease on [l_1, l_1*] keeps the plan */
  int lower = 0;
  for (int k = l1; k <= l1s; ++k)
    if (Rnew[k] < AT(I->R, j1, k)) lower = 1;
  if (!lower) return OR_OK;
  /* Eq. 5: the best extension of a later task within J_1's released budget
   * sum_{l'=l_1+1}^{l_1*} p_{1l'} (reading R19: the extension's own stages l_i*+1..l),
   * kept EDF-feasible (SPEC S:L217 strengthening).  Ties: earliest EDF position, then
   * the shallower depth. */
  const int64_t released = AT(I->C, j1, l1s) - AT(I->C, j1, l1);
  const int64_t rem_gain = Rnew[l1s] - Rnew[l1];
  int* plan = (int*)malloc(sizeof(int) * (size_t)(n > 0 ? n : 1));
  int64_t* st = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1) * 2);
  int64_t* fi = st + (n > 0 ? n : 1);
  int best_i = -1, best_l = -1;
  int64_t best_gain = 0;
  for (int pos = p1 + 1; pos < n; ++pos) {
    const int i = I->pi[pos];
    const int ki = kept_in[i];
    for (int l = ki + 1; l <= I->S[i]; ++l) {
      const int64_t cost = AT(I->C, i, l) - (ki >= 0 ? AT(I->C, i, ki) : 0);
      if (cost > released) break;
      const int64_t gain = AT(I->R, i, l) - (ki >= 0 ? AT(I->R, i, ki) : 0);
      if (best_i >= 0 && gain <= best_gain) continue;
      for (int q = 0; q < n; ++q) plan[q] = kept_in[q];
      plan[j1] = l1;
      plan[i] = l;
      int64_t F;
      if (!schedule_plan(I, plan, st, fi, &F)) continue;
      best_i = i; best_l = l; best_gain = gain;
    }
  }
  free(plan);
  free(st);
  /* "If R_i^{l^} - R_i^{l*} > R_1^{l_1*} - R_1^{l_1}, we replace the depth assignment" */
  if (best_i >= 0 && best_gain > rem_gain) {
    kept_out[j1] = l1;
    kept_out[best_i] = best_l;
    *swapped = 1;
  }
  return OR_OK;
}

int or_reassign_batch(const or_cfg* cfg, const or_in* in, const int8_t* kept_in, const int8_t* done,
                      const uint32_t* observed, int heuristic, const or_out* out, uint8_t* swapped) {
  if (!cfg || !in || !out || !kept_in || !done || !observed || heuristic < 0 || heuristic > 3) return -1;
  for (int64_t b = 0; b < in->n_instances; ++b) {
    inst_t* I = (inst_t*)malloc(sizeof(inst_t));
    prep(cfg, in, b, I);
    const int64_t lo = in->task_begin[b], n_all = in->task_begin[b + 1] - lo;
    for (int64_t i = 0; i < n_all; ++i) {
      out->kept[lo + i] = -1; out->start[lo + i] = -1; out->finish[lo + i] = -1;
    }
    int st = OR_BAD_INPUT, sw = 0;
    int64_t F = 0, conf = 0;
    if (!I->bad) {
      int* kept = (int*)malloc(sizeof(int) * (size_t)(I->n > 0 ? I->n : 1));
      int64_t* Rnew = (int64_t*)malloc(sizeof(int64_t) * (size_t)(I->smax + 1));
      int64_t* s = (int64_t*)malloc(sizeof(int64_t) * (size_t)(I->n > 0 ? I->n : 1) * 2);
      int64_t* f = s + (I->n > 0 ? I->n : 1);
      int j1;
      for (int i = 0; i < I->n; ++i)
        if (kept_in[lo + i] < -1 || kept_in[lo + i] > I->S[i]) I->bad = 1;
      st = I->bad ? OR_BAD_INPUT
                  : reassign_one(I, kept_in + lo, done[b], observed[b], heuristic, kept, Rnew, &j1, &sw);
      if (st == OR_OK) {
        if (!schedule_plan(I, kept, s, f, &F)) st = OR_INFEASIBLE;  /* the given plan was infeasible */
        for (int i = 0; i < I->n; ++i) {
          if (kept[i] < 0) continue;
          out->kept[lo + i] = (int8_t)kept[i];
          out->start[lo + i] = (int32_t)s[i];
          out->finish[lo + i] = (int32_t)f[i];
          conf += (i == j1) ? Rnew[kept[i]] : AT(I->R, i, kept[i]);
        }
      }
      free(kept); free(Rnew); free(s);
    }
    if (st != OR_OK) {
      for (int64_t i = 0; i < n_all; ++i) {
        out->kept[lo + i] = -1; out->start[lo + i] = -1; out->finish[lo + i] = -1;
      }
      F = 0; conf = 0; sw = 0;
    }
    out->q_total[b] = 0;
    out->conf_micro[b] = conf;
    out->makespan[b] = (int32_t)F;
    out->status[b] = (uint8_t)st;
    swapped[b] = (uint8_t)sw;
    release_inst(I);
    free(I);
  }
  return 0;
}

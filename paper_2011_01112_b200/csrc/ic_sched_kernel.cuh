// ic_sched_kernel.cuh — sm_100a kernel for the batched depth assignment.
//
// One CTA solves one instance at a time (persistent grid-stride loop over
// instances).  Per instance:
//   a1  task descriptors: coalesced loads, one thread per task
//   a2  prefix sums C_i(k), R_i(k), Delta (P:L78 / Thm 1),
//       q = R div Delta, packed option keys (q << 4) | (15 - code)
//   a3  EDF order by (d, r, idx): warp-shuffle bitonic sort for
//       N <= 32, shared-memory bitonic otherwise
//   a4  the DP sweep — the time-indexed dual of Eqs. 1-2:
//         G_i(t) = max( G_{i-1}(t) [drop],
//                       max_k G_{i-1}(min(t,d_i) - C_i(k)) + q_i(k) )
//       with options invalid before the release masked by a NEG row value.
//       Each thread owns columns t = m*NT + tid (m < COLS) and keeps its
//       G_{i-1}(t) in registers (the drop option costs no shared-memory
//       load); the option reads G_{i-1}(t - C_k) come from a shared-memory row
//       (double-buffered, or single-buffered with a read/write barrier pair).
//       One VIADDMNMX (__viaddmax_s32) per (cell, option) on packed keys
//       carries the argmax in the low 4 bits, ties resolving to the smaller
//       code (drop < 0 < 1 < ...).  4-bit decisions per cell go to shared
//       memory or to a per-CTA global slab.
//   a5  Q* = G_N(T), t* = least t with G_N(t) = Q*
//   a6  backtrack through the decision nibbles
//   a7  EDF schedule times, outputs in input order
//   a8  batch statistics (one int64 atomic per slot per CTA)
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <type_traits>

namespace icsched {

constexpr int NEG = -(1 << 30);
constexpr int MAXK = 15;  // options per task: 0..14 optional stages

struct Params {
  // inputs (device pointers)
  int64_t B;
  const int64_t* task_begin;
  const int32_t *release, *deadline, *mand_wcet;
  const uint8_t* n_opt;
  const int32_t* opt_wcet;
  const uint32_t* mand_conf;
  const int32_t* opt_gain;
  // outputs
  int8_t* kept;
  int32_t *start, *finish;
  int64_t *q_total, *conf_micro;
  double* conf_total;
  int32_t* makespan;
  uint8_t* status;
  unsigned long long* stats;
  // config
  int drop_mode;
  uint32_t delta_micro, eps_micro;
  int max_tasks, smax, H;
  // geometry
  int pad, nbuf, dec_smem, kp, np2max;
  uint32_t* dec_global;
  int64_t dec_slab_words;
  // shared-memory layout (byte offsets)
  int off_rowbuf, off_dec, off_rowp, off_tR, off_info, off_key, off_tr, off_td, off_tS, off_chosen,
      off_misc;
};

__device__ __forceinline__ int viaddmax(int a, int b, int c) { return __viaddmax_s32(a, b, c); }

// One DP row with exactly K valid options (compile-time), all COLS column groups.
template <int NT, int COLS, int K, bool SB, typename RowPtr>
__device__ __forceinline__ void dp_row(int (&G)[COLS], const Params& p, const int32_t* __restrict__ cur,
                                       RowPtr nxt, uint32_t* __restrict__ decrow,
                                       const int2* __restrict__ op, const int d, const int r_next,
                                       const int store_lim, const bool has_next, const int ncols) {
  constexpr bool single_buf = SB;
  constexpr int NQ = (COLS + 7) / 8;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int C[K > 0 ? K : 1], key[K > 0 ? K : 1];
#pragma unroll
  for (int k = 0; k < K; ++k) {
    const int2 o = op[k];
    C[k] = o.x;
    key[k] = o.y;
  }
  // admit-only value at column d, used by every column t > d (min(t, d) = d)
  int A = NEG;
  if (K > 0 && d < ncols - 1) {
    int v = NEG;
    if (lane < K) {
      const int2 o = op[lane];
      v = cur[d - o.x] + o.y;
    }
    A = __reduce_max_sync(0xffffffffu, v);
  }
  const int w0 = warp * 32;
  const int mact = d >= w0 ? min(COLS, (d - w0) / NT + 1) : 0;  // groups holding a column t <= d
  const int mlive = min(COLS, (ncols - 1 - w0) >= 0 ? (ncols - 1 - w0) / NT + 1 : 0);
  uint32_t dw[NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q) dw[q] = 0;
#pragma unroll
  for (int m = 0; m < COLS; ++m) {
    if (m < mlive) {
      const int t = m * NT + tid;
      const int drop = p.drop_mode ? NEG : (G[m] | 15);
      int v = drop;
      if (m < mact) {
#pragma unroll
        for (int k = 0; k < K; ++k) v = viaddmax(cur[t - C[k]], key[k], v);
      }
      const int tail = max(drop, A);
      v = (t <= d) ? v : tail;
      dw[m >> 3] |= (uint32_t)(v & 15) << (4 * (m & 7));
      G[m] = v & ~15;
      if (!single_buf && has_next && m * NT + w0 <= store_lim) nxt[t] = (t >= r_next) ? G[m] : NEG;
    }
  }
#pragma unroll
  for (int q = 0; q < NQ; ++q) decrow[q * NT + tid] = dw[q];
  if (single_buf) {
    __syncthreads();  // every read of the row is done before it is overwritten
    if (has_next) {
#pragma unroll
      for (int m = 0; m < COLS; ++m) {
        const int t = m * NT + tid;
        if (m < mlive && m * NT + w0 <= store_lim) nxt[t] = (t >= r_next) ? G[m] : NEG;
      }
    }
  }
}

template <int NT, int COLS, bool SB>
__device__ __forceinline__ void dp_row_dispatch(int K, int (&G)[COLS], const Params& p, const int32_t* cur,
                                                int32_t* nxt, uint32_t* decrow, const int2* op, int d,
                                                int r_next, int store_lim, bool has_next, int ncols) {
  // double-buffered rows never alias: let the compiler interleave loads and stores freely
  using RowPtr = typename std::conditional<SB, int32_t*, int32_t* __restrict__>::type;
#define IC_ROW(KK) \
  case KK: dp_row<NT, COLS, KK, SB, RowPtr>(G, p, cur, nxt, decrow, op, d, r_next, store_lim, has_next, ncols); break;
  switch (K) {
    IC_ROW(0) IC_ROW(1) IC_ROW(2) IC_ROW(3) IC_ROW(4) IC_ROW(5) IC_ROW(6) IC_ROW(7)
    IC_ROW(8) IC_ROW(9) IC_ROW(10) IC_ROW(11) IC_ROW(12) IC_ROW(13) IC_ROW(14) IC_ROW(15)
    default: break;
  }
#undef IC_ROW
}

// Slow path for rows whose longest usable option reaches further left than
// the NEG pad: source index clamped per lane to -1 (a NEG cell).
template <int NT, int COLS, bool SB>
__device__ __forceinline__ void dp_row_general(int K, int (&G)[COLS], const Params& p, const int32_t* cur,
                                               int32_t* nxt, uint32_t* decrow, const int2* op, int d,
                                               int r_next, int store_lim, bool has_next, int ncols) {
  constexpr bool single_buf = SB;
  constexpr int NQ = (COLS + 7) / 8;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int A = NEG;
  if (K > 0 && d < ncols - 1) {
    int v = NEG;
    if (lane < K) {
      const int2 o = op[lane];
      v = cur[d - o.x] + o.y;
    }
    A = __reduce_max_sync(0xffffffffu, v);
  }
  const int w0 = warp * 32;
  uint32_t dw[NQ];
#pragma unroll
  for (int q = 0; q < NQ; ++q) dw[q] = 0;
#pragma unroll
  for (int m = 0; m < COLS; ++m) {
    const int t = m * NT + tid;
    if (m * NT + w0 <= ncols - 1) {
      const int drop = p.drop_mode ? NEG : (G[m] | 15);
      int v = drop;
      if (t <= d) {
        for (int k = 0; k < K; ++k) {
          const int2 o = op[k];
          v = viaddmax(cur[max(t - o.x, -1)], o.y, v);
        }
      } else {
        v = max(drop, A);
      }
      dw[m >> 3] |= (uint32_t)(v & 15) << (4 * (m & 7));
      G[m] = v & ~15;
      if (!single_buf && has_next && m * NT + w0 <= store_lim) nxt[t] = (t >= r_next) ? G[m] : NEG;
    }
  }
#pragma unroll
  for (int q = 0; q < NQ; ++q) decrow[q * NT + tid] = dw[q];
  if (single_buf) {
    __syncthreads();
    if (has_next) {
#pragma unroll
      for (int m = 0; m < COLS; ++m) {
        const int t = m * NT + tid;
        if (m * NT + w0 <= ncols - 1 && m * NT + w0 <= store_lim) nxt[t] = (t >= r_next) ? G[m] : NEG;
      }
    }
  }
}

// Warp-level bitonic sort of up to 32 64-bit keys (one per lane), ascending.
__device__ __forceinline__ unsigned long long warp_bitonic_sort(unsigned long long x, int lane) {
#pragma unroll
  for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      const unsigned long long y = __shfl_xor_sync(0xffffffffu, x, j);
      const bool up = ((lane & k) == 0);
      const bool lower = ((lane & j) == 0);
      const bool take_min = (lower == up);
      x = take_min ? (x < y ? x : y) : (x < y ? y : x);
    }
  }
  return x;
}

template <int NT, int COLS, bool SB>
__global__ void __launch_bounds__(NT) ic_dp_kernel(const Params p) {
  extern __shared__ __align__(16) unsigned char smem[];
  constexpr int NQ = (COLS + 7) / 8;
  constexpr int CAP = NT * COLS;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  int32_t* rowbuf = (int32_t*)(smem + p.off_rowbuf);
  uint32_t* dec = p.dec_smem ? (uint32_t*)(smem + p.off_dec)
                             : p.dec_global + (int64_t)blockIdx.x * p.dec_slab_words;
  int2* rowp = (int2*)(smem + p.off_rowp);
  int32_t* tR = (int32_t*)(smem + p.off_tR);
  int4* info = (int4*)(smem + p.off_info);
  unsigned long long* skey = (unsigned long long*)(smem + p.off_key);
  int32_t* tr = (int32_t*)(smem + p.off_tr);
  int32_t* td = (int32_t*)(smem + p.off_td);
  int32_t* tS = (int32_t*)(smem + p.off_tS);
  int32_t* chosen = (int32_t*)(smem + p.off_chosen);
  int32_t* misc = (int32_t*)(smem + p.off_misc);
  unsigned long long* misc64 = (unsigned long long*)(smem + p.off_misc + 64);
  const int RS = p.pad + CAP;
  const int R1 = p.smax + 1;
  constexpr bool single_buf = SB;

  for (int bb = 0; bb < p.nbuf; ++bb)
    for (int i = tid; i < p.pad; i += NT) rowbuf[bb * RS + i] = NEG;

  unsigned long long acc[8];
#pragma unroll
  for (int s = 0; s < 8; ++s) acc[s] = 0;

  for (int64_t b = blockIdx.x; b < p.B; b += gridDim.x) {
    const int64_t lo = p.task_begin[b];
    const int64_t n64 = p.task_begin[b + 1] - lo;
    if (tid == 0) {
      misc[0] = 0;          // Rmax
      misc[1] = 0;          // dmax (T = max(0, max d))
      misc[2] = 0x7fffffff; // t*
      misc[3] = 0;          // Q* packed
      misc64[0] = 0;        // sum_i max_k q
    }
    __syncthreads();
    const bool too_many = n64 < 0 || n64 > p.max_tasks;
    const int n = too_many ? 0 : (int)n64;

    // ---- a1/a2: descriptors, validation, prefix sums, feasible-reward max
    int bad = too_many ? 1 : 0;
    int rmax_l = 0, dmax_l = 0;
    for (int i = tid; i < n; i += NT) {
      const int64_t t = lo + i;
      const int r = p.release[t], d = p.deadline[t], m = p.mand_wcet[t];
      const int S = p.n_opt[t];
      const uint32_t a0 = p.mand_conf[t];
      int tb = (S > p.smax) | (r < 0) | (d >= p.H) | (m < 1) | (a0 > 1000000u);
      tr[i] = r;
      td[i] = d;
      tS[i] = S;
      dmax_l = max(dmax_l, d);
      if (!tb) {
        int64_t C = m, R = a0;
        for (int k = 0; k <= S; ++k) {
          if (k > 0) {
            const int w = p.opt_wcet[t * p.smax + (k - 1)];
            const int g = p.opt_gain[t * p.smax + (k - 1)];
            tb |= (w < 1);
            C += w;
            R += g;
            tb |= (R < 0) | (R > 1000000);
          }
          rowp[i * p.kp + k].x = (int)min(C, (int64_t)(1 << 30));
          tR[i * R1 + k] = (int)R;
          if ((int64_t)r + C <= d && R > rmax_l) rmax_l = (int)R;
        }
      }
      bad |= tb;
    }
    bad = __syncthreads_or(bad);
    if (!bad) {
      atomicMax(&misc[0], rmax_l);
      atomicMax(&misc[1], dmax_l);
    }
    __syncthreads();
    int64_t delta = 1;
    if (p.delta_micro > 0) {
      delta = p.delta_micro;
    } else if (n > 0) {
      delta = ((int64_t)p.eps_micro * (int64_t)misc[0]) / (1000000LL * n);
      if (delta < 1) delta = 1;
    }
    if (!bad) {
      for (int i = tid; i < n; i += NT) {
        const int S = tS[i], d = td[i];
        int qmax = 0;
        for (int k = 0; k <= S; ++k) {
          const int q = (int)(tR[i * R1 + k] / delta);
          qmax = max(qmax, q);
          rowp[i * p.kp + k].y = (q << 4) | (14 - k);
        }
        atomicAdd(&misc64[0], (unsigned long long)qmax);
        const uint32_t dk = (uint32_t)d ^ 0x80000000u;
        const uint32_t rk = (uint32_t)min(tr[i], (1 << 20) - 1);
        skey[i] = ((unsigned long long)dk << 32) | ((unsigned long long)rk << 12) | (unsigned)i;
      }
    }
    int np2 = 1;
    while (np2 < n) np2 <<= 1;
    for (int i = n + tid; i < np2; i += NT) skey[i] = ~0ull;
    __syncthreads();
    const bool limit = !bad && (misc64[0] * 16ull + 16ull * (unsigned long long)n >= (1ull << 30));

    if (bad || limit) {
      // ---- per-instance error: everything dropped, status says why
      for (int64_t i = tid; i < n64; i += NT) {
        p.kept[lo + i] = -1;
        p.start[lo + i] = -1;
        p.finish[lo + i] = -1;
      }
      if (tid == 0) {
        p.q_total[b] = 0;
        p.conf_micro[b] = 0;
        p.conf_total[b] = 0.0;
        p.makespan[b] = 0;
        p.status[b] = bad ? 2 : 3;
        acc[0] += 1;
        acc[3] += 1;
      }
      __syncthreads();
      continue;
    }

    // ---- a3: EDF order (d, r, idx)
    if (np2 <= 32) {
      if (warp == 0) {
        unsigned long long x = lane < np2 ? skey[lane] : ~0ull;
        x = warp_bitonic_sort(x, lane);
        if (lane < np2) skey[lane] = x;
      }
    } else {
      for (int k = 2; k <= np2; k <<= 1) {
        for (int j = k >> 1; j > 0; j >>= 1) {
          for (int i = tid; i < np2; i += NT) {
            const int ixj = i ^ j;
            if (ixj > i) {
              const unsigned long long a = skey[i], c = skey[ixj];
              const bool up = (i & k) == 0;
              if ((a > c) == up) {
                skey[i] = c;
                skey[ixj] = a;
              }
            }
          }
          __syncthreads();
        }
      }
    }
    __syncthreads();
    for (int pos = tid; pos < n; pos += NT) {
      const int task = (int)(skey[pos] & 0xFFF);
      const int d = td[task], S = tS[task];
      int K = 0;
      while (K <= S && rowp[task * p.kp + K].x <= d) ++K;  // options with C_k <= d
      int r_next = 0, store_lim = -0x7fffffff;
      if (pos + 1 < n) {
        const int t2 = (int)(skey[pos + 1] & 0xFFF);
        r_next = tr[t2];
        store_lim = td[t2] - rowp[t2 * p.kp].x;  // the next row reads sources <= d' - C'(0)
      }
      const int fast = (K == 0 || rowp[task * p.kp + K - 1].x <= p.pad) ? 1 : 0;
      info[pos] = make_int4(d, r_next, (task << 8) | (fast << 7) | K, store_lim);
    }
    const int ncols = misc[1] + 1;
    {
      const int r0 = n > 0 ? tr[(int)(skey[0] & 0xFFF)] : 0;
      int32_t* buf0 = rowbuf + p.pad;
      for (int t = tid; t < ncols; t += NT) buf0[t] = (t >= r0) ? 0 : NEG;
    }
    __syncthreads();

    // ---- a4: the DP sweep
    int G[COLS];
#pragma unroll
    for (int m = 0; m < COLS; ++m) G[m] = 0;
    for (int pos = 0; pos < n; ++pos) {
      const int4 inf = info[pos];
      const int d = inf.x, r_next = inf.y, task = inf.z >> 8, K = inf.z & 0x7F;
      const bool fast = (inf.z >> 7) & 1;
      const int32_t* cur = rowbuf + (single_buf ? 0 : (pos & 1)) * RS + p.pad;
      int32_t* nxt = rowbuf + (single_buf ? 0 : ((pos + 1) & 1)) * RS + p.pad;
      uint32_t* decrow = dec + (int64_t)pos * NQ * NT;
      const int2* op = rowp + task * p.kp;
      const bool has_next = pos + 1 < n;
      if (fast)
        dp_row_dispatch<NT, COLS, SB>(K, G, p, cur, nxt, decrow, op, d, r_next, inf.w, has_next, ncols);
      else
        dp_row_general<NT, COLS, SB>(K, G, p, cur, nxt, decrow, op, d, r_next, inf.w, has_next, ncols);
      __syncthreads();
    }

    // ---- a5: Q* = G_N(T), t* = least t attaining it
    {
      const int tl = ncols - 1;
#pragma unroll
      for (int m = 0; m < COLS; ++m)
        if (m * NT + tid == tl) misc[3] = n > 0 ? G[m] : 0;
    }
    __syncthreads();
    const int Qp = misc[3];
    {
      int best = 0x7fffffff;
#pragma unroll
      for (int m = COLS - 1; m >= 0; --m) {
        const int t = m * NT + tid;
        if (t < ncols && G[m] == Qp) best = t;
      }
      if (n == 0) best = 0;
      if (best != 0x7fffffff) atomicMin(&misc[2], best);
    }
    __syncthreads();

    // ---- a6/a7: backtrack and the EDF schedule, by one thread
    if (tid == 0) {
      const bool feasible = Qp >= 0;
      int t = misc[2];
      if (feasible) {
        for (int pos = n - 1; pos >= 0; --pos) {
          const int m = t / NT, tt = t - m * NT;
          const uint32_t w = dec[((int64_t)pos * NQ + (m >> 3)) * NT + tt];
          const int code = 15 - (int)((w >> (4 * (m & 7))) & 15u);
          chosen[pos] = code;
          if (code > 0) {
            const int4 inf = info[pos];
            const int task = inf.z >> 8;
            t = min(t, inf.x) - rowp[task * p.kp + code - 1].x;
          }
        }
      }
      int64_t F = 0, Q = 0, conf = 0;
      int ndrop = 0, nopt = 0, noff = 0;
      for (int pos = 0; pos < n; ++pos) {
        const int4 inf = info[pos];
        const int task = inf.z >> 8;
        noff += tS[task];
        const int code = feasible ? chosen[pos] : 0;
        if (code > 0) {
          const int k = code - 1;
          const int2 o = rowp[task * p.kp + k];
          const int64_t s = max(F, (int64_t)tr[task]);
          const int64_t f = s + o.x;
          p.kept[lo + task] = (int8_t)k;
          p.start[lo + task] = (int32_t)s;
          p.finish[lo + task] = (int32_t)f;
          F = f;
          Q += o.y >> 4;
          conf += tR[task * R1 + k];
          nopt += k;
        } else {
          p.kept[lo + task] = -1;
          p.start[lo + task] = -1;
          p.finish[lo + task] = -1;
          ++ndrop;
        }
      }
      p.q_total[b] = Q;
      p.conf_micro[b] = conf;
      p.conf_total[b] = (double)conf / 1e6;
      p.makespan[b] = (int32_t)F;
      p.status[b] = feasible ? 0 : 1;
      acc[0] += 1;
      if (feasible) {
        acc[1] += n;
        acc[2] += ndrop;
        acc[4] += nopt;
        acc[5] += noff;
        acc[6] += conf;
        acc[7] += Q;
      } else {
        acc[3] += 1;
      }
    }
    __syncthreads();
  }
  if (tid == 0 && p.stats) {
#pragma unroll
    for (int s = 0; s < 8; ++s)
      if (acc[s]) atomicAdd(&p.stats[s], acc[s]);
  }
}

}  // namespace icsched

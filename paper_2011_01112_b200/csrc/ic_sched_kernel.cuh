// ic_sched_kernel.cuh — sm_100a kernel for the batched depth assignment.
//
// Persistent grid; a CTA = NW "DP warps" + 1 "tail warp", one instance at a
// time, warp-specialised so the DP warps only ever sweep the table:
//
//   tail warp  a1 descriptor loads + validation, a2 prefix sums C_i(k),
//              R_i(k), Delta (P:L78 / Theorem 1), packed
//              option keys, a3 EDF order (d, r, idx) by warp bitonic
//              sort — all for instance b+1 while the DP warps sweep b;
//              then a6 backtrack of b, a7 EDF schedule times
//              via a warp max-plus scan and the outputs, a8 stats.
//   DP warps   a4 the time-indexed dual of Eqs. 1-2:
//                 G_i(t) = max( G_{i-1}(t) [drop],
//                               max_k G_{i-1}(min(t,d_i) - C_i(k)) + q_i(k) )
//              a5 Q* = G_N(T), t* by a 32-ary search.
//
// Two identities keep the sweep at one shared-memory load per (cell, option):
//   * packed keys: a cell stores Q*16 + 15; option k adds (q_k << 4) - (k+1),
//     so one VIADDMNMX (fused add+max) per option yields value *and* argmax
//     (low nibble = 15 - code; ties resolve to the smaller code, drop first);
//   * tail collapse: EDF rows are sorted by deadline, so for t > d_i every
//     G_i(t) equals one constant M_i = max(M_{i-1}, A_i) with
//     A_i = max_k G_{i-1}(d_i - C_i(k)) + q_i(k).  Only the active columns
//     t <= d_i are swept; (d_i, d_{i+1}] is filled with M_i for the next row,
//     and the tail decision is one nibble per row.
// Threads own columns t = g*NT + tid, so every shifted read t - C_k is
// conflict-free.  Rows are double-buffered, or (H = 32768) updated in place
// chunk by chunk from high to low columns with a barrier per chunk.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <type_traits>

#ifndef IC_SB_CHUNK
#define IC_SB_CHUNK 8
#endif
#ifndef IC_WS_DISCARD
// 1: the warp-specialised kernel's tail warp can discard dead decision lines (tuning.discard);
// compiled out by default: even unexecuted, that code costs the C5 sweep 2 % (same-box A/B)
#define IC_WS_DISCARD 0
#endif
#ifndef IC_DEC_KEEP
#define IC_DEC_KEEP 1
#endif
#ifndef IC_SB_CHUNK15
#define IC_SB_CHUNK15 8  // chunk of the 15-warp in-place kernel (128 registers)
#endif
#ifndef IC_BATCH_KSPLIT
#define IC_BATCH_KSPLIT 6
#endif
#ifndef IC_BATCH_HI
#define IC_BATCH_HI 4
#endif

namespace icsched {

constexpr int NEG = -(1 << 30);
constexpr int INFV = 1 << 30;  // reward axis: unreachable (packed finish time)
constexpr int KMAX = 15;           // options per task: mandatory-only .. 14 optional stages
constexpr int BAR_DP = 1, BAR_READY = 2, BAR_DONE = 3;
constexpr int ST_OK = 0, ST_INFEASIBLE = 1, ST_BAD = 2, ST_LIMIT = 3, ST_END = -1;

struct Params {
  int64_t B;
  const int64_t* task_begin;
  const int32_t *release, *deadline, *mand_wcet;
  const uint8_t* n_opt;
  const int32_t* opt_wcet;
  const uint32_t* mand_conf;
  const int32_t* opt_gain;
  int8_t* kept;
  int32_t *start, *finish;
  int64_t *q_total, *conf_micro;
  double* conf_total;
  int32_t* makespan;
  uint8_t* status;
  unsigned long long* stats;
  uint32_t delta_micro, eps_micro;
  int max_tasks, smax, H;
  int pad, nq, kp, r1, np2;
  int dec_smem;
  uint32_t* dec_global;
  int64_t dec_slab_words;
  int ndec;            // decision buffers: 2 = the backtrack of b overlaps the sweep of b+1
  int64_t dec_words;   // words per decision buffer
  // shared-memory layout (byte offsets); slot arrays are [2][...]
  int off_rowbuf, off_dec, off_rowp, off_info, off_tR, off_task, off_tail, off_misc, off_chosen, off_sd, off_sr,
      off_sS, off_key;
  int nslots;  // 2: set up instance b+1 while the DP sweeps b; 1: serialised (large N)
  int cap;     // row buffer capacity in columns (32 NW x COLS)
  int off_aux, off_sQ;
  int solo_warp_bytes;  // solo kernel: shared-memory bytes of one warp's private region (0: ws kernel)
  int nw;               // DP warps of the warp-specialised kernel
  int axis_mode;  // 0 auto (per instance), 1 time axis only, 2 reward axis whenever eligible
  // NEXT-2 (incremental re-plan): per-instance state = every DP row (its active
  // columns and tail value, stride H+1), the decisions and the tail nibbles
  char* state;
  int64_t state_stride, state_dec_off, state_tail_off;
  int replan;  // 1: re-plan from the changed row (an arrival appended last, or a departure)
  const int32_t *dep_index, *dep_deadline, *dep_release;  // departures: the removed task per instance
  int ckpt;    // rows kept in the state: every ckpt-th (rows ckpt-1, 2 ckpt-1, ...), power of two
  unsigned long long* work;  // [2] dynamic instance counter, CTAs finished (reset by the last CTA)
  // hybrid solves (fixed Delta, long horizon): the solo kernel runs the instances whose sweep
  // fits its short row and lists the others in defer_ids; the warp-specialised kernel then
  // solves exactly the listed ids (ids / nids non-null)
  int64_t* defer_ids;
  unsigned long long* defer_n;
  const int64_t* ids;
  const unsigned long long* nids;
  int rowbuf_stride;  // ints per row buffer (pad + capacity)
  // large task sets: the tail warp's option tables of both slots live in a per-CTA global
  // (L2) slab and the DP warps copy the current one into their single shared-memory table
  int2* rowp_g;
  int64_t rowp_slab;  // int2 per CTA slab ([2][max_tasks][kp])
  int opt_vec4;       // optional-stage rows are 16-byte aligned multiples of 4: LDG.128 loads
  int discard;        // invalidate an instance's decision lines in L2 after its backtrack
};

__device__ __forceinline__ int32_t* state_rows(const Params& p, int64_t b) {
  return (int32_t*)(p.state + b * p.state_stride);
}
__device__ __forceinline__ uint32_t* state_dec(const Params& p, int64_t b) {
  return (uint32_t*)(p.state + b * p.state_stride + p.state_dec_off);
}
__device__ __forceinline__ int32_t* state_tail(const Params& p, int64_t b) {
  return (int32_t*)(p.state + b * p.state_stride + p.state_tail_off);
}

__device__ __forceinline__ void bar_sync(int id, int n) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ void bar_arrive(int id, int n) {
  asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory");
}
__device__ __forceinline__ int viaddmax(int a, int b, int c) { return __viaddmax_s32(a, b, c); }
// Shared-memory load at a 32-bit shared address.  The double-buffered sweep addresses its row
// through one opaque shared base per row (cvta below) so the window base is not re-derived
// (S2UR) at the head of every chunk's address chain; ptxas folds the constant cell offsets
// into the LDS immediates.  Volatile: never merged across the row barriers.
__device__ __forceinline__ int lds32(uint32_t a) {
  int v;
  asm volatile("ld.shared.b32 %0, [%1];" : "=r"(v) : "r"(a));
  return v;
}
__device__ __forceinline__ void sts32(uint32_t a, int v) {
  asm volatile("st.shared.b32 [%0], %1;" ::"r"(a), "r"(v));
}
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  uint32_t a;
  asm volatile("{ .reg .u64 t; cvta.to.shared.u64 t, %1; cvt.u32.u64 %0, t; }" : "=r"(a) : "l"(p));
  return a;
}
// Decision words are re-read by the backtrack microseconds later and then dead: they are
// stored under an L2 evict_last policy (the policy descriptor is a compile-time constant, no
// instruction) so the streaming descriptor and output traffic is evicted before them
// (C5: +0.2 % throughput and 18 % fewer DRAM writes than plain stores; with the discard below,
// DRAM traffic 1.1x the algorithmic bytes).  IC_DEC_KEEP=0 builds plain stores (A/B).
__device__ __forceinline__ void st_dec(uint32_t* a, uint32_t v, bool dglob) {
#if IC_DEC_KEEP
  // dglob: the launch keeps decisions in global memory (tuning.decisions = 1 puts them in shared
  // memory: a plain store).  A uniform kernel-parameter test, not a per-store __isGlobal (QSPC),
  // which cost the C5 sweep 2 %.
  if (dglob) {
    unsigned long long pol;
    asm("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
    asm volatile("st.global.L2::cache_hint.b32 [%0], %1, %2;" ::"l"(a), "r"(v), "l"(pol) : "memory");
  } else {
    *a = v;
  }
#else
  *a = v;
#endif
}
// the least column t >= first that thread tid owns (t = tid mod NT; NT need not be a power of 2)
template <int NT>
__device__ __forceinline__ int first_col(int first, int tid) {
  if constexpr ((NT & (NT - 1)) == 0) return first + ((tid - first) & (NT - 1));
  int m = (tid - first) % NT;
  return first + (m < 0 ? m + NT : m);
}

// Packed option entries (the solo kernel at a fixed Delta, PK): one 32-bit word per option
// instead of an int2, two 16-bit fields.  Time axis: shift C (low, unsigned) and key
// (q << 4) - (k+1) (high, signed); reward axis: addend C*16 + k+1 (low, unsigned) and shift q
// (high).  The host enables it only when every field fits (q <= 2047, C <= 4095).
// The int2 form is (shift, addend) on both axes.
__device__ __forceinline__ int2 pk_get(int e, bool rw) {
  const int lo = e & 0xFFFF, hi = e >> 16;
  return rw ? make_int2(hi, lo) : make_int2(lo, hi);
}
__device__ __forceinline__ int pk_put(int2 v, bool rw) {
  return rw ? (int)((unsigned)(v.y & 0xFFFF) | ((unsigned)v.x << 16)) : (int)((unsigned)(v.x & 0xFFFF) | ((unsigned)v.y << 16));
}
template <bool PK>
__device__ __forceinline__ int2 opt_get(const int2* tab, size_t idx, bool rw) {
  if constexpr (PK) return pk_get(((const int*)tab)[idx], rw);
  return tab[idx];
}
template <bool PK>
__device__ __forceinline__ void opt_put(int2* tab, size_t idx, int2 v, bool rw) {
  if constexpr (PK)
    ((int*)tab)[idx] = pk_put(v, rw);
  else
    tab[idx] = v;
}

// ---------------------------------------------------------------------------
// DP warps: one row, active columns t <= d.  K options (compile-time), or GEN = the
// general path with runtime kr options, per-option release masks, and sources left of
// the pad redirected to the pad cell at -1 (rows with releases, or whose longest option
// reaches past the pad: the tail warp flags them, so the common rows carry no bounds code).
// RW = the reward-indexed axis (NEXT-1, the paper's own Eqs. 1-2): a cell holds the
// least finish time P(i, r)*16 of the first i EDF tasks reaching exactly quantised
// reward r; option k shifts by q_k and adds C_k*16 + (k+1) (the code), so one
// VIADDMNMX (add + min) per option yields value and argmin, ties to the smaller
// code (drop, then fewer stages).  Admits are valid iff P <= d_i ("lim").
template <int NW, bool SB, bool DROP, int K, bool GEN, bool RW, bool PK = false>
__device__ __forceinline__ void dp_row(const int32_t* cur, int32_t* nxt, uint32_t* __restrict__ decrow,
                                       const int4* __restrict__ ops4, const int4 (&pre)[4], const int d,
                                       const int r, const int kr, const int lim, const bool dglob) {
  constexpr int NT = 32 * NW;
  // the solo kernel's general path loops over the options at run time, reading each from
  // shared memory (no option registers: it keeps the row loop's registers from spilling)
  constexpr bool RTK = GEN && SB && NW == 1;
  constexpr int KK = RTK ? 0 : GEN ? KMAX : K;
  // one-warp rows are swept by warp 0 of the warp-specialised kernel or by any warp of the
  // solo kernel: the lane is the thread's column offset there
  // the thread index through an opaque read: kept in a register for the whole row instead of
  // re-read (S2R) at the head of every chunk's address chain under register pressure
  int tix;
  asm volatile("mov.u32 %0, %%tid.x;" : "=r"(tix));
  const int tid = NW == 1 ? (tix & 31) : tix, warp = NW == 1 ? 0 : tid >> 5;
  int C[KK > 0 ? KK : 1], key[KK > 0 ? KK : 1];
  if constexpr (PK) {  // 16 packed entries were loaded before the dispatch
#pragma unroll
    for (int k = 0; k < KK; ++k) {
      if (!GEN || k < kr) {
        const int4 o = pre[k >> 2];
        const int2 e = pk_get((k & 3) == 0 ? o.x : (k & 3) == 1 ? o.y : (k & 3) == 2 ? o.z : o.w, RW);
        C[k] = e.x;
        key[k] = e.y;
      }
    }
  } else {
#pragma unroll
    for (int k = 0; k < KK; k += 2) {
      if (!GEN || k < kr) {
        const int4 o = k < 8 ? pre[k >> 1] : ops4[k >> 1];  // the first 8 were loaded before the dispatch
        C[k] = o.x;
        key[k] = o.y;
        if (k + 1 < KK) {
          C[k + 1] = o.z;
          key[k + 1] = o.w;
        }
      }
    }
  }
  const int w0 = warp * 32;
  const int ng = d >= w0 ? (d - w0) / NT + 1 : 0;  // this warp's groups holding a column t <= d
  auto cell = [&](int t) -> int {
    if constexpr (RTK) {
      const int2* o2 = (const int2*)ops4;
      if constexpr (RW) {
        int a = INFV;
#pragma unroll 1
        for (int k = 0; k < kr; ++k) {
          const int2 o = opt_get<PK>(o2, k, RW);
          a = __viaddmin_s32(cur[max(t - o.x, -1)], o.y, a);
        }
        a = a <= lim ? a : INFV;
        return DROP ? min(cur[t], a) : a;
      } else {
        int v = DROP ? cur[t] : NEG;
#pragma unroll 1
        for (int k = 0; k < kr; ++k) {
          const int2 o = opt_get<PK>(o2, k, RW);
          const int src = t - o.x;
          v = viaddmax(cur[src >= r ? src : -1], o.y, v);
        }
        return v;
      }
    } else if constexpr (RW) {
      int a = INFV;
#pragma unroll
      for (int k = 0; k < KK; ++k) {
        if (!GEN || k < kr) a = __viaddmin_s32(cur[GEN ? max(t - C[k], -1) : t - C[k]], key[k], a);
      }
      a = a <= lim ? a : INFV;
      return DROP ? min(cur[t], a) : a;
    } else {
      int v = DROP ? cur[t] : NEG;
#pragma unroll
      for (int k = 0; k < KK; ++k) {
        if (GEN) {  // sources before the release (or left of the pad) read the NEG pad cell at -1
          if (k < kr) {
            const int src = t - C[k];
            v = viaddmax(cur[src >= r ? src : -1], key[k], v);
          }
        } else {
          v = viaddmax(cur[t - C[k]], key[k], v);
        }
      }
      return v;
    }
  };
  // stored value: time axis keeps low nibble 15 (the drop key), reward axis keeps it 0
  auto stv = [](int v) { return RW ? (v & ~15) : (v | 15); };
  if constexpr (!SB) {
    constexpr int BATCH = (KK <= IC_BATCH_KSPLIT) ? 8 : IC_BATCH_HI;  // cells whose loads are in flight together
    // full chunks of the common rows (no bounds): loads through the row's opaque shared base
    const uint32_t cs = smem_addr(cur), ns = smem_addr(nxt);
    auto cell_s = [&](int t) -> int {
      const uint32_t at = cs + 4u * (uint32_t)t;
      if constexpr (RW) {
        int a = INFV;
#pragma unroll
        for (int k = 0; k < KK; ++k) a = __viaddmin_s32(lds32(at - 4u * (uint32_t)C[k]), key[k], a);
        a = a <= lim ? a : INFV;
        return DROP ? min(lds32(at), a) : a;
      } else {
        int v = DROP ? lds32(at) : NEG;
#pragma unroll
        for (int k = 0; k < KK; ++k) v = viaddmax(lds32(at - 4u * (uint32_t)C[k]), key[k], v);
        return v;
      }
    };
    auto cellx = [&](int t) -> int {
      if constexpr (GEN)
        return cell(t);
      else
        return cell_s(t);
    };
    auto store = [&](int t, int v) {
      if constexpr (GEN)
        nxt[t] = stv(v);
      else
        sts32(ns + 4u * (uint32_t)t, stv(v));
    };
    for (int g0 = 0; g0 < ng; g0 += 8) {
      const int tb = g0 * NT + tid;
      uint32_t dw = 0;
      if (g0 + 8 <= ng) {
#pragma unroll
        for (int h = 0; h < 8; h += BATCH) {
          int v[BATCH];
#pragma unroll
          for (int u = 0; u < BATCH; ++u) v[u] = cellx(tb + (h + u) * NT);
#pragma unroll
          for (int u = 0; u < BATCH; ++u) {
            dw |= (uint32_t)(v[u] & 15) << (4 * (h + u));
            store(tb + (h + u) * NT, v[u]);
          }
        }
      } else {
        // ragged last chunk: 4 + 2 + 1 groups, each sub-batch issuing its loads together
        const int rem = ng - g0;
        int u0 = 0;
        auto sub = [&](auto nb_tag) {
          constexpr int NB = decltype(nb_tag)::value;
          int v[NB];
#pragma unroll
          for (int u = 0; u < NB; ++u) v[u] = cellx(tb + (u0 + u) * NT);
#pragma unroll
          for (int u = 0; u < NB; ++u) {
            dw |= (uint32_t)(v[u] & 15) << (4 * (u0 + u));
            store(tb + (u0 + u) * NT, v[u]);
          }
          u0 += NB;
        };
        if (rem & 4) sub(std::integral_constant<int, 4>{});
        if (rem & 2) sub(std::integral_constant<int, 2>{});
        if (rem & 1) sub(std::integral_constant<int, 1>{});
      }
      st_dec(&decrow[(g0 >> 3) * NT + tid], dw, dglob);
    }
  } else if constexpr (NW == 1) {
    // one warp per instance (the solo kernel), in place from high to low columns: blocks of
    // NB consecutive groups, each loads -> __syncwarp -> stores.  A block reads only columns
    // below its top, so its stores cannot disturb a lower block still to be computed.  The
    // ragged top chunk goes first as blocks of 1, 2 and 4 groups (highest first), then full
    // chunks of 8 groups (two blocks of 4 when K is large, to bound the values in flight).
    auto blk = [&](int g, auto nb_tag) -> uint32_t {
      constexpr int NB = decltype(nb_tag)::value;
      const int tb = g * NT + tid;
      int v[NB];
#pragma unroll
      for (int u = 0; u < NB; ++u) v[u] = cell(tb + u * NT);
      __syncwarp();
      uint32_t dw = 0;
#pragma unroll
      for (int u = 0; u < NB; ++u) {
        dw |= (uint32_t)(v[u] & 15) << (4 * (u + (g & 7)));
        nxt[tb + u * NT] = stv(v[u]);
      }
      return dw;
    };
    using I1 = std::integral_constant<int, 1>;
    using I2 = std::integral_constant<int, 2>;
    using I4 = std::integral_constant<int, 4>;
    using I8 = std::integral_constant<int, 8>;
    const int gtop = ng & ~7, rem = ng - gtop;
    if (rem) {
      uint32_t dw = 0;
      if (rem & 1) dw |= blk(gtop + (rem & 6), I1{});
      if (rem & 2) dw |= blk(gtop + (rem & 4), I2{});
      if (rem & 4) dw |= blk(gtop, I4{});
      st_dec(&decrow[(gtop >> 3) * NT + tid], dw, dglob);
    }
#pragma unroll 1
    for (int g0 = gtop - 8; g0 >= 0; g0 -= 8) {
      uint32_t dw;
      if constexpr (KK <= IC_BATCH_KSPLIT) {
        dw = blk(g0, I8{});
      } else {
        dw = blk(g0 + 4, I4{});
        dw |= blk(g0, I4{});
      }
      st_dec(&decrow[(g0 >> 3) * NT + tid], dw, dglob);
    }
  } else {
    // in place, chunks of 8 groups from high to low columns, one barrier per chunk:
    // chunk c reads only columns below its top, so writing it after the barrier
    // cannot disturb a lower chunk still to be computed.
    constexpr int CH = NW == 15 ? IC_SB_CHUNK15 : IC_SB_CHUNK;  // groups per chunk (a multiple of 8: one decision word per 8)
    const int nch = d >= 0 ? (d / NT) / CH + 1 : 0;  // CTA-uniform chunk count (warp 0 has the most groups)
    for (int c = nch - 1; c >= 0; --c) {
      const int g0 = c * CH;
      const int tb = g0 * NT + tid;
      int v[CH];
      if (g0 + CH <= ng) {
        // a full chunk (every chunk but this warp's top one): no per-cell predicates, so the
        // loads of all CH cells share one address per option (immediate offsets u * NT)
#pragma unroll
        for (int u = 0; u < CH; ++u) v[u] = cell(tb + u * NT);
        bar_sync(BAR_DP, NT);
#pragma unroll
        for (int w8 = 0; w8 < CH; w8 += 8) {
          uint32_t dw = 0;
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            dw |= (uint32_t)(v[w8 + u] & 15) << (4 * u);
            nxt[tb + (w8 + u) * NT] = stv(v[w8 + u]);
          }
          st_dec(&decrow[((g0 + w8) >> 3) * NT + tid], dw, dglob);
        }
      } else {
#pragma unroll
        for (int u = 0; u < CH; ++u) v[u] = (g0 + u < ng) ? cell(tb + u * NT) : 0;
        bar_sync(BAR_DP, NT);
#pragma unroll
        for (int w8 = 0; w8 < CH; w8 += 8) {
          uint32_t dw = 0;
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            if (g0 + w8 + u < ng) {
              dw |= (uint32_t)(v[w8 + u] & 15) << (4 * u);
              nxt[tb + (w8 + u) * NT] = stv(v[w8 + u]);
            }
          }
          if (g0 + w8 < ng) st_dec(&decrow[((g0 + w8) >> 3) * NT + tid], dw, dglob);
        }
      }
    }
  }
}

// gen: the row takes the general path (releases, or an option longer than the pad).
// KC: the largest option count with its own unrolled sweep; rows with more take the
// general path (the solo kernel compiles K <= 9, i.e. up to 8 optional stages).
template <int NW, bool SB, bool DROP, bool RW, int KC = 15, bool PK = false>
__device__ __forceinline__ void dp_row_dispatch(int K, bool gen, const int32_t* cur, int32_t* nxt,
                                                uint32_t* decrow, const int4* ops4, int d, int r, int lim,
                                                bool dglob = true) {
  const int4 pre[4] = {ops4[0], ops4[1], ops4[2], ops4[3]};  // issued ahead of the K dispatch
  if (gen || K > KC) {
    dp_row<NW, SB, DROP, KMAX, true, RW, PK>(cur, nxt, decrow, ops4, pre, d, r, K, lim, dglob);
    return;
  }
#define IC_ROW(KK) \
  case KK: if constexpr (KK <= KC) dp_row<NW, SB, DROP, KK, false, RW, PK>(cur, nxt, decrow, ops4, pre, d, r, K, lim, dglob); break;
  switch (K) {
    IC_ROW(0) IC_ROW(1) IC_ROW(2) IC_ROW(3) IC_ROW(4) IC_ROW(5) IC_ROW(6) IC_ROW(7)
    IC_ROW(8) IC_ROW(9) IC_ROW(10) IC_ROW(11) IC_ROW(12) IC_ROW(13) IC_ROW(14) IC_ROW(15)
    default: break;
  }
#undef IC_ROW
}

// ---------------------------------------------------------------------------
// Tail warp helpers.
__device__ __forceinline__ unsigned long long warp_bitonic_sort(unsigned long long x, int lane) {
#pragma unroll
  for (int k = 2; k <= 32; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      const unsigned long long y = __shfl_xor_sync(0xffffffffu, x, j);
      const bool up = ((lane & k) == 0);
      const bool lower = ((lane & j) == 0);
      x = (lower == up) ? (x < y ? x : y) : (x < y ? y : x);
    }
  }
  return x;
}

// Ascending sort of key[0..n) by one warp (the EDF order, keys (d, r, index)): in registers
// for n <= 64 (one or two keys per lane, bitonic network over shuffles), else a bitonic
// network over shared memory (key must hold the next power of two >= n entries).
__device__ __forceinline__ void warp_sort_keys(unsigned long long* key, int n, int lane) {
  int np2 = 1;
  while (np2 < n) np2 <<= 1;
  if (np2 <= 32) {
    unsigned long long x = lane < n ? key[lane] : ~0ull;
    x = warp_bitonic_sort(x, lane);
    if (lane < n) key[lane] = x;
  } else if (np2 == 64) {  // two keys per lane (positions lane, lane + 32), in registers
    unsigned long long x0 = key[lane], x1 = lane + 32 < n ? key[lane + 32] : ~0ull;
#pragma unroll
    for (int k = 2; k <= 64; k <<= 1) {
#pragma unroll
      for (int j = k >> 1; j > 0; j >>= 1) {
        if (j == 32) {  // k = 64: partners lane and lane + 32, ascending
          const unsigned long long lo2 = x0 < x1 ? x0 : x1;
          x1 = x0 < x1 ? x1 : x0;
          x0 = lo2;
        } else {
          const unsigned long long y0 = __shfl_xor_sync(0xffffffffu, x0, j);
          const unsigned long long y1 = __shfl_xor_sync(0xffffffffu, x1, j);
          const bool lower = (lane & j) == 0;
          const bool up0 = (lane & k) == 0, up1 = ((lane + 32) & k) == 0;
          x0 = (lower == up0) ? (x0 < y0 ? x0 : y0) : (x0 < y0 ? y0 : x0);
          x1 = (lower == up1) ? (x1 < y1 ? x1 : y1) : (x1 < y1 ? y1 : x1);
        }
      }
    }
    key[lane] = x0;
    if (lane + 32 < n) key[lane + 32] = x1;
  } else {
    for (int i = n + lane; i < np2; i += 32) key[i] = ~0ull;
    __syncwarp();
    for (int k = 2; k <= np2; k <<= 1) {
      for (int j = k >> 1; j > 0; j >>= 1) {
        for (int i = lane; i < np2; i += 32) {
          const int ixj = i ^ j;
          if (ixj > i) {
            const unsigned long long a = key[i], c = key[ixj];
            if ((a > c) == ((i & k) == 0)) {
              key[i] = c;
              key[ixj] = a;
            }
          }
        }
        __syncwarp();
      }
    }
  }
  __syncwarp();
}

__device__ __forceinline__ long long warp_sum64(long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

struct Smem {
  int32_t* rowbuf;
  uint32_t* dec;
  int2* rowp;    // [2][max_tasks][kp]  (C_k, key_k) of EDF row pos; reward axis: (q_k, C_k*16 + k+1)
                 //   ([1][...] when the tables live in global memory: the DP's copy)
  int4* info;    // [2][max_tasks]      (d, K | gen<<8 | S<<16, r, d_next)
  int32_t* task; // [2][max_tasks]      input index of EDF row pos
  int32_t* tail; // [2][max_tasks]      tail nibble of row pos
  long long* misc;  // [2][16]
  int32_t* chosen;  // [max_tasks]
  int32_t *sd, *sr, *sS;  // staging (input order), tail warp only
  int32_t* aux;  // [2][max_tasks]  reward axis: admit limit d_i*16+15 of EDF row pos
  int32_t* sQ;   // [max_tasks]     staging: prefix of max quantised reward
  unsigned long long* key;
};

// Global option tables are compiled only into the wide kernels (NW >= 8: the large task
// sets that need them), so the small kernels keep their register budget.
template <int NW>
__device__ __forceinline__ bool rowp_global(const Params& p) {
  if constexpr (NW >= 8) return p.rowp_g != nullptr;
  return false;
}
// The tail warp's option table of slot s: shared memory, or the CTA's global slab.
template <int NW>
__device__ __forceinline__ int2* rowp_slot(const Params& p, const Smem& S, int s) {
  return rowp_global<NW>(p) ? p.rowp_g + (int64_t)blockIdx.x * p.rowp_slab + (int64_t)s * p.max_tasks * p.kp
                            : S.rowp + (size_t)s * p.max_tasks * p.kp;
}

// Write the "everything dropped" outputs of an instance that the DP never sees.
__device__ __forceinline__ void write_dropped(const Params& p, int64_t b, int64_t lo, int64_t n, int status,
                                              int lane) {
  for (int64_t i = lane; i < n; i += 32) {
    p.kept[lo + i] = -1;
    p.start[lo + i] = -1;
    p.finish[lo + i] = -1;
  }
  if (lane == 0) {
    p.q_total[b] = 0;
    p.conf_micro[b] = 0;
    p.conf_total[b] = 0.0;
    p.makespan[b] = 0;
    p.status[b] = (uint8_t)status;
  }
}

// Visit task t's optional stages k = 1..Sn with (wcet, gain), loading them in
// batches of 4 (the tail warp's register budget is small): one 128-bit load per
// array and batch when the rows allow it (lane-per-task: a warp reads 32 whole
// consecutive rows, so every sector fetched is used), else 4 scalar loads.
template <typename F>
__device__ __forceinline__ void for_each_opt(const Params& p, int64_t t, int Sn, F&& f) {
  for (int k0 = 0; k0 < Sn; k0 += 4) {
    int w[4], g[4];
    if (p.opt_vec4) {  // k0 + 3 < smax: the load stays inside task t's row
      const int4 w4 = *(const int4*)(p.opt_wcet + t * p.smax + k0);
      const int4 g4 = *(const int4*)(p.opt_gain + t * p.smax + k0);
      w[0] = w4.x; w[1] = w4.y; w[2] = w4.z; w[3] = w4.w;
      g[0] = g4.x; g[1] = g4.y; g[2] = g4.z; g[3] = g4.w;
    } else {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        if (k0 + u < Sn) {
          w[u] = p.opt_wcet[t * p.smax + k0 + u];
          g[u] = p.opt_gain[t * p.smax + k0 + u];
        }
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (k0 + u < Sn) f(k0 + u + 1, w[u], g[u]);
  }
}

// a1-a3 for instance b into slot s.  Returns ST_OK if the DP must run it;
// otherwise the outputs are already written (bad input, limit, empty set).
// Pass 1 (input order): validation, the best individually feasible reward
// (Theorem 1's R), the EDF keys.  Pass 2 (EDF order, descriptors re-read):
// prefix sums, q = R div Delta, packed keys, the row table of the DP.
template <int NW, bool PK = false>
__device__ int tail_setup(const Params& p, const Smem& S, int64_t b, int s, int lane,
                          unsigned long long* acc) {
  const int64_t lo = p.task_begin[b];
  const int64_t n64 = p.task_begin[b + 1] - lo;
  if (n64 < 0 || n64 > p.max_tasks) {
    write_dropped(p, b, lo, n64 > 0 ? n64 : 0, ST_BAD, lane);
    if (lane == 0) { acc[0] += 1; acc[3] += 1; }
    return ST_BAD;
  }
  const int n = (int)n64;
  if (n == 0) {
    write_dropped(p, b, lo, 0, ST_OK, lane);
    if (lane == 0) acc[0] += 1;
    return ST_BAD + 100;  // handled (empty task set: Q = 0, status OK)
  }
  int bad = 0, rmax = 0;
  for (int i = lane; i < n; i += 32) {
    const int64_t t = lo + i;
    const int r = p.release[t], d = p.deadline[t], m = p.mand_wcet[t];
    const int Sn = p.n_opt[t];
    const uint32_t a0 = p.mand_conf[t];
    int tb = (Sn > p.smax) | (r < 0) | (d >= p.H) | (m < 1) | (a0 > 1000000u);
    S.sd[i] = d;
    S.sr[i] = r;
    S.sS[i] = Sn;
    if (!tb) {
      long long C = m, R = a0;
      if ((long long)r + C <= d && R > rmax) rmax = (int)R;
      for_each_opt(p, t, Sn, [&](int, int w, int g) {
        tb |= (w < 1);
        C += w;
        R += g;
        tb |= (R < 0) | (R > 1000000);
        if ((long long)r + C <= d && R > rmax) rmax = (int)R;
      });
    }
    bad |= tb;
    const uint32_t dk = (uint32_t)d ^ 0x80000000u;
    const uint32_t rk = (uint32_t)min(max(r, 0), (1 << 20) - 1);
    S.key[i] = ((unsigned long long)dk << 32) | ((unsigned long long)rk << 12) | (unsigned)i;
  }
  bad = __any_sync(0xffffffffu, bad);
  if (bad) {
    write_dropped(p, b, lo, n, ST_BAD, lane);
    if (lane == 0) { acc[0] += 1; acc[3] += 1; }
    return ST_BAD;
  }
  rmax = __reduce_max_sync(0xffffffffu, rmax);
  long long delta = p.delta_micro;
  if (delta == 0) {
    delta = ((long long)p.eps_micro * rmax) / (1000000LL * n);
    if (delta < 1) delta = 1;
  }
  // a3: EDF order
  warp_sort_keys(S.key, n, lane);
  __syncwarp();
  // pass 2: the row table in EDF order (32 rows at a time, prefix of max q by warp scan)
  long long qsum = 0, wt = 0, wr = 0;
  int anyrel = 0, qcarry = 0;
  for (int base = 0; base < n; base += 32) {
    const int pos = base + lane;
    int qmax = 0, K = 0, d = 0;
    if (pos < n) {
      const int tk = (int)(S.key[pos] & 0xFFF);
      const int64_t t = lo + tk;
      d = S.sd[tk];
      const int r = S.sr[tk], Sn = S.sS[tk];
      int2* rp = rowp_slot<NW>(p, S, s);
      const size_t r0 = (size_t)pos * p.kp;
      long long C = p.mand_wcet[t], R = p.mand_conf[t];
      int Clast = 0;
      auto option = [&](int k) {
        if (C <= (long long)d - r) {  // options that can fit (C increasing in k); only they
          // q = R div Delta in 32 bits: pass 1 bounds every prefix R to [0, 1e6] and
          // 1 <= Delta < 2^32 (a 64-bit division is a called subroutine, 5 per option)
          const int q = (int)((uint32_t)R / (uint32_t)delta);  // bound the packed keys and the reward columns
          qmax = max(qmax, q);
          opt_put<PK>(rp, r0 + k, make_int2((int)C, (q << 4) - (k + 1)), false);
          Clast = (int)C;
          K = k + 1;
        }
      };
      option(0);
      for_each_opt(p, t, Sn, [&](int k, int w, int g) {
        C += w;
        R += g;
        option(k);
      });
      // the general path: releases, or (per axis) an option reaching past the pad
      const bool gen = r > 0 || (K > 0 && Clast > p.pad);
      const bool genr = qmax > p.pad;
      anyrel |= r > 0;
      const int dn = pos + 1 < n ? S.sd[(int)(S.key[pos + 1] & 0xFFF)] : INT32_MIN;
      S.info[s * p.max_tasks + pos] = make_int4(d, K | (gen ? 256 : 0) | (genr ? 512 : 0) | (Sn << 16), r, dn);
      S.task[s * p.max_tasks + pos] = tk;
      S.aux[s * p.max_tasks + pos] = d * 16 + 15;
    }
    qsum += qmax;
    int inc = qmax;  // inclusive scan: Qpre(pos) = sum of max q over EDF rows <= pos
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += y;
    }
    const int qpre = qcarry + inc;
    if (pos < n) {
      S.sQ[pos] = qpre;
      wt += (long long)max(d + 1, 0) * (K + 1);  // active cells x options, both axes
      wr += (long long)(qpre + 1) * (K + 1);
    }
    qcarry = __shfl_sync(0xffffffffu, qpre, 31);
  }
  qsum = warp_sum64(qsum);
  wt = warp_sum64(wt);
  wr = warp_sum64(wr);
  anyrel = __any_sync(0xffffffffu, anyrel);
  if (qsum * 16 + 16LL * n >= (1LL << 30)) {
    write_dropped(p, b, lo, n, ST_LIMIT, lane);
    if (lane == 0) { acc[0] += 1; acc[3] += 1; }
    return ST_LIMIT;
  }
  __syncwarp();
  // a4 axis: the paper's reward-indexed table (Eqs. 1-2) when it is the smaller sweep
  // (e.g. Delta = 0.1), else its time-indexed dual.  Releases need the
  // budget-tracked backtrack, so they stay on the time axis.
  const bool rw = p.axis_mode != 1 && !anyrel && qcarry + 1 <= p.cap && (!p.state || qcarry < p.H) &&
                 (p.axis_mode == 2 || wr < wt);
  if (!rw && p.defer_ids && S.info[s * p.max_tasks + n - 1].x >= p.cap) {
    // the time axis does not fit this kernel's row (the solo kernel sized for the reward
    // axis): hand the instance to the warp-specialised kernel's second launch
    if (lane == 0) p.defer_ids[atomicAdd(p.defer_n, 1ull)] = b;
    __syncwarp();
    return ST_BAD + 200;
  }
  if (rw) {
    for (int pos = lane; pos < n; pos += 32) {
      int4* f = S.info + s * p.max_tasks + pos;
      f->x = S.sQ[pos];
      f->w = pos + 1 < n ? S.sQ[pos + 1] : INT32_MIN;
      // option table in the reward-axis form, once per row here rather than per row and
      // thread in the sweep: (C, (q << 4) - (k+1)) -> (q, C*16 + k+1)
      int2* rp = rowp_slot<NW>(p, S, s);
      const size_t r0 = (size_t)pos * p.kp;
      const int K = f->y & 255;
      for (int k = 0; k < K; ++k) {
        const int2 o = opt_get<PK>(rp, r0 + k, false);
        opt_put<PK>(rp, r0 + k, make_int2((o.y + k + 1) >> 4, min(o.x, 1 << 20) * 16 + (k + 1)), true);
      }
    }
  }
  __syncwarp();
  if (lane == 0) {
    long long* mi = S.misc + s * 16;
    mi[0] = n;
    mi[1] = lo;
    mi[2] = b;
    mi[3] = ST_OK;
    mi[4] = delta;
    mi[7] = S.info[s * p.max_tasks].x;
    mi[8] = S.info[s * p.max_tasks + n - 1].x;
    mi[9] = rw ? 1 : 0;
    mi[10] = 0;
  }
  if (p.replan) {  // rows before the changed EDF position stand (Alg. 1 from row k)
    int k = 0;
    if (p.dep_index) {
      // departure: the removed task j (input index in the previous instance, whose other tasks
      // keep their order) sat after exactly the remaining tasks that precede it in (d, r, index)
      const int j = p.dep_index[b], dj = p.dep_deadline[b], rj = min(max(p.dep_release[b], 0), (1 << 20) - 1);
      for (int i = lane; i < n; i += 32) {
        const int di = S.sd[i], ri = min(max(S.sr[i], 0), (1 << 20) - 1);
        k += (di < dj) || (di == dj && (ri < rj || (ri == rj && i < j)));
      }
      k = (int)__reduce_add_sync(0xffffffffu, (unsigned)k);
    } else {  // arrival: the instance's last task
      for (int pos = lane; pos < n; pos += 32)
        if ((int)(S.key[pos] & 0xFFF) == n - 1) k = pos;
      k = __reduce_max_sync(0xffffffffu, k);
    }
    k = min(k, n - 1);        // a departure past the last row still recomputes the last row
    k = k / p.ckpt * p.ckpt;  // restart after the last checkpointed row before the change
    const int32_t* st = state_tail(p, b);
    if (st[p.max_tasks] != (rw ? 1 : 0)) k = 0;  // the sweep axis changed: nothing to reuse
    if (S.tail)
      for (int pos = lane; pos < k; pos += 32) S.tail[s * p.max_tasks + pos] = st[pos];
    if (lane == 0) S.misc[s * 16 + 10] = k;
    // the backtrack will walk the kept rows' decisions (written by an earlier call, likely
    // evicted to HBM): pull their lines into L2 now so they arrive while the rows >= k sweep
    const int NTs = p.solo_warp_bytes ? 32 : 32 * p.nw;
    const char* db = (const char*)state_dec(p, b);
    for (int pos = lane; pos < k; pos += 32) {
      const int cols = S.info[s * p.max_tasks + pos].x + 1;
      const int lines = cols > 0 ? (((cols - 1) / NTs) / 8 + 1) * (NTs / 32) : 0;
      const char* row = db + (int64_t)pos * p.nq * NTs * 4;
      for (int l = 0; l < lines; ++l) asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(row + l * 128));
    }
  }
  __syncwarp();
  return ST_OK;
}

// a6: backtrack from (Q*, t*) through the decision nibbles (one lane).
// SOLO: the solo kernel keeps no tail nibbles; a column past a row's deadline takes the
// decision of the deadline column itself (every G_i(t), t > d_i, equals G_i(d_i) with the
// same argmax: the options read G_{i-1}(d_i - C_k) and the drop reads M_{i-1} there).
template <int NW, bool SOLO = false, bool PK = false>
__device__ __forceinline__ void tail_backtrack(const Params& p, const Smem& S, int s, int lane, int db) {
  constexpr int NT = 32 * NW;
  const long long* mi = S.misc + s * 16;
  const int n = (int)mi[0];
  if (mi[5] >= 0) {
    // Two rows per decision-word latency: while lane 31 fetches row pos's nibble at t,
    // lanes 0..K_pos fetch row pos-1's nibble at every column its code could lead to
    // (lane c: code c, 0 = drop); the true one is picked by a shuffle once row pos is
    // decoded.  The chain of dependent (L2/HBM) loads halves; the result is unchanged.
    int t = (int)mi[6];
    const int4* inf = S.info + s * p.max_tasks;
    const int2* rp = rowp_slot<NW>(p, S, s);
    const bool rw = mi[9] != 0;
    const uint32_t* dbase = p.state ? state_dec(p, mi[2]) : S.dec + db * p.dec_words;
    const int32_t* tailn = S.tail + s * p.max_tasks;
    // column the decision of code c at row `pos` (column t) leads to in row pos-1
    auto step = [&](int pos, int tt, int code) -> int {
      if (code == 0) return tt;
      const int sh = opt_get<PK>(rp, (size_t)pos * p.kp + code - 1, rw).x;  // time axis: C; reward axis: q
      return rw ? tt - sh : min(tt, inf[pos].x) - sh;
    };
    auto nibble = [&](int row, int tt) -> int {
      if (!rw && tt > inf[row].x) {  // past the deadline
        if constexpr (SOLO) {
          if (inf[row].x < 0) return 15;  // no active column: the task is dropped
          tt = inf[row].x;
        } else {
          return tailn[row];  // the row's tail nibble
        }
      }
      const int g = tt / NT, l = tt - g * NT;
      const uint32_t w = dbase[((size_t)row * p.nq + (g >> 3)) * NT + l];
      return (int)((w >> (4 * (g & 7))) & 15u);
    };
    if (rowp_global<NW>(p)) {
      // option tables in global memory: a speculative step would add a dependent global
      // read per candidate, so the backtrack stays serial (C4: 5 % faster this way)
      if (lane == 0) {
        for (int pos = n - 1; pos >= 0; --pos) {
          const int nb = nibble(pos, t);
          const int code = rw ? nb : 15 - nb;
          S.chosen[pos] = code;
          t = step(pos, t, code);
        }
      }
      __syncwarp();
      return;
    }
    int pos = n - 1;
    while (pos >= 0) {
      const int K = inf[pos].y & 255;
      int nib = 0;
      if (lane == 31) {
        nib = nibble(pos, t);
      } else if (lane <= K && pos >= 1) {
        const int tt = step(pos, t, lane);
        if (tt >= 0) nib = nibble(pos - 1, tt);
      }
      const int nib0 = __shfl_sync(0xffffffffu, nib, 31);
      const int code0 = rw ? nib0 : 15 - nib0;
      const int t1 = step(pos, t, code0);
      if (lane == 0) S.chosen[pos] = code0;
      if (pos == 0) break;
      const int nib1 = __shfl_sync(0xffffffffu, nib, code0);
      const int code1 = rw ? nib1 : 15 - nib1;
      t = step(pos - 1, t1, code1);
      if (lane == 0) S.chosen[pos - 1] = code1;
      pos -= 2;
    }
  }
  __syncwarp();
}

// After the backtrack the instance's decision nibbles are dead: invalidate their L2 lines
// (discard.global.L2, no write-back) so they never travel to HBM.  Row pos wrote
// ceil(groups / 8) chunks of NT words from the start of its row (the active columns
// t <= info.x: the deadline, or Qpre on the reward axis).  Only for the per-CTA scratch
// buffers; decisions kept in a caller's re-plan state are not touched.
template <int NW>
__device__ __forceinline__ void discard_decisions(const Params& p, const Smem& S, int s, int lane, int db) {
  constexpr int NT = 32 * NW;
  if (!p.discard || p.state || p.dec_smem) return;
  const int n = (int)S.misc[s * 16];
  const int4* inf = S.info + s * p.max_tasks;
  const char* base = (const char*)(S.dec + db * p.dec_words);
  const int64_t row_bytes = (int64_t)p.nq * NT * 4;
  for (int pos = lane; pos < n; pos += 32) {  // a lane per row
    const int cols = inf[pos].x + 1;
    const int lines = cols > 0 ? (((cols - 1) / NT) / 8 + 1) * NW : 0;  // 128-byte lines: NW per chunk
    const char* row = base + pos * row_bytes;
    for (int l = 0; l < lines; ++l) asm volatile("discard.global.L2 [%0], 128;" ::"l"(row + l * 128) : "memory");
  }
}

// a7/a8: EDF schedule (warp max-plus scan), outputs in input order, stats.
template <int NW, bool PK = false>
__device__ __forceinline__ void tail_outputs(const Params& p, const Smem& S, int s, int lane,
                                             unsigned long long* acc) {
  const long long* mi = S.misc + s * 16;
  const int n = (int)mi[0];
  const int64_t lo = mi[1], b = mi[2];
  const bool feasible = mi[5] >= 0;
  const bool rw = mi[9] != 0;  // option table in the reward-axis form (q, C*16 + code)
  const int4* inf = S.info + s * p.max_tasks;
  long long F = 0, Q = 0, conf = 0, ndrop = 0, nopt = 0, noff = 0;
  for (int base = 0; base < n; base += 32) {
    const int pos = base + lane;
    const bool valid = pos < n;
    int code = 0, tk = 0, Cc = 0, r = 0, Sn = 0;
    if (valid) {
      const int4 f = inf[pos];
      r = f.z;
      Sn = f.y >> 16;
      tk = S.task[s * p.max_tasks + pos];
      code = feasible ? S.chosen[pos] : 0;
    }
    long long a = 0, bb = -(1LL << 62);  // map x -> max(x + a, bb)
    if (code > 0) {
      const int2 o = opt_get<PK>(rowp_slot<NW>(p, S, s), (size_t)pos * p.kp + code - 1, rw);
      Cc = rw ? (o.y - code) >> 4 : o.x;
      a = Cc;
      bb = (long long)r + Cc;
      Q += rw ? o.x : (o.y + code) >> 4;
      {  // R_i(code-1), re-read from the (L2-resident) descriptors
        const int64_t t = lo + tk;
        long long R = p.mand_conf[t];
        for (int j = 0; j < code - 1; ++j) R += p.opt_gain[t * p.smax + j];
        conf += R;
      }
      nopt += code - 1;
    } else if (valid) {
      ndrop += 1;
    }
    noff += Sn;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {  // inclusive scan of map composition
      const long long a2 = __shfl_up_sync(0xffffffffu, a, o);
      const long long b2 = __shfl_up_sync(0xffffffffu, bb, o);
      if (lane >= o) {
        bb = max(b2 + a, bb);
        a = a2 + a;
      }
    }
    const long long f = max(F + a, bb);
    if (valid) {
      if (code > 0) {
        p.kept[lo + tk] = (int8_t)(code - 1);
        p.start[lo + tk] = (int32_t)(f - Cc);
        p.finish[lo + tk] = (int32_t)f;
      } else {
        p.kept[lo + tk] = -1;
        p.start[lo + tk] = -1;
        p.finish[lo + tk] = -1;
      }
    }
    F = __shfl_sync(0xffffffffu, f, 31);
  }
  Q = warp_sum64(Q);
  conf = warp_sum64(conf);
  ndrop = warp_sum64(ndrop);
  nopt = warp_sum64(nopt);
  noff = warp_sum64(noff);
  if (lane == 0) {
    p.q_total[b] = Q;
    p.conf_micro[b] = conf;
    p.conf_total[b] = (double)conf / 1e6;
    p.makespan[b] = (int32_t)F;
    p.status[b] = feasible ? ST_OK : ST_INFEASIBLE;
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
  __syncwarp();
}

// ---------------------------------------------------------------------------
// Resident CTAs per SM the register budget is sized for (NW = 1: 14 CTAs, 72 registers,
// +5 % on C2 over 12 CTAs / 85 registers; 16 CTAs / 64 registers spill and lose 2 %).
#ifndef IC_MINB1
#define IC_MINB1 14
#endif
constexpr int min_blocks(int nw) { return nw == 1 ? IC_MINB1 : nw == 2 ? 6 : nw == 4 ? 4 : nw == 8 ? 2 : 1; }

template <int NW, bool SB, bool DROP>
__global__ void __launch_bounds__(32 * (NW + 1), min_blocks(NW)) ic_dp_kernel(const Params p) {
  extern __shared__ __align__(16) unsigned char smem[];
  constexpr int NT = 32 * NW;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  Smem S;
  S.rowbuf = (int32_t*)(smem + p.off_rowbuf);
  S.dec = p.dec_smem ? (uint32_t*)(smem + p.off_dec) : p.dec_global + (int64_t)blockIdx.x * p.dec_slab_words;
  S.rowp = (int2*)(smem + p.off_rowp);
  S.info = (int4*)(smem + p.off_info);
  S.task = (int32_t*)(smem + p.off_task);
  S.tail = (int32_t*)(smem + p.off_tail);
  S.misc = (long long*)(smem + p.off_misc);
  S.chosen = (int32_t*)(smem + p.off_chosen);
  S.sd = (int32_t*)(smem + p.off_sd);
  S.sr = (int32_t*)(smem + p.off_sr);
  S.sS = (int32_t*)(smem + p.off_sS);
  S.key = (unsigned long long*)(smem + p.off_key);
  S.aux = (int32_t*)(smem + p.off_aux);
  S.sQ = (int32_t*)(smem + p.off_sQ);
  const int RS = p.rowbuf_stride;
  for (int bb = 0; bb < (SB ? 1 : 2); ++bb)
    for (int i = tid; i < p.pad; i += blockDim.x) S.rowbuf[bb * RS + i] = NEG;
  __syncthreads();

  if (warp == NW) {
    // ================= tail warp =================
    unsigned long long acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    // instances are claimed dynamically (work varies with U): one atomic per instance
    auto claim = [&]() -> int64_t {
      unsigned long long v = 0;
      if (lane == 0) v = atomicAdd(&p.work[0], 1ull);
      v = __shfl_sync(0xffffffffu, v, 0);
      if (p.ids) return v < *p.nids ? p.ids[v] : p.B;  // the instances the solo kernel deferred
      return (int64_t)v;
    };
    int64_t b = claim();
    while (b < p.B && tail_setup<NW>(p, S, b, 0, lane, acc) != ST_OK) b = claim();
    if (b >= p.B && lane == 0) S.misc[3] = ST_END;
    if (rowp_global<NW>(p)) __threadfence_block();  // the global option table is visible to the DP warps
    __syncwarp();
    bar_arrive(BAR_READY, NT + 32);
    if (p.nslots == 2) {
      int it = 0;
      while (b < p.B) {
        const int s = it & 1;
        const int db = p.ndec == 2 ? s : 0;
        int64_t nb = claim();
        while (nb < p.B && tail_setup<NW>(p, S, nb, s ^ 1, lane, acc) != ST_OK) nb = claim();
        if (nb >= p.B && lane == 0) S.misc[(s ^ 1) * 16 + 3] = ST_END;
        if (rowp_global<NW>(p)) __threadfence_block();
        __syncwarp();
        bar_sync(BAR_DONE, NT + 32);  // the DP warps finished instance b
        if (p.ndec == 2) {
          bar_arrive(BAR_READY, NT + 32);  // nb sweeps into the other decision buffer
          tail_backtrack<NW>(p, S, s, lane, db);
          if (IC_WS_DISCARD) discard_decisions<NW>(p, S, s, lane, db);
        } else {
          tail_backtrack<NW>(p, S, s, lane, db);
          if (IC_WS_DISCARD) discard_decisions<NW>(p, S, s, lane, db);
          __syncwarp();
          bar_arrive(BAR_READY, NT + 32);  // decisions free: the DP warps may start nb
        }
        tail_outputs<NW>(p, S, s, lane, acc);
        b = nb;
        ++it;
      }
    } else {
      while (b < p.B) {
        bar_sync(BAR_DONE, NT + 32);
        tail_backtrack<NW>(p, S, 0, lane, 0);
        if (IC_WS_DISCARD) discard_decisions<NW>(p, S, 0, lane, 0);
        tail_outputs<NW>(p, S, 0, lane, acc);
        int64_t nb = claim();
        while (nb < p.B && tail_setup<NW>(p, S, nb, 0, lane, acc) != ST_OK) nb = claim();
        if (nb >= p.B && lane == 0) S.misc[3] = ST_END;
        if (rowp_global<NW>(p)) __threadfence_block();
        __syncwarp();
        bar_arrive(BAR_READY, NT + 32);
        b = nb;
      }
    }
    if (lane == 0 && p.stats) {
#pragma unroll
      for (int i = 0; i < 8; ++i)
        if (acc[i]) atomicAdd(&p.stats[i], acc[i]);
    }
    if (lane == 0) {  // the last CTA out resets the counters for the next launch
      __threadfence();
      if (atomicAdd(&p.work[1], 1ull) == gridDim.x - 1) {
        p.work[0] = 0;
        p.work[1] = 0;
      }
    }
    return;
  }

  // ================= DP warps =================
  const int RSb = SB ? 0 : RS;
  int32_t* buf0 = S.rowbuf + p.pad;
  int padmode = 0;  // value in the pad cells: 0 NEG (time axis), 1 INFV (reward axis)
  int* rmax_slot = (int*)(S.misc + 2 * 16);  // reward axis: CTA max over finite columns
  for (int it = 0;; ++it) {
    bar_sync(BAR_READY, NT + 32);
    const int s = p.nslots == 2 ? (it & 1) : 0;
    uint32_t* decb = S.dec + (p.ndec == 2 && p.nslots == 2 ? (it & 1) : 0) * p.dec_words;
    long long* mi = S.misc + s * 16;
    if (mi[3] == ST_END) break;
    const int n = (int)mi[0];
    const int d_first = (int)mi[7];
    const bool rw = mi[9] != 0;
    const int64_t bcur = mi[2];
    const int k0 = p.replan ? (int)mi[10] : 0;  // first row to (re)compute
    if (p.state) {
      decb = state_dec(p, bcur);
      if (tid == 0) state_tail(p, bcur)[p.max_tasks] = rw ? 1 : 0;
    }
    if ((int)rw != padmode) {  // the pad left of column 0 must read as "invalid" for this axis
      padmode = rw;
      for (int bb = 0; bb < (SB ? 1 : 2); ++bb)
        for (int i = tid; i < p.pad; i += NT) S.rowbuf[bb * RS + i] = rw ? INFV : NEG;
    }
    if (rowp_global<NW>(p)) {  // this instance's option table: global (L2) slab -> shared memory
      const int4* src = (const int4*)rowp_slot<NW>(p, S, s);
      int4* dst = (int4*)S.rowp;
      for (int i = tid; i < n * p.kp / 2; i += NT) dst[i] = src[i];
    }
    if (rw) {  // P(0, 0) = 0, P(0, r > 0) = infinity
      // both row buffers start at infinity over every column the instance reaches
      // (Qpre_N): Qpre is non-decreasing, so a row's unreachable columns
      // (Qpre_pos, Qpre_next] were never written and need no per-row fill
      const int qn = (int)mi[8];
      for (int bb = 0; bb < (SB ? 1 : 2); ++bb)
        for (int t = tid; t <= qn; t += NT) buf0[bb * RSb + t] = (t == 0 && bb == 0) ? 0 : INFV;
      if (tid == 0) *rmax_slot = -1;
    } else {
      for (int t = tid; t <= d_first; t += NT) buf0[t] = 15;  // G_0(t) = 0
    }
    bar_sync(BAR_DP, NT);
    const int4* inf = S.info + s * p.max_tasks;
    const int2* rpb = rowp_global<NW>(p) ? S.rowp : S.rowp + (size_t)s * p.max_tasks * p.kp;
    const int32_t* auxp = S.aux + s * p.max_tasks;
    int M = 15;
    const size_t dec_row_words = (size_t)p.nq * NT;
    const int kp = p.kp;
    const int64_t rstride = p.H + 1;
    if (k0 > 0) {  // restore row k0-1 (its active columns, then its tail value up to d_k0)
      const int32_t* srow = state_rows(p, bcur) + (int64_t)(k0 / p.ckpt - 1) * rstride;
      int32_t* dst = buf0 + (k0 & 1) * RSb;
      const int dprev = inf[k0 - 1].x, dk = inf[k0].x;  // deadlines, or Qpre on the reward axis
      M = srow[p.H];
      for (int t = tid; t <= dprev; t += NT) dst[t] = srow[t];
      const int first = dprev + 1 > 0 ? dprev + 1 : 0;
      for (int t = first_col<NT>(first, tid); t <= dk; t += NT) dst[t] = rw ? INFV : M;
      bar_sync(BAR_DP, NT);
    }
    int4 f = inf[k0];
    int32_t* const tailp = S.tail + s * p.max_tasks;
    const int2* ops = rpb + (size_t)k0 * kp;
    uint32_t* decrow = decb + (size_t)k0 * dec_row_words;
    const bool keep_state = p.state != nullptr;  // loop invariants, read once per instance
    const bool dglob = !p.dec_smem || keep_state;  // decisions in global memory (hinted stores)
    const int ckm = p.ckpt - 1;
#pragma unroll 1
    for (int pos = k0; pos < n; ++pos) {
      const int4 fn = pos + 1 < n ? inf[pos + 1] : f;  // next row's header, off the critical path
      const int d = f.x, K = f.y & 255, r = f.z, dn = f.w;
      const bool gen = (f.y >> 8) & 1;
      const int32_t* cur = buf0 + (pos & 1) * RSb;
      int32_t* nxt = buf0 + ((pos + 1) & 1) * RSb;
      if (rw) {
        // reward axis: columns r <= Qpre_pos; (Qpre_pos, Qpre_next] are unreachable
        dp_row_dispatch<NW, SB, DROP, true>(K, (f.y >> 9) & 1, cur, nxt, decrow, (const int4*)ops, d, 0,
                                            auxp[pos], dglob);
        if (keep_state && ((pos + 1) & ckm) == 0) {  // checkpoint row for later re-plans
          int32_t* srow = state_rows(p, bcur) + (int64_t)((pos + 1) / p.ckpt - 1) * rstride;
          for (int t = tid; t <= d; t += NT) srow[t] = nxt[t];
        }
      } else {
        // admit value at column d: every column t > d shares it (tail collapse).  In
        // double-buffered mode its loads are issued here and consumed after the sweep.
        int av = NEG;
        if (lane < K) {
          const int2 o = ops[lane];
          const int src = d - o.x;
          if (src >= r) av = cur[src] + o.y;
        }
        int A = 0;
        if (SB) A = __reduce_max_sync(0xffffffffu, av);
        dp_row_dispatch<NW, SB, DROP, false>(K, gen, cur, nxt, decrow, (const int4*)ops, d, r, 0, dglob);
        if (!SB) A = __reduce_max_sync(0xffffffffu, av);
        const int Mv = DROP ? max(M, A) : A;
        if (tid == 0) tailp[pos] = Mv & 15;
        const int Mn = Mv | 15;
        // G_pos(t) = M_pos on (d, d_next]: the next row reads it there
        if (dn > d) {
          const int first = d + 1 > 0 ? d + 1 : 0;
#pragma unroll 1
          for (int t = first_col<NT>(first, tid); t <= dn; t += NT) nxt[t] = Mn;
        }
        M = Mn;
        if (keep_state) {  // keep checkpoint rows for later re-plans: active columns, tail value
          if (((pos + 1) & ckm) == 0) {
            int32_t* srow = state_rows(p, bcur) + (int64_t)((pos + 1) / p.ckpt - 1) * rstride;
            for (int t = tid; t <= d; t += NT) srow[t] = nxt[t];
            if (tid == 0) srow[p.H] = Mn;
          }
          if (tid == 0) state_tail(p, bcur)[pos] = Mv & 15;
        }
      }
      f = fn;
      ops += kp;
      decrow += dec_row_words;
      if (NW == 1)
        __syncwarp();
      else
        bar_sync(BAR_DP, NT);
    }
    const int32_t* fin = buf0 + (n & 1) * RSb;
    const int dl = (int)mi[8];
    if (rw) {
      // a5 (reward axis): r* = the largest finite column of row N (reading R6)
      int best = -1;
      for (int t = tid; t <= dl; t += NT)
        if (fin[t] < INFV) best = t;
      best = __reduce_max_sync(0xffffffffu, best);
      if (lane == 0) atomicMax(rmax_slot, best);
      bar_sync(BAR_DP, NT);
      if (tid == 0) {
        mi[5] = *rmax_slot;
        mi[6] = *rmax_slot;
      }
    } else if (warp == 0) {
      // a5: Q* = G_N(T), t* = least t with G_N(t) = Q*  (G_N non-decreasing on [0, d_N])
      long long Qv, ts = 0;
      if (dl < 0) {
        Qv = M;
      } else {
        Qv = fin[dl];
        int lo = 0, hi = dl;  // predicate fin[t] >= Qv is false below t*, true from t*
        while (lo < hi) {
          const int step = (hi - lo + 32) / 32;
          int x = lo + (lane + 1) * step - 1;
          if (x > hi) x = hi;
          const unsigned m = __ballot_sync(0xffffffffu, fin[x] >= Qv);
          const int fl = __ffs(m) - 1;
          const int nhi = fl == 0 ? min(lo + step - 1, hi) : min(lo + (fl + 1) * step - 1, hi);
          const int nlo = fl == 0 ? lo : lo + fl * step;
          lo = nlo;
          hi = nhi;
        }
        ts = lo;
      }
      if (lane == 0) {
        mi[5] = Qv >= 0 ? (Qv >> 4) : -1;
        mi[6] = ts;
      }
    }
    bar_sync(BAR_DP, NT);
    bar_arrive(BAR_DONE, NT + 32);
  }
}

typedef void (*KernelFn)(const Params);
KernelFn kernel_nw1(bool sb, bool drop);
KernelFn kernel_nw2(bool sb, bool drop);
KernelFn kernel_nw4(bool sb, bool drop);
KernelFn kernel_nw8(bool sb, bool drop);
KernelFn kernel_nw15(bool sb, bool drop);
KernelFn kernel_nw16(bool sb, bool drop);

}  // namespace icsched

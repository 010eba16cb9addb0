// ic_solo_kernel.cuh — one warp per instance, for short rows (H <= 1024: C1, C2).
//
// The warp-specialised kernel (ic_sched_kernel.cuh) pairs every sweep with a tail warp
// that sets up instance b+1 and backtracks b.  When a row is one warp wide that pairing
// costs half of the SM's warp slots and registers for a warp that idles two thirds of
// the time, and it lands the DP warps and the tail warps on different SM sub-partitions
// (ncu, profiles/r01_ncu_C2_summary.json: 33 % of all stall samples are idle tail warps).
// Here every warp runs the whole path a1-a8 for its own instances, one after another:
//
//   a1-a3  tail_setup (descriptor loads, prefix sums, Delta, packed keys, EDF sort)
//   a4     the time-indexed dual of Eqs. 1-2 or the paper's reward-indexed
//          table, one row at a time IN PLACE (a single row buffer: chunks from high to
//          low columns, loads -> __syncwarp -> stores, dp_row<1, true, ...>), so a warp
//          needs only (pad + H) * 4 bytes of shared memory for its row;
//   a5     Q* = G_N(T) and the least t* (32-ary ballot search), or r* on the reward axis;
//   a6-a8  tail_backtrack<1, true> / tail_outputs, as in the other kernel.
//
// Tail collapse without tail codes: after row i's sweep, the cell at column d_i already
// holds M_i = max(M_{i-1}, A_i) (the drop term reads G_{i-1}(d_i) = M_{i-1}), so the
// warp reads it back, fills (d_i, d_{i+1}] with it, and the backtrack reads the decision
// at min(t, d_i).  Latency of one warp's dependent steps (setup loads, backtrack chain)
// is hidden by the other resident warps instead of by warp specialisation.
#pragma once
#include "ic_sched_kernel.cuh"

#ifndef IC_SOLO_WPC
#define IC_SOLO_WPC 1  // warps per CTA (independent instances; 1: the finest shared-memory packing)
#endif
#ifndef IC_SOLO_KC
#define IC_SOLO_KC 9  // option counts with an unrolled sweep (more: the general path)
#endif
#ifndef IC_SOLO_MINB
#define IC_SOLO_MINB 28  // CTAs per SM the register budget is sized for (28 warps, 72 registers)
#endif

namespace icsched {

// One warp's view of its private shared-memory region (offsets from make_solo_layout).
__device__ __forceinline__ Smem solo_smem(const Params& p, unsigned char* base, uint32_t* dec) {
  Smem S;
  S.rowbuf = (int32_t*)(base + p.off_rowbuf);
  S.dec = dec;
  S.rowp = (int2*)(base + p.off_rowp);
  S.info = (int4*)(base + p.off_info);
  S.task = (int32_t*)(base + p.off_task);
  S.tail = nullptr;
  S.misc = (long long*)(base + p.off_misc);
  S.chosen = (int32_t*)(base + p.off_chosen);
  S.sd = (int32_t*)(base + p.off_sd);
  S.sr = (int32_t*)(base + p.off_sr);
  S.sS = (int32_t*)(base + p.off_sS);
  S.key = (unsigned long long*)(base + p.off_key);
  S.aux = (int32_t*)(base + p.off_aux);
  S.sQ = (int32_t*)(base + p.off_sQ);
  return S;
}
// the warp's statistics accumulators live in its misc block (slots 16..23), not in registers
__device__ __forceinline__ unsigned long long* solo_acc(const Params& p, unsigned char* base) {
  return (unsigned long long*)(base + p.off_misc) + 16;
}

// a1-a3 for instance b (tail_setup); ST_OK if the sweep must run.  The three phases are
// separate (non-inlined) functions so that each gets the whole register budget: the
// setup's sort keys and the sweep's option tables are never live at the same time.
template <bool PK>
static __device__ __noinline__ int solo_setup(const Params& p, unsigned char* base, int64_t b, int lane) {
  const Smem S = solo_smem(p, base, nullptr);
  return tail_setup<1, PK>(p, S, b, 0, lane, solo_acc(p, base));
}

// a4 + a5: the rows in place, then the optimum of row N into misc[5], misc[6].
template <bool DROP, bool STATE, bool PK, int KC>
__device__ __noinline__ void solo_sweep(const Params& p, unsigned char* base, uint32_t* dec, int lane) {
  // (dec: the warp's decision slab; replaced by the instance's state when one is kept)
  int32_t* const rowbuf = (int32_t*)(base + p.off_rowbuf);
  int32_t* const buf = rowbuf + p.pad;
  long long* mi = (long long*)(base + p.off_misc);
  const int n = (int)mi[0];
  const bool rw = mi[9] != 0;
  const int d_first = (int)mi[7], dl = (int)mi[8];
  // NEXT-2 (re-plan state): decisions go to the caller's state, every ckpt-th row is kept
  const int64_t bcur = mi[2];
  const int k0 = STATE && p.replan ? (int)mi[10] : 0;  // first row to (re)compute
  if (STATE) {
    dec = state_dec(p, bcur);
    if (lane == 0) state_tail(p, bcur)[p.max_tasks] = (rw ? 1 : 0) | 2;  // axis | written by the solo kernel
  }
  const bool refill = (int)rw != (int)mi[12];
  __syncwarp();
  if (refill) {  // the pad left of column 0 reads as "invalid" on this axis
    for (int i = lane; i < p.pad; i += 32) rowbuf[i] = rw ? INFV : NEG;
    if (lane == 0) mi[12] = rw;
  }
  if (rw) {  // P(0, 0) = 0, P(0, r > 0) = infinity over every column the instance reaches
    for (int t = lane; t <= dl; t += 32) buf[t] = t == 0 ? 0 : INFV;
  } else {
    for (int t = lane; t <= d_first; t += 32) buf[t] = 15;  // G_0(t) = 0
  }
  __syncwarp();
  const int4* inf = (const int4*)(base + p.off_info);
  const int32_t* aux = (const int32_t*)(base + p.off_aux);
  const int kp = p.kp;
  const int dec_row_words = p.nq * 32;
  // option entries of row pos start at entry pos * kp (int2, or one packed word with PK)
  const char* ops = (const char*)(base + p.off_rowp) + (size_t)k0 * kp * (PK ? 4 : 8);
  uint32_t* decrow = dec + (size_t)k0 * dec_row_words;
  int M = 15;
  if (STATE && k0 > 0) {  // restore row k0-1 (its active columns, then its tail value up to d_k0)
    const int32_t* srow = state_rows(p, bcur) + (int64_t)(k0 / p.ckpt - 1) * (p.H + 1);
    const int dprev = inf[k0 - 1].x, dk = inf[k0].x;  // deadlines, or Qpre on the reward axis
    M = srow[p.H];
    for (int t = lane; t <= dprev; t += 32) buf[t] = srow[t];
    const int first = dprev + 1 > 0 ? dprev + 1 : 0;
    for (int t = first + lane; t <= dk; t += 32) buf[t] = rw ? INFV : M;
    __syncwarp();
  }
#pragma unroll 1
  for (int pos = k0; pos < n; ++pos) {
    const int4 f = inf[pos];
    const int d = f.x, K = f.y & 255;
    if (rw) {
      // reward axis: columns r <= Qpre_pos; unreachable columns above stay infinite
      dp_row_dispatch<1, true, DROP, true, KC, PK>(K, (f.y >> 9) & 1, buf, buf, decrow, (const int4*)ops, d, 0, aux[pos]);
      __syncwarp();
      if (STATE && ((pos + 1) & (p.ckpt - 1)) == 0) {  // checkpoint row for later re-plans
        int32_t* srow = state_rows(p, bcur) + (int64_t)((pos + 1) / p.ckpt - 1) * (p.H + 1);
        for (int t = lane; t <= d; t += 32) srow[t] = buf[t];
      }
    } else {
      dp_row_dispatch<1, true, DROP, false, KC, PK>(K, (f.y >> 8) & 1, buf, buf, decrow, (const int4*)ops, d, f.z, 0);
      __syncwarp();
      // M_pos = G_pos(d) (tail collapse); G_pos(t) = M_pos on (d, d_next] for the next row
      if (d >= 0)
        M = buf[d];
      else if (!DROP)
        M = NEG | 15;
      if (STATE && ((pos + 1) & (p.ckpt - 1)) == 0) {  // checkpoint: active columns and tail value
        int32_t* srow = state_rows(p, bcur) + (int64_t)((pos + 1) / p.ckpt - 1) * (p.H + 1);
        for (int t = lane; t <= d; t += 32) srow[t] = buf[t];
        if (lane == 0) srow[p.H] = M;
      }
      const int dn = f.w;
      const int first = d + 1 > 0 ? d + 1 : 0;
#pragma unroll 1
      for (int t = first + lane; t <= dn; t += 32) buf[t] = M;
      __syncwarp();
    }
    ops += kp * (PK ? 4 : 8);
    decrow += dec_row_words;
  }
  // a5: the optimum of row N
  if (rw) {  // r* = the largest finite column (reading R6)
    int best = -1;
    for (int t = lane; t <= dl; t += 32)
      if (buf[t] < INFV) best = t;
    best = __reduce_max_sync(0xffffffffu, best);
    if (lane == 0) {
      mi[5] = best;
      mi[6] = best;
    }
  } else {  // Q* = G_N(T), t* = least t with G_N(t) = Q* (G_N non-decreasing on [0, d_N])
    long long Qv, ts = 0;
    if (dl < 0) {
      Qv = M;
    } else {
      Qv = buf[dl];
      int lo = 0, hi = dl;
      while (lo < hi) {
        const int step = (hi - lo + 32) / 32;
        int x = lo + (lane + 1) * step - 1;
        if (x > hi) x = hi;
        const unsigned m = __ballot_sync(0xffffffffu, buf[x] >= Qv);
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
  __syncwarp();
}

// a6-a8: backtrack, schedule times and outputs, stats.
template <bool PK>
static __device__ __noinline__ void solo_finish(const Params& p, unsigned char* base, uint32_t* dec, int lane) {
  const Smem S = solo_smem(p, base, dec);
  tail_backtrack<1, true, PK>(p, S, 0, lane, 0);
  discard_decisions<1>(p, S, 0, lane, 0);
  tail_outputs<1, PK>(p, S, 0, lane, solo_acc(p, base));
}

// STATE: the re-plan entry points (decisions and checkpoint rows kept in the caller's state);
// plain solves run the variant without any of that code.
// KC: the largest option count with an unrolled sweep body; task sets with at most 4 optional
// stages get KC = 5, whose smaller bodies leave the row loop's registers unspilled
template <bool DROP, bool STATE, bool PK, int KC = IC_SOLO_KC>
__global__ void __launch_bounds__(32 * IC_SOLO_WPC, IC_SOLO_MINB) ic_solo_kernel(const __grid_constant__ Params p) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned char* base = smem + (size_t)warp * p.solo_warp_bytes;
  uint32_t* dec = p.dec_global + ((int64_t)blockIdx.x * IC_SOLO_WPC + warp) * p.dec_slab_words;
  unsigned long long* acc = solo_acc(p, base);
  if (lane < 8) acc[lane] = 0;
  if (lane == 0) ((long long*)(base + p.off_misc))[12] = -1;  // pad contents: none yet
  __syncwarp();
  for (;;) {
    int64_t b;
    do {  // claim instances until one needs the DP (the others are answered in the setup)
      unsigned long long v = 0;
      if (lane == 0) v = atomicAdd(&p.work[0], 1ull);
      b = (int64_t)__shfl_sync(0xffffffffu, v, 0);
    } while (b < p.B && solo_setup<PK>(p, base, b, lane) != ST_OK);
    if (b >= p.B) break;
    solo_sweep<DROP, STATE, PK, KC>(p, base, dec, lane);
    solo_finish<PK>(p, base, dec, lane);
  }
  __syncwarp();
  if (lane < 8 && p.stats && acc[lane]) atomicAdd(&p.stats[lane], acc[lane]);
  if (lane == 0) {  // the last warp out resets the counters for the next launch
    __threadfence();
    if (atomicAdd(&p.work[1], 1ull) == (unsigned long long)gridDim.x * IC_SOLO_WPC - 1) {
      p.work[0] = 0;
      p.work[1] = 0;
    }
  }
}

KernelFn kernel_solo(bool drop, bool state, bool packed);
KernelFn kernel_solo5(bool drop, bool state, bool packed);

}  // namespace icsched

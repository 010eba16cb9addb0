// ic_reassign.cu — NEXT-3: the stage-completion event of the paper's scheduler
// (P:L235): re-predict the EDF-current task's utility from its observed confidence
// (Max / Exp / Lin heuristics) and apply the greedy depth reassignment of
// Eq. 5.  One warp per instance; batched O(N·S) candidate search with an
// O(1) (no releases: suffix slack) or O(N) EDF-feasibility check per candidate.
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/ic_sched.h"
#include "ic_sched_kernel.cuh"  // warp_sort_keys, warp_sum64

namespace {

constexpr int KMAXR = 15;

struct RParams {
  ic_batch_in in;
  const int8_t* kept_in;
  const int8_t* done;
  const uint32_t* observed;
  int heuristic;
  ic_batch_out out;
  uint8_t* swapped;
  int max_tasks, smax, H, np2, W;  // W = smax + 1: prefix-table row length
  int warp_bytes, opt_vec4;
};

__device__ __forceinline__ unsigned long long warp_max_u64(unsigned long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    const unsigned long long y = __shfl_xor_sync(0xffffffffu, v, o);
    v = y > v ? y : v;
  }
  return v;
}

// One step of the utility heuristics, micro-units, integer floor.
__device__ __forceinline__ long long predict_next(int h, long long r, long long pc, long long pn) {
  if (h == IC_UTIL_MAX) return 1000000;
  if (h == IC_UTIL_EXP) return r + (1000000 - r) / 2;
  if (h == IC_UTIL_LIN) {
    const long long v = pc > 0 ? r * pn / pc : 1000000;
    return v < 1000000 ? v : 1000000;
  }
  return r;
}

// One warp per instance.  The descriptors are read once (lane per task, 128-bit loads when
// the optional-stage rows allow it) into per-warp shared prefix tables C_i(k), R_i(k);
// the EDF sort, the Eq. 5 candidate search and the schedule all read those tables.
__global__ void __launch_bounds__(256, 4) reassign_kernel(const __grid_constant__ RParams p) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  unsigned char* base = smem + wib * p.warp_bytes;
  const int W = p.W, mt = p.max_tasks;
  unsigned long long* key = (unsigned long long*)base;
  int* Ct = (int*)(key + p.np2);  // [mt][W] cumulative WCET C_i(k) by input index
  int* Rt = Ct + mt * W;          // [mt][W] cumulative confidence R_i(k)
  int* ord = Rt + mt * W;         // EDF position -> input index; later the suffix slack
  int* rr = ord + mt;             // by EDF position: release, deadline, C of the (truncated) plan
  int* dd = rr + mt;
  int* ck = dd + mt;
  int* fb = ck + mt;              // finish of the kept tasks before pos (J_1 truncated)
  int* kk = fb + mt;              // kept depth by input index
  int* Sn = kk + mt;              // S_i by input index
  int* Rn = Sn + mt;              // [KMAXR] J_1's re-predicted curve
  const ic_batch_in& in = p.in;
  const int warps = gridDim.x * (blockDim.x >> 5);
  for (int64_t b = (int64_t)blockIdx.x * (blockDim.x >> 5) + wib; b < in.n_instances; b += warps) {
    const int64_t lo = in.task_begin[b], n64 = in.task_begin[b + 1] - lo;
    int bad = n64 < 0 || n64 > mt;
    const int n = bad ? 0 : (int)n64;
    // descriptors -> prefix tables, validation, EDF keys
    for (int i = lane; i < n; i += 32) {
      const int64_t t = lo + i;
      const int r = in.release[t], d = in.deadline[t], m = in.mand_wcet[t], S = in.n_opt[t], k = p.kept_in[t];
      const uint32_t a0 = in.mand_conf[t];
      int tb = (S > p.smax) | (r < 0) | (d >= p.H) | (m < 1) | (a0 > 1000000u) | (k < -1) | (k > S);
      long long C = m, R = a0;
      int* ci = Ct + i * W;
      int* ri = Rt + i * W;
      ci[0] = m;
      ri[0] = (int)a0;
      for (int j0 = 0; j0 < S && !tb; j0 += 4) {
        int w[4], g[4];
        if (p.opt_vec4) {
          const int4 w4 = *(const int4*)(in.opt_wcet + t * p.smax + j0);
          const int4 g4 = *(const int4*)(in.opt_gain + t * p.smax + j0);
          w[0] = w4.x; w[1] = w4.y; w[2] = w4.z; w[3] = w4.w;
          g[0] = g4.x; g[1] = g4.y; g[2] = g4.z; g[3] = g4.w;
        } else {
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (j0 + u < S) {
              w[u] = in.opt_wcet[t * p.smax + j0 + u];
              g[u] = in.opt_gain[t * p.smax + j0 + u];
            }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          if (j0 + u < S) {
            tb |= w[u] < 1;
            C += w[u];
            R += g[u];
            tb |= (R < 0) | (R > 1000000);
            ci[j0 + u + 1] = (int)min(C, 1ll << 30);  // only compared with deadlines < H
            ri[j0 + u + 1] = (int)R;
          }
        }
      }
      kk[i] = k;
      Sn[i] = S;
      bad |= tb;
      key[i] = ((unsigned long long)((uint32_t)d ^ 0x80000000u) << 32) |
               ((unsigned long long)min(max(r, 0), (1 << 20) - 1) << 12) | (unsigned)i;
    }
    bad = __any_sync(0xffffffffu, bad);
    if (!bad && n > 0) icsched::warp_sort_keys(key, n, lane);
    __syncwarp();
    // J_1: the first kept task in EDF order (the one on the GPU)
    int p1 = -1;
    if (!bad) {
      for (int base0 = 0; base0 < n && p1 < 0; base0 += 32) {
        const int pos = base0 + lane;
        const bool kept = pos < n && kk[(int)(key[pos] & 0xFFF)] >= 0;
        const unsigned m = __ballot_sync(0xffffffffu, kept);
        if (m) p1 = base0 + __ffs(m) - 1;
      }
    }
    int j1 = -1, l1 = 0, l1s = 0;
    long long rem_gain = 0, released = 0;
    bool search = false;
    if (!bad && p1 >= 0) {
      j1 = (int)(key[p1] & 0xFFF);
      l1 = p.done[b];
      l1s = kk[j1];
      const long long obs = p.observed[b];
      if (l1 < 0 || l1 > l1s || obs > 1000000) bad = 1;
      if (!bad) {
        // J_1's re-predicted curve, by lane 0 into shared memory
        const int* cj = Ct + j1 * W;
        const int* rj = Rt + j1 * W;
        int lower = 0;
        if (lane == 0) {
          const int S = Sn[j1];
          long long prev = 0;
          for (int k = 0; k <= S; ++k) {
            long long v;
            if (k < l1) v = rj[k];
            else if (k == l1) v = obs;
            else v = p.heuristic == IC_UTIL_GIVEN ? prev + (rj[k] - rj[k - 1])
                                                  : predict_next(p.heuristic, prev, cj[k - 1], cj[k]);
            Rn[k] = (int)v;
            prev = v;
            if (k >= l1 && k <= l1s && v < rj[k]) lower = 1;
          }
        }
        __syncwarp();
        lower = __shfl_sync(0xffffffffu, lower, 0);
        released = cj[l1s] - cj[l1];
        rem_gain = (long long)Rn[l1s] - Rn[l1];
        search = lower;
      }
    }
    // candidate search (Eq. 5): later tasks, extensions within the released budget
    unsigned long long best = 0;  // 0 = none
    if (search) {
      int norel = 1;
      for (int pos = lane; pos < n; pos += 32) {
        const int i = (int)(key[pos] & 0xFFF);
        ord[pos] = i;
        rr[pos] = in.release[lo + i];
        dd[pos] = in.deadline[lo + i];
        const int k = pos == p1 ? l1 : kk[i];
        ck[pos] = k >= 0 ? Ct[i * W + k] : -1;
        norel &= rr[pos] == 0;
      }
      norel = __all_sync(0xffffffffu, norel);
      __syncwarp();
      // finish times before each position (warp max-plus scan of x -> max(x + C, r + C))
      long long F = 0;
      for (int base0 = 0; base0 < n; base0 += 32) {
        const int pos = base0 + lane;
        const bool on = pos < n && ck[pos] >= 0;
        long long a = on ? ck[pos] : 0, bb = on ? (long long)rr[pos] + ck[pos] : -(1ll << 62);
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const long long a2 = __shfl_up_sync(0xffffffffu, a, o);
          const long long b2 = __shfl_up_sync(0xffffffffu, bb, o);
          if (lane >= o) {
            bb = max(b2 + a, bb);
            a = a2 + a;
          }
        }
        const long long f = max(F + a, bb);  // finish after pos
        long long prevf = __shfl_up_sync(0xffffffffu, f, 1);
        if (lane == 0) prevf = F;
        if (pos < n) fb[pos] = (int)prevf;
        F = __shfl_sync(0xffffffffu, f, 31);
      }
      __syncwarp();
      if (norel) {  // suffix minimum slack of the truncated schedule after each position (reuses ord)
        int carry = 1 << 30;  // min over the positions of the later chunks
        for (int base0 = (n - 1) & ~31; base0 >= 0; base0 -= 32) {
          const int pos = base0 + lane;
          int sl = pos < n && ck[pos] >= 0 ? (int)min((long long)dd[pos] - (fb[pos] + ck[pos]), 1ll << 30) : 1 << 30;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {  // inclusive suffix minimum within the chunk
            const int y = __shfl_down_sync(0xffffffffu, sl, o);
            if (lane + o < 32) sl = min(sl, y);
          }
          int after = __shfl_down_sync(0xffffffffu, sl, 1);  // positions strictly after pos
          if (lane == 31) after = 1 << 30;
          if (pos < n) ord[pos] = min(after, carry);
          carry = min(carry, __shfl_sync(0xffffffffu, sl, 0));
        }
      }
      __syncwarp();
      for (int pos = p1 + 1 + lane; pos < n; pos += 32) {
        const int i = (int)(key[pos] & 0xFFF);
        const int S = Sn[i], ki = kk[i];
        const int* ci = Ct + i * W;
        const int* ri = Rt + i * W;
        const long long C0 = ki >= 0 ? ci[ki] : 0, R0 = ki >= 0 ? ri[ki] : 0;
        for (int l = ki + 1 > 0 ? ki + 1 : 0; l <= S; ++l) {
          const long long C = ci[l];
          const long long cost = C - C0;
          if (cost > released) break;
          const long long gain = ri[l] - R0;
          // EDF feasibility of the plan with J_1 truncated and task i at depth l
          long long Fq = max((long long)fb[pos], (long long)rr[pos]) + C;
          bool ok = Fq <= dd[pos];
          if (norel) {  // no releases: every later finish moves by exactly the delay
            ok = ok && Fq - (ki >= 0 ? (long long)fb[pos] + ck[pos] : (long long)fb[pos]) <= ord[pos];
          } else {
            for (int q = pos + 1; q < n && ok; ++q) {
              if (ck[q] < 0) continue;
              Fq = max(Fq, (long long)rr[q]) + ck[q];
              ok = Fq <= dd[q];
            }
          }
          if (!ok) continue;
          const unsigned long long kv = ((unsigned long long)(gain + (1ll << 31)) << 32) |
                                        ((unsigned long long)(0xFFFF - pos) << 16) | (unsigned)(0xFFFF - l);
          best = kv > best ? kv : best;
        }
      }
      best = warp_max_u64(best);
    }
    int swap_i = -1, swap_l = -1;
    if (best != 0) {
      const long long g = (long long)(best >> 32) - (1ll << 31);
      if (g > rem_gain) {
        swap_i = (int)(key[0xFFFF - (int)((best >> 16) & 0xFFFF)] & 0xFFF);
        swap_l = 0xFFFF - (int)(best & 0xFFFF);
      }
    }
    // outputs: the plan's EDF schedule (warp max-plus scan with a carried finish time)
    long long conf = 0, F = 0;
    int status = bad ? IC_INST_BAD_INPUT : IC_INST_OK;
    if (!bad) {
      for (int base0 = 0; base0 < n; base0 += 32) {
        const int pos = base0 + lane;
        int k = -1, i = 0;
        long long C = 0, R = 0, r = 0;
        if (pos < n) {
          i = (int)(key[pos] & 0xFFF);
          k = kk[i];
          if (i == j1 && swap_i >= 0) k = l1;
          if (i == swap_i) k = swap_l;
          r = in.release[lo + i];
          if (k >= 0) {
            C = Ct[i * W + k];
            R = i == j1 ? Rn[k] : Rt[i * W + k];
          }
        }
        long long a = k >= 0 ? C : 0, bb = k >= 0 ? r + C : -(1ll << 62);  // x -> max(x + a, bb)
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const long long a2 = __shfl_up_sync(0xffffffffu, a, o);
          const long long b2 = __shfl_up_sync(0xffffffffu, bb, o);
          if (lane >= o) {
            bb = max(b2 + a, bb);
            a = a2 + a;
          }
        }
        const long long f = max(F + a, bb);
        if (pos < n) {
          const int64_t t = lo + i;
          p.out.kept[t] = (int8_t)k;
          p.out.start[t] = k >= 0 ? (int32_t)(f - C) : -1;
          p.out.finish[t] = k >= 0 ? (int32_t)f : -1;
          if (k >= 0) {
            conf += R;
            if (f > in.deadline[t]) status = IC_INST_INFEASIBLE;  // the given plan was infeasible
          }
        }
        F = __shfl_sync(0xffffffffu, f, 31);
      }
      conf = icsched::warp_sum64(conf);
      status = __reduce_max_sync(0xffffffffu, status);
    }
    if (status != IC_INST_OK) {
      for (int64_t i = lane; i < (n64 > 0 ? n64 : 0); i += 32) {
        p.out.kept[lo + i] = -1;
        p.out.start[lo + i] = -1;
        p.out.finish[lo + i] = -1;
      }
      conf = 0;
      F = 0;
      swap_i = -1;
    }
    if (lane == 0) {
      p.out.q_total[b] = 0;
      p.out.conf_micro[b] = conf;
      p.out.conf_total[b] = (double)conf / 1e6;
      p.out.makespan[b] = (int32_t)F;
      p.out.status[b] = (uint8_t)status;
      p.swapped[b] = swap_i >= 0 ? 1 : 0;
    }
    __syncwarp();
  }
}

}  // namespace

// Declared in include/ic_sched.h.  Uses only the handle's configuration (limits).
extern "C" __attribute__((visibility("hidden"))) int ic_sched_reassign_impl(const ic_sched_config* cfg, int sms, const ic_batch_in* in,
                                      const ic_stage_update* upd, ic_batch_out* out, uint8_t* swapped,
                                      void* cuda_stream) {
  RParams p{};
  p.in = *in;
  p.kept_in = upd->kept;
  p.done = upd->done;
  p.observed = upd->observed;
  p.heuristic = upd->heuristic;
  p.out = *out;
  p.swapped = swapped;
  p.max_tasks = cfg->max_tasks;
  p.smax = cfg->max_opt_stages;
  p.W = p.smax + 1;
  p.H = cfg->max_horizon;
  int np2 = 1;
  while (np2 < p.max_tasks) np2 <<= 1;
  p.np2 = np2 < 32 ? 32 : np2;
  p.warp_bytes = ((p.np2 * 8 + (2 * p.W + 8) * p.max_tasks * 4 + KMAXR * 4) + 15) & ~15;
  p.opt_vec4 = (p.smax & 3) == 0 && p.smax > 0 && ((uintptr_t)in->opt_wcet & 15) == 0 &&
               ((uintptr_t)in->opt_gain & 15) == 0;
  int wpb = (227 * 1024) / p.warp_bytes;
  if (wpb > 8) wpb = 8;
  if (wpb < 1) return IC_ERR_LIMIT;
  const int smem = wpb * p.warp_bytes;
  if (cudaFuncSetAttribute(reassign_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess)
    return IC_ERR_CUDA;
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, reassign_kernel, 32 * wpb, smem) != cudaSuccess)
    return IC_ERR_CUDA;
  int64_t blocks = (in->n_instances + wpb - 1) / wpb;
  const int64_t cap = (int64_t)sms * (per_sm > 0 ? per_sm : 1);
  if (blocks > cap) blocks = cap;
  reassign_kernel<<<(unsigned)blocks, 32 * wpb, smem, (cudaStream_t)cuda_stream>>>(p);
  return cudaGetLastError() == cudaSuccess ? IC_OK : IC_ERR_CUDA;
}

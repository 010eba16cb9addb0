// ic_reassign.cu — NEXT-3: the stage-completion event of the paper's scheduler
// (P:L235): re-predict the EDF-current task's utility from its observed confidence
// (Max / Exp / Lin heuristics) and apply the greedy depth reassignment of
// Eq. 5.  One warp per instance; batched O(N·S) candidate search with an
// O(N) EDF-feasibility check per candidate.
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/ic_sched.h"

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
  int max_tasks, smax, H, np2;
  int warp_bytes;
};

__device__ __forceinline__ long long warp_sum(long long v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

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

__global__ void __launch_bounds__(256) reassign_kernel(const RParams p) {
  extern __shared__ __align__(16) unsigned char smem[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  unsigned char* base = smem + wib * p.warp_bytes;
  unsigned long long* key = (unsigned long long*)base;
  int* ord = (int*)(key + p.np2);  // EDF position -> input index
  int* rr = ord + p.max_tasks;     // by EDF position: release, deadline, C of the planned option
  int* dd = rr + p.max_tasks;
  int* ck = dd + p.max_tasks;      // -1: not kept
  int* fb = ck + p.max_tasks;      // finish of the kept tasks before pos (J_1 truncated)
  const ic_batch_in& in = p.in;
  const int warps = gridDim.x * (blockDim.x >> 5);
  for (int64_t b = (int64_t)blockIdx.x * (blockDim.x >> 5) + wib; b < in.n_instances; b += warps) {
    const int64_t lo = in.task_begin[b], n64 = in.task_begin[b + 1] - lo;
    int bad = n64 < 0 || n64 > p.max_tasks;
    const int n = bad ? 0 : (int)n64;
    // descriptors, validation, EDF keys
    for (int i = lane; i < n; i += 32) {
      const int64_t t = lo + i;
      const int r = in.release[t], d = in.deadline[t], m = in.mand_wcet[t], S = in.n_opt[t], k = p.kept_in[t];
      const uint32_t a0 = in.mand_conf[t];
      int tb = (S > p.smax) | (r < 0) | (d >= p.H) | (m < 1) | (a0 > 1000000u) | (k < -1) | (k > S);
      long long R = a0;
      for (int j = 0; j < S && !tb; ++j) {
        tb |= in.opt_wcet[t * p.smax + j] < 1;
        R += in.opt_gain[t * p.smax + j];
        tb |= (R < 0) | (R > 1000000);
      }
      bad |= tb;
      key[i] = ((unsigned long long)((uint32_t)d ^ 0x80000000u) << 32) |
               ((unsigned long long)min(max(r, 0), (1 << 20) - 1) << 12) | (unsigned)i;
    }
    bad = __any_sync(0xffffffffu, bad);
    int np2 = 1;
    while (np2 < n) np2 <<= 1;
    if (!bad && n > 0) {
      for (int i = n + lane; i < np2; i += 32) key[i] = ~0ull;
      __syncwarp();
      for (int k = 2; k <= np2; k <<= 1)
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
    // J_1: the first kept task in EDF order (the one on the GPU)
    int p1 = -1;
    if (!bad) {
      for (int base0 = 0; base0 < n && p1 < 0; base0 += 32) {
        const int pos = base0 + lane;
        const bool kk = pos < n && p.kept_in[lo + (int)(key[pos] & 0xFFF)] >= 0;
        const unsigned m = __ballot_sync(0xffffffffu, kk);
        if (m) p1 = base0 + __ffs(m) - 1;
      }
    }
    int j1 = -1, l1 = 0, l1s = 0;
    long long rem_gain = 0, released = 0;
    long long Rnew[KMAXR];
    bool search = false;
    if (!bad && p1 >= 0) {
      j1 = (int)(key[p1] & 0xFFF);
      l1 = p.done[b];
      l1s = p.kept_in[lo + j1];
      const long long obs = p.observed[b];
      if (l1 < 0 || l1 > l1s || obs > 1000000) bad = 1;
      if (!bad) {
        // J_1's re-predicted curve; every lane computes it (uniform)
        const int64_t t = lo + j1;
        const int S = in.n_opt[t];
        long long C[KMAXR], R[KMAXR];
        C[0] = in.mand_wcet[t];
        R[0] = in.mand_conf[t];
#pragma unroll
        for (int k = 1; k < KMAXR; ++k)
          if (k <= S) {
            C[k] = C[k - 1] + in.opt_wcet[t * p.smax + k - 1];
            R[k] = R[k - 1] + in.opt_gain[t * p.smax + k - 1];
          }
        bool lower = false;
#pragma unroll
        for (int k = 0; k < KMAXR; ++k) {
          if (k > S) break;
          if (k < l1) Rnew[k] = R[k];
          else if (k == l1) Rnew[k] = obs;
          else Rnew[k] = p.heuristic == IC_UTIL_GIVEN ? Rnew[k - 1] + (R[k] - R[k - 1])
                                                      : predict_next(p.heuristic, Rnew[k - 1], C[k - 1], C[k]);
          if (k >= l1 && k <= l1s && Rnew[k] < R[k]) lower = true;
        }
        released = C[l1s] - C[l1];
        long long a = 0, z = 0;
#pragma unroll
        for (int k = 0; k < KMAXR; ++k) {
          if (k == l1) a = Rnew[k];
          if (k == l1s) z = Rnew[k];
        }
        rem_gain = z - a;
        search = lower;
      }
    }
    // candidate search (Eq. 5): later tasks, extensions within the released budget
    unsigned long long best = 0;  // 0 = none
    if (search) {
      // positions: release, deadline, planned C (J_1 truncated to l1) and the prefix finish
      for (int pos = lane; pos < n; pos += 32) {
        const int i = (int)(key[pos] & 0xFFF);
        ord[pos] = i;
        const int64_t t = lo + i;
        rr[pos] = in.release[t];
        dd[pos] = in.deadline[t];
        const int k = pos == p1 ? l1 : p.kept_in[t];
        int c = -1;
        if (k >= 0) {
          long long C = in.mand_wcet[t];
          for (int j = 0; j < k; ++j) C += in.opt_wcet[t * p.smax + j];
          c = (int)min(C, (long long)(1 << 30));
        }
        ck[pos] = c;
      }
      __syncwarp();
      int norel = 1;
      for (int pos = lane; pos < n; pos += 32) norel &= rr[pos] == 0;
      norel = __all_sync(0xffffffffu, norel);
      if (lane == 0) {
        long long F = 0;
        for (int pos = 0; pos < n; ++pos) {
          fb[pos] = (int)F;
          if (ck[pos] >= 0) F = max(F, (long long)rr[pos]) + ck[pos];
        }
        if (norel) {  // suffix minimum slack of the truncated schedule (reuses ord: no longer needed)
          long long smin = 1ll << 40;
          for (int pos = n - 1; pos >= 0; --pos) {
            ord[pos] = (int)min(smin, (long long)(1 << 30));
            if (ck[pos] >= 0) smin = min(smin, (long long)dd[pos] - (fb[pos] + ck[pos]));
          }
        }
      }
      __syncwarp();
      for (int pos = p1 + 1 + lane; pos < n; pos += 32) {
        const int i = (int)(key[pos] & 0xFFF);
        const int64_t t = lo + i;
        const int S = in.n_opt[t], ki = p.kept_in[t];
        long long C = in.mand_wcet[t], R = in.mand_conf[t], C0 = 0, R0 = 0;
        for (int l = 0; l <= S; ++l) {
          if (l > 0) {
            C += in.opt_wcet[t * p.smax + l - 1];
            R += in.opt_gain[t * p.smax + l - 1];
          }
          if (l == ki) {
            C0 = C;
            R0 = R;
          }
          if (l <= ki) continue;
          const long long cost = C - C0;
          if (cost > released) break;
          const long long gain = R - R0;
          // EDF feasibility of the plan with J_1 truncated and task i at depth l
          long long F = max((long long)fb[pos], (long long)rr[pos]) + C;
          bool ok = F <= dd[pos];
          if (norel) {  // no releases: every later finish moves by exactly the delay
            ok = ok && F - (ki >= 0 ? (long long)fb[pos] + ck[pos] : (long long)fb[pos]) <= ord[pos];
          } else {
            for (int q = pos + 1; q < n && ok; ++q) {
              if (ck[q] < 0) continue;
              F = max(F, (long long)rr[q]) + ck[q];
              ok = F <= dd[q];
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
    // outputs: the plan's EDF schedule (lane-serial chunks with a carried finish time)
    long long conf = 0, F = 0;
    int status = bad ? IC_INST_BAD_INPUT : IC_INST_OK;
    if (!bad) {
      for (int base0 = 0; base0 < n; base0 += 32) {
        const int pos = base0 + lane;
        int k = -1, i = 0;
        long long C = 0, R = 0, r = 0;
        if (pos < n) {
          i = (int)(key[pos] & 0xFFF);
          const int64_t t = lo + i;
          k = p.kept_in[t];
          if (i == j1 && swap_i >= 0) k = l1;
          if (i == swap_i) k = swap_l;
          r = in.release[t];
          if (k >= 0) {
            C = in.mand_wcet[t];
            R = in.mand_conf[t];
            for (int j = 0; j < k; ++j) {
              C += in.opt_wcet[t * p.smax + j];
              R += in.opt_gain[t * p.smax + j];
            }
            if (i == j1) {
#pragma unroll
              for (int kk = 0; kk < KMAXR; ++kk)
                if (kk == k) R = Rnew[kk];
            }
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
      conf = warp_sum(conf);
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
  p.H = cfg->max_horizon;
  int np2 = 1;
  while (np2 < p.max_tasks) np2 <<= 1;
  p.np2 = np2 < 32 ? 32 : np2;
  p.warp_bytes = ((p.np2 * 8 + 5 * p.max_tasks * 4) + 15) & ~15;
  int wpb = (227 * 1024) / p.warp_bytes;
  if (wpb > 8) wpb = 8;
  if (wpb < 1) return IC_ERR_LIMIT;
  const int smem = wpb * p.warp_bytes;
  if (cudaFuncSetAttribute(reassign_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem) != cudaSuccess)
    return IC_ERR_CUDA;
  int64_t blocks = (in->n_instances + wpb - 1) / wpb;
  const int64_t cap = (int64_t)sms * 8;
  if (blocks > cap) blocks = cap;
  reassign_kernel<<<(unsigned)blocks, 32 * wpb, smem, (cudaStream_t)cuda_stream>>>(p);
  return cudaGetLastError() == cudaSuccess ? IC_OK : IC_ERR_CUDA;
}

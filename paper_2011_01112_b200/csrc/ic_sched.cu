// ic_sched.cu — the C ABI of include/ic_sched.h: handle, launch geometry,
// workspace, and the host-buffer (end-to-end) entry point.
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "../../include/ic_sched.h"
#include "ic_sched_kernel.cuh"
#include "ic_solo_kernel.cuh"

using icsched::Params;

namespace {

constexpr int kMaxTasks = 4096;
constexpr int kMaxOpt = 14;
constexpr int kMaxHorizon = 32768;
constexpr int kSmemLimit = 227 * 1024;

using icsched::KernelFn;

KernelFn kernel_for(int nw, bool sb, bool drop) {
  switch (nw) {
    case 1: return icsched::kernel_nw1(sb, drop);
    case 2: return icsched::kernel_nw2(sb, drop);
    case 4: return icsched::kernel_nw4(sb, drop);
    case 8: return icsched::kernel_nw8(sb, drop);
    case 15: return icsched::kernel_nw15(sb, drop);
    case 16: return icsched::kernel_nw16(sb, drop);
    default: return nullptr;
  }
}

inline int align16(int x) { return (x + 15) & ~15; }

struct Layout {
  int bytes, nq, kp, r1, np2, pad, rs, nbuf;
  int off_rowbuf, off_dec, off_rowp, off_info, off_tR, off_task, off_tail, off_misc, off_chosen, off_sd, off_sr,
      off_sS, off_key, off_aux, off_sQ;
  int nslots, ndec, cap, rowp_global;
};

Layout make_layout(const ic_sched_config& c, int nw, bool sb, int pad, bool dec_smem, int nslots = 2,
                   int ndec = 1, int rowp_global = 0) {
  Layout L{};
  const int nt = 32 * nw;
  const int cols = (c.max_horizon + nt - 1) / nt;
  const int cap = nt * cols;
  const int mt = c.max_tasks;
  L.nq = (cols + 7) / 8;
  L.kp = (c.max_opt_stages + 2) & ~1;  // (C, key) pairs per row, even for int4 loads
  L.r1 = c.max_opt_stages + 1;
  int np2 = 1;
  while (np2 < mt) np2 <<= 1;
  L.np2 = np2 < 32 ? 32 : np2;
  L.pad = pad;
  L.rs = (pad + cap + 3) & ~3;
  L.nbuf = sb ? 1 : 2;
  L.nslots = nslots;
  const int ns = nslots;
  int o = 0;
  L.off_rowbuf = o; o = align16(o + L.nbuf * L.rs * 4);
  L.off_dec = o;    if (dec_smem) o = align16(o + ndec * mt * L.nq * nt * 4);
  L.ndec = ndec;
  L.rowp_global = rowp_global;  // option tables of both slots in global memory, one copy in smem
  L.off_rowp = o;   o = align16(o + ((rowp_global ? 1 : ns) * mt * L.kp + 8) * 8);
  L.off_info = o;   o = align16(o + ns * mt * 16);
  L.off_task = o;   o = align16(o + ns * mt * 4);
  L.off_tail = o;   o = align16(o + ns * mt * 4);
  L.off_misc = o;   o = align16(o + 3 * 16 * 8);
  L.off_chosen = o; o = align16(o + mt * 4);
  L.off_sd = o;     o = align16(o + mt * 4);
  L.off_sr = o;     o = align16(o + mt * 4);
  L.off_sS = o;     o = align16(o + mt * 4);
  L.off_key = o;    o = align16(o + L.np2 * 8);
  L.off_aux = o;    o = align16(o + ns * mt * 4);
  L.off_sQ = o;     o = align16(o + mt * 4);
  L.cap = cap;
  L.bytes = o;
  return L;
}

// One warp's private region in the solo kernel (ic_solo_kernel.cuh): a single in-place row
// and one slot of the per-task tables.  Offsets are relative to the warp's base.
Layout make_solo_layout(const ic_sched_config& c, int pad, int cap_cols = 0, bool packed = false) {
  Layout L{};
  const int cols = ((cap_cols ? cap_cols : c.max_horizon) + 31) / 32;
  const int cap = 32 * cols;
  const int mt = c.max_tasks;
  L.nq = (cols + 7) / 8;
  // option entries per row: int2 pairs (even count, 16-byte rows), or packed words (a
  // multiple of 4); the table ends with 64 bytes of slack for the sweep's 4 x int4 preload
  L.kp = packed ? (c.max_opt_stages + 4) & ~3 : (c.max_opt_stages + 2) & ~1;
  L.r1 = c.max_opt_stages + 1;
  int np2 = 1;
  while (np2 < mt) np2 <<= 1;
  L.np2 = np2 < 32 ? 32 : np2;
  L.pad = pad;
  L.rs = (pad + cap + 3) & ~3;
  L.nbuf = 1;
  L.nslots = 1;
  L.ndec = 1;
  int o = 0;
  L.off_rowbuf = o; o = align16(o + L.rs * 4);
  L.off_dec = o;
  L.off_rowp = o;   o = align16(o + mt * L.kp * (packed ? 4 : 8) + 64);
  L.off_info = o;   o = align16(o + mt * 16);
  L.off_task = o;   o = align16(o + mt * 4);
  L.off_tail = o;
  L.off_misc = o;   o = align16(o + 24 * 8);  // [0..15] instance header, [16..23] stats
  L.off_aux = o;    o = align16(o + mt * 4);
  // The setup's staging (sd, sr, sS, sQ, sort keys) and the backtrack's chosen codes are
  // never live during the sweep, and the sweep initialises every column it reads: they
  // share the row's column area (never the pad, whose contents persist across instances).
  // Fewer bytes per warp, more resident warps (C3 at Delta = 0.1: 17 -> 20 warps per SM).
  const int staged = align16(mt * 4) * 5 + align16(L.np2 * 8);
  int so = L.off_rowbuf + ((pad * 4 + 15) & ~15);  // the first column (past the pad)
  if (so + staged <= L.off_rowbuf + L.rs * 4) {
    L.off_chosen = so; so += align16(mt * 4);
    L.off_sd = so;     so += align16(mt * 4);
    L.off_sr = so;     so += align16(mt * 4);
    L.off_sS = so;     so += align16(mt * 4);
    L.off_sQ = so;     so += align16(mt * 4);
    L.off_key = so;
  } else {
    L.off_chosen = o; o = align16(o + mt * 4);
    L.off_sd = o;     o = align16(o + mt * 4);
    L.off_sr = o;     o = align16(o + mt * 4);
    L.off_sS = o;     o = align16(o + mt * 4);
    L.off_key = o;    o = align16(o + L.np2 * 8);
    L.off_sQ = o;     o = align16(o + mt * 4);
  }
  L.cap = cap;
  L.bytes = o;  // per warp
  return L;
}

}  // namespace

struct ic_sched {
  ic_sched_config cfg;
  int nw;
  bool sb;
  KernelFn fn;
  Layout L;
  int dec_smem, sms, ctas_per_sm, grid;
  uint32_t* dec_global;
  int64_t dec_slab_words;
  int2* rowp_g;
  int64_t rowp_slab;
  unsigned long long* work;
  void* stage;
  size_t stage_bytes;
  cudaStream_t s_in, s_comp, s_out;  // host entry point: copy-in / compute / copy-out pipeline
  cudaEvent_t ev[3 * 4 + 2];
  int64_t* tb_pinned;  // [3][chunk+1] rebased CSR offsets of the staged chunks
  int64_t tb_cap;
  // solo kernel (one warp per instance) for plain solves when chosen; the state / re-plan
  // entry points always use the warp-specialised kernel above
  KernelFn solo_fn, solo_state_fn;  // plain solves / the re-plan state entry points
  int hybrid;                 // 1: the solo kernel's row holds the reward axis only (fixed Delta,
                              // long horizon); instances it cannot sweep go to the ws kernel
  int64_t* defer_ids;         // [defer_cap] ids the solo kernel deferred; defer_n = their count
  unsigned long long* defer_n;
  int64_t defer_cap;
  Layout SL;
  int solo_grid, solo_ctas_per_sm;
  uint32_t* solo_dec;
  int64_t solo_dec_warp_words;
  int axis_mode;       // tuning, fixed at create: 0 auto per instance, 1 time, 2 reward
  int ckpt;            // re-plan checkpoint spacing (rows), power of two
  int no_vec_loads;    // 1: scalar descriptor loads only
  int solo_packed;     // the solo kernel's option tables hold packed words
  int discard;         // tuning.discard: 0 default (solo kernel on, warp-specialised off), 1 on, 2 off
};

extern "C" int ic_sched_create(const ic_sched_config* cfg, ic_sched** out) {
  return ic_sched_create_tuned(cfg, nullptr, out);
}

extern "C" int ic_sched_create_tuned(const ic_sched_config* cfg, const ic_sched_tuning* tuning, ic_sched** out) {
  if (!cfg || !out) return IC_ERR_INVALID_ARG;
  *out = nullptr;
  const ic_sched_config c = *cfg;
  ic_sched_tuning tu{};
  if (tuning) tu = *tuning;
  if (c.drop_mode != IC_DROP_ALLOWED && c.drop_mode != IC_MANDATORY_ENFORCED) return IC_ERR_INVALID_ARG;
  if (c.delta_micro == 0 && c.epsilon_micro == 0) return IC_ERR_INVALID_ARG;
  if (c.max_tasks < 1 || c.max_opt_stages < 0 || c.max_horizon < 1) return IC_ERR_INVALID_ARG;
  if (c.max_tasks > kMaxTasks || c.max_opt_stages > kMaxOpt || c.max_horizon > kMaxHorizon)
    return IC_ERR_LIMIT;
  if (tu.dp_warps < 0 || tu.pad_cols < 0 || tu.in_place < 0 || tu.in_place > 1 || tu.slots < 0 || tu.slots > 2 ||
      tu.decisions < 0 || tu.decisions > 2 || tu.option_tables < 0 || tu.option_tables > 1 || tu.axis < 0 ||
      tu.axis > 2 || tu.ckpt < 0 || (tu.ckpt & (tu.ckpt - 1)) != 0 || tu.ctas_per_sm < 0 || tu.no_vec_loads < 0 ||
      tu.no_vec_loads > 1 || tu.kernel < 0 || tu.kernel > 2 || tu.packed_options < 0 || tu.packed_options > 2 ||
      tu.discard < 0 || tu.discard > 2)
    return IC_ERR_INVALID_ARG;
  if (cudaSetDevice(c.device) != cudaSuccess) return IC_ERR_CUDA;
  int sms = 0;
  if (cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c.device) != cudaSuccess)
    return IC_ERR_CUDA;
  const bool drop = c.drop_mode == IC_DROP_ALLOWED;

  // DP warps per instance: about 32 column groups per thread (tuning.dp_warps overrides).
  int nw = 1;
  while (nw < 16 && 32 * nw * 32 < c.max_horizon) nw *= 2;
  // 16 DP warps + the tail warp = 17 warps: 5 on one SM sub-partition caps the registers at 96
  // (spills); 15 + 1 = 4 per sub-partition, 128 registers (C4: 6.07e4 -> 6.82e4 instances/s)
  if (nw == 16) nw = 15;
  if (tu.dp_warps) nw = tu.dp_warps;
  if (nw != 1 && nw != 2 && nw != 4 && nw != 8 && nw != 15 && nw != 16) return IC_ERR_INVALID_ARG;
  // NEG pad left of column 0: rows whose longest usable option reaches further use
  // the masked general path, so the pad only trades shared memory for speed.
  int pad = c.max_horizon / 16 < 64 ? 64 : (c.max_horizon / 16 > 256 ? 256 : c.max_horizon / 16);
  if (pad > c.max_horizon) pad = c.max_horizon;
  if (tu.pad_cols) pad = tu.pad_cols;
  pad = (pad + 31) & ~31;

  bool sb = tu.in_place != 0;  // in-place rows (tests force it at small H)
  if (sb && nw < 8) nw = 8;
  Layout Lg = make_layout(c, nw, sb, pad, false);
  if (!sb && Lg.bytes > kSmemLimit) {
    sb = true;
    if (nw < 8) nw = 8;
    Lg = make_layout(c, nw, true, pad, false);
  }
  int nslots = tu.slots == 1 ? 1 : 2;
  // large task sets: keep both slots' option tables in a global (L2) slab so the setup
  // and backtrack still overlap the sweep (tuning.option_tables = 1 forces it for tests)
  int rowp_global = tu.option_tables;
  if (nslots == 2 && nw >= 8 && (Lg.bytes > kSmemLimit || rowp_global)) {  // compiled for NW >= 8 only
    rowp_global = 1;
    Lg = make_layout(c, nw, sb, pad, false, 2, 1, 1);
  }
  if (Lg.bytes > kSmemLimit || nslots == 1) {  // serialise setup and sweep to fit large task sets
    nslots = 1;
    rowp_global = 0;
    Lg = make_layout(c, nw, sb, pad, false, 1);
  }
  if (Lg.bytes > kSmemLimit) return IC_ERR_LIMIT;
  // decisions: a global (L2-resident) double buffer by default, so the backtrack of
  // instance b overlaps the sweep of b+1; tuning.decisions = 1 keeps one buffer in smem.
  int ndec = nslots == 2 ? 2 : 1;
  bool dec_smem = false;
  if (tu.decisions == 1) {
    Layout Ls = make_layout(c, nw, sb, pad, true, nslots, 1, rowp_global);
    dec_smem = Ls.bytes <= kSmemLimit;
    if (dec_smem) ndec = 1;
  }
  if (tu.decisions == 2) ndec = 1;
  Layout L = make_layout(c, nw, sb, pad, dec_smem, nslots, ndec, rowp_global);

  KernelFn fn = kernel_for(nw, sb, drop);
  if (!fn) return IC_ERR_LIMIT;
  if (cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemLimit) != cudaSuccess)
    return IC_ERR_CUDA;
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, 32 * (nw + 1), L.bytes) != cudaSuccess)
    return IC_ERR_CUDA;
  if (per_sm < 1) return IC_ERR_LIMIT;
  // Spend the shared memory the occupancy leaves over on a wider pad: rows whose options
  // reach past it take the (slower) edge path for their first chunk.
  if (!tu.pad_cols) {
    for (int p2 = pad + 32; p2 <= c.max_horizon; p2 += 32) {
      const Layout L2 = make_layout(c, nw, sb, p2, dec_smem, nslots, ndec, rowp_global);
      int o2 = 0;
      if (L2.bytes > kSmemLimit ||
          cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o2, fn, 32 * (nw + 1), L2.bytes) != cudaSuccess ||
          o2 < per_sm)
        break;
      L = L2;
    }
  }
  if (tu.ctas_per_sm && tu.ctas_per_sm < per_sm) per_sm = tu.ctas_per_sm;

  ic_sched* h = (ic_sched*)calloc(1, sizeof(ic_sched));
  if (!h) return IC_ERR_OOM;
  h->cfg = c;
  h->nw = nw;
  h->sb = sb;
  h->fn = fn;
  h->L = L;
  h->dec_smem = dec_smem ? 1 : 0;
  h->sms = sms;
  h->ctas_per_sm = per_sm;
  h->grid = sms * per_sm;
  h->axis_mode = tu.axis;
  h->ckpt = tu.ckpt ? tu.ckpt : 4;
  h->no_vec_loads = tu.no_vec_loads;
  h->discard = tu.discard;
  if (cudaMalloc(&h->work, 16) != cudaSuccess || cudaMemset(h->work, 0, 16) != cudaSuccess) {
    free(h);
    return IC_ERR_OOM;
  }
  if (!dec_smem) {
    h->dec_slab_words = (int64_t)c.max_tasks * L.nq * 32 * nw * L.ndec;
    if (cudaMalloc(&h->dec_global, (size_t)h->dec_slab_words * 4 * h->grid) != cudaSuccess) {
      cudaFree(h->work);
      free(h);
      return IC_ERR_OOM;
    }
  }
  if (L.rowp_global) {
    h->rowp_slab = (int64_t)2 * c.max_tasks * L.kp + 8;
    if (cudaMalloc(&h->rowp_g, (size_t)h->rowp_slab * 8 * h->grid) != cudaSuccess) {
      if (h->dec_global) cudaFree(h->dec_global);
      cudaFree(h->work);
      free(h);
      return IC_ERR_OOM;
    }
  }
  // one warp per instance for one-warp rows (H <= 1024) unless the warp-specialised kernel
  // is asked for (tuning.kernel = 1); tuning.kernel = 2 forces it at any horizon
  const bool ws_knobs = tu.dp_warps || tu.in_place || tu.slots || tu.decisions || tu.option_tables;
  const bool solo = tu.kernel == 2 || (tu.kernel == 0 && !ws_knobs && nw == 1 && !sb);
  // Hybrid: with a fixed Delta every reward-axis row has at most N * floor(1e6 / Delta) + 1
  // columns (C3 at the paper's Delta = 0.1: 641).  When that is one warp's row but the
  // horizon is not, the solo kernel sweeps every instance whose chosen axis fits that row
  // (the reward axis, or a time axis with all deadlines below it) and defers the rest to
  // the warp-specialised kernel in a second launch.
  const int64_t qcap = c.delta_micro ? (int64_t)c.max_tasks * (1000000 / c.delta_micro) + 1 : (int64_t)1 << 40;
  const bool hybrid = !solo && tu.kernel == 0 && !ws_knobs && !tu.axis && qcap <= 1024 && c.max_horizon > 1024;
  if (solo || hybrid) {
    int rc = IC_OK;
    const int spad = tu.pad_cols ? ((tu.pad_cols + 31) & ~31) : 64 > c.max_horizon ? ((c.max_horizon + 31) & ~31) : 64;
    // packed option entries (one word per option: more resident warps) whenever a fixed Delta
    // bounds q <= 1e6 / Delta <= 2047 and the horizon bounds C <= 4095 (ic_sched_kernel.cuh pk_get)
    const bool packed = tu.packed_options != 2 && c.delta_micro > 0 && 1000000 / c.delta_micro <= 2047 &&
                        c.max_horizon <= 4096;
    Layout S = make_solo_layout(c, spad, hybrid ? (int)qcap : 0, packed);
    h->hybrid = hybrid ? 1 : 0;
    h->solo_packed = packed ? 1 : 0;
    // at most 4 optional stages: the instantiation whose unrolled sweeps stop at K = 5
    const bool k5 = c.max_opt_stages <= 4;
    KernelFn sf = k5 ? icsched::kernel_solo5(drop, false, packed) : icsched::kernel_solo(drop, false, packed);
    KernelFn sfs = k5 ? icsched::kernel_solo5(drop, true, packed) : icsched::kernel_solo(drop, true, packed);
    const int bytes = S.bytes * IC_SOLO_WPC;
    int sp = 0;
    if (bytes > kSmemLimit) rc = IC_ERR_LIMIT;
    if (rc == IC_OK && (cudaFuncSetAttribute(sf, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemLimit) != cudaSuccess ||
                        cudaFuncSetAttribute(sfs, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemLimit) != cudaSuccess))
      rc = IC_ERR_CUDA;
    if (rc == IC_OK &&
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&sp, sf, 32 * IC_SOLO_WPC, bytes) != cudaSuccess)
      rc = IC_ERR_CUDA;
    if (rc == IC_OK && sp < 1) rc = IC_ERR_LIMIT;
    if (rc == IC_OK && tu.ctas_per_sm && tu.ctas_per_sm < sp) sp = tu.ctas_per_sm;
    if (rc == IC_OK) {
      h->solo_fn = sf;
      h->solo_state_fn = sfs;
      h->SL = S;
      h->solo_ctas_per_sm = sp;
      h->solo_grid = sms * sp;
      h->solo_dec_warp_words = (int64_t)c.max_tasks * S.nq * 32;
      if (cudaMalloc(&h->solo_dec, (size_t)h->solo_dec_warp_words * 4 * h->solo_grid * IC_SOLO_WPC) != cudaSuccess)
        rc = IC_ERR_OOM;
    }
    if (rc != IC_OK) {
      ic_sched_destroy(h);
      return rc;
    }
  }
  *out = h;
  return IC_OK;
}

extern "C" int ic_sched_destroy(ic_sched* h) {
  if (!h) return IC_ERR_INVALID_ARG;
  cudaSetDevice(h->cfg.device);
  if (h->dec_global) cudaFree(h->dec_global);
  if (h->rowp_g) cudaFree(h->rowp_g);
  if (h->solo_dec) cudaFree(h->solo_dec);
  if (h->defer_ids) cudaFree(h->defer_ids);
  if (h->defer_n) cudaFree(h->defer_n);
  if (h->work) cudaFree(h->work);
  if (h->stage) cudaFree(h->stage);
  if (h->s_in) {
    cudaStreamDestroy(h->s_in);
    cudaStreamDestroy(h->s_comp);
    cudaStreamDestroy(h->s_out);
    for (cudaEvent_t e : h->ev) cudaEventDestroy(e);
  }
  if (h->tb_pinned) cudaFreeHost(h->tb_pinned);
  free(h);
  return IC_OK;
}

extern "C" int ic_sched_get_info(const ic_sched* h, ic_sched_info* info) {
  if (!h || !info) return IC_ERR_INVALID_ARG;
  if (h->solo_fn) {  // plain solves run one warp per instance
    info->threads_per_cta = 32 * IC_SOLO_WPC;
    info->cols_per_thread = (h->cfg.max_horizon + 31) / 32;
    info->ctas_per_sm = h->solo_ctas_per_sm;
    info->grid = h->solo_grid;
    info->smem_bytes = h->SL.bytes * IC_SOLO_WPC;
    info->decisions_in_smem = 0;
    info->double_buffered = 0;
    info->pad_cols = h->SL.pad;
    info->workspace_bytes = h->solo_dec_warp_words * 4 * h->solo_grid * IC_SOLO_WPC;
    info->kernels_per_solve = h->hybrid ? 2 : 1;
    info->hybrid = h->hybrid;
    info->packed_options = h->solo_packed;
    return IC_OK;
  }
  info->kernels_per_solve = 1;
  info->hybrid = 0;
  info->threads_per_cta = 32 * (h->nw + 1);
  info->cols_per_thread = (h->cfg.max_horizon + 32 * h->nw - 1) / (32 * h->nw);
  info->ctas_per_sm = h->ctas_per_sm;
  info->grid = h->grid;
  info->smem_bytes = h->L.bytes;
  info->decisions_in_smem = h->dec_smem;
  info->double_buffered = h->sb ? 0 : 1;
  info->pad_cols = h->L.pad;
  info->workspace_bytes = (h->dec_smem ? 0 : h->dec_slab_words * 4 * h->grid) + h->rowp_slab * 8 * h->grid;
  return IC_OK;
}

static int check_io(const ic_batch_in* in, const ic_batch_out* out) {
  if (!in || !out || in->n_instances < 0) return IC_ERR_INVALID_ARG;
  if (in->n_instances == 0) return IC_OK;
  if (!in->task_begin || !in->release || !in->deadline || !in->mand_wcet || !in->n_opt ||
      !in->mand_conf)
    return IC_ERR_INVALID_ARG;
  if (!out->kept || !out->start || !out->finish || !out->q_total || !out->conf_micro ||
      !out->conf_total || !out->makespan || !out->status)
    return IC_ERR_INVALID_ARG;
  return IC_OK;
}

static int64_t state_rows_bytes(const ic_sched* h) {  // every ckpt-th DP row (fixed at create)
  return (int64_t)(h->cfg.max_tasks / h->ckpt + 1) * (h->cfg.max_horizon + 1) * 4;
}
static int64_t state_dec_bytes(const ic_sched* h) { return (int64_t)h->cfg.max_tasks * h->L.nq * 32 * h->nw * 4; }
static int64_t state_stride(const ic_sched* h) {
  return (state_rows_bytes(h) + state_dec_bytes(h) + (int64_t)(h->cfg.max_tasks + 1) * 4 + 255) & ~(int64_t)255;
}

struct Departure {
  const int32_t *index, *deadline, *release;
};
static int launch_solve(ic_sched* h, const ic_batch_in* in, ic_batch_out* out, void* cuda_stream, void* state,
                        int replan, const Departure* dep = nullptr);

extern "C" int ic_sched_solve_batch(ic_sched* h, const ic_batch_in* in, ic_batch_out* out,
                                    void* cuda_stream) {
  return launch_solve(h, in, out, cuda_stream, nullptr, 0);
}

extern "C" int64_t ic_sched_state_bytes(const ic_sched* h, int64_t n_instances) {
  if (!h || n_instances < 0) return IC_ERR_INVALID_ARG;
  return state_stride(h) * n_instances;
}

static int state_ok(const ic_sched* h, const void* state) {
  if (!h || !state) return IC_ERR_INVALID_ARG;
  if (h->cfg.delta_micro == 0) return IC_ERR_INVALID_ARG;  // FPTAS Delta changes with every arrival
  return IC_OK;
}

extern "C" int ic_sched_solve_batch_state(ic_sched* h, const ic_batch_in* in, ic_batch_out* out, void* state,
                                          void* cuda_stream) {
  const int rc = state_ok(h, state);
  return rc != IC_OK ? rc : launch_solve(h, in, out, cuda_stream, state, 0);
}

extern "C" int ic_sched_replan_batch(ic_sched* h, const ic_batch_in* in, void* state, ic_batch_out* out,
                                     void* cuda_stream) {
  const int rc = state_ok(h, state);
  return rc != IC_OK ? rc : launch_solve(h, in, out, cuda_stream, state, 1);
}

extern "C" int ic_sched_depart_batch(ic_sched* h, const ic_batch_in* in, const int32_t* removed_index,
                                     const int32_t* removed_deadline, const int32_t* removed_release, void* state,
                                     ic_batch_out* out, void* cuda_stream) {
  const int rc = state_ok(h, state);
  if (rc != IC_OK) return rc;
  if (!in || (in->n_instances > 0 && (!removed_index || !removed_deadline || !removed_release)))
    return IC_ERR_INVALID_ARG;
  const Departure dep{removed_index, removed_deadline, removed_release};
  return launch_solve(h, in, out, cuda_stream, state, 1, &dep);
}

static int launch_solve(ic_sched* h, const ic_batch_in* in, ic_batch_out* out, void* cuda_stream, void* state,
                        int replan, const Departure* dep) {
  if (!h) return IC_ERR_INVALID_ARG;
  int rc = check_io(in, out);
  if (rc != IC_OK) return rc;
  if (h->cfg.max_opt_stages > 0 && in->n_instances > 0 && (!in->opt_wcet || !in->opt_gain))
    return IC_ERR_INVALID_ARG;
  if (in->n_instances == 0) return IC_OK;
  if (cudaSetDevice(h->cfg.device) != cudaSuccess) return IC_ERR_CUDA;
  Params p{};
  p.B = in->n_instances;
  p.task_begin = in->task_begin;
  p.release = in->release;
  p.deadline = in->deadline;
  p.mand_wcet = in->mand_wcet;
  p.n_opt = in->n_opt;
  p.opt_wcet = in->opt_wcet;
  p.mand_conf = in->mand_conf;
  p.opt_gain = in->opt_gain;
  p.kept = out->kept;
  p.start = out->start;
  p.finish = out->finish;
  p.q_total = out->q_total;
  p.conf_micro = out->conf_micro;
  p.conf_total = out->conf_total;
  p.makespan = out->makespan;
  p.status = out->status;
  p.stats = (unsigned long long*)out->stats;
  p.delta_micro = h->cfg.delta_micro;
  p.eps_micro = h->cfg.epsilon_micro;
  p.max_tasks = h->cfg.max_tasks;
  p.smax = h->cfg.max_opt_stages;
  p.H = h->cfg.max_horizon;
  const Layout& L = h->L;
  p.pad = L.pad;
  p.nq = L.nq;
  p.kp = L.kp;
  p.r1 = L.r1;
  p.np2 = L.np2;
  p.dec_smem = h->dec_smem;
  p.dec_global = h->dec_global;
  p.dec_slab_words = h->dec_slab_words;
  p.off_rowbuf = L.off_rowbuf;
  p.off_dec = L.off_dec;
  p.off_rowp = L.off_rowp;
  p.off_info = L.off_info;
  p.off_task = L.off_task;
  p.off_tail = L.off_tail;
  p.off_misc = L.off_misc;
  p.off_chosen = L.off_chosen;
  p.off_sd = L.off_sd;
  p.off_sr = L.off_sr;
  p.off_sS = L.off_sS;
  p.off_key = L.off_key;
  p.rowbuf_stride = L.rs;
  p.nslots = L.nslots;
  p.cap = L.cap;
  p.off_aux = L.off_aux;
  p.off_sQ = L.off_sQ;
  p.axis_mode = h->axis_mode;
  p.state = (char*)state;
  p.state_stride = state_stride(h);
  p.state_dec_off = state_rows_bytes(h);
  p.state_tail_off = state_rows_bytes(h) + state_dec_bytes(h);
  p.replan = replan;
  p.nw = h->nw;
  if (dep) {
    p.dep_index = dep->index;
    p.dep_deadline = dep->deadline;
    p.dep_release = dep->release;
  }
  p.ckpt = h->ckpt;
  p.work = h->work;
  p.ndec = L.ndec;
  p.dec_words = (int64_t)h->cfg.max_tasks * L.nq * 32 * h->nw;
  p.rowp_g = h->rowp_g;
  p.rowp_slab = h->rowp_slab;
  p.opt_vec4 = (p.smax & 3) == 0 && p.smax > 0 && ((uintptr_t)p.opt_wcet & 15) == 0 &&
               ((uintptr_t)p.opt_gain & 15) == 0 && !h->no_vec_loads;
  // Discarding dead decision lines keeps them from HBM (C5: 64 -> 1 KB written per instance)
  // but its L2 operations cost the warp-specialised kernel 2.5 % (C5 4.74e6 -> 4.62e6) while
  // the one-warp kernel gains from it (C2 +3 %): default on for the solo kernel only.
  p.discard = h->discard == 1;
  const Params pw = p;  // the warp-specialised kernel's parameters
  if (h->solo_fn) {  // one warp per instance (ic_solo_kernel.cuh); hybrid: then the deferred ids
    const Layout& S = h->SL;
    if (h->hybrid) {  // room for every id the solo kernel may defer, and a zeroed count
      if (in->n_instances > h->defer_cap) {
        if (h->defer_ids) cudaFree(h->defer_ids);
        h->defer_ids = nullptr;
        h->defer_cap = 0;
        if (cudaMalloc(&h->defer_ids, (size_t)in->n_instances * 8) != cudaSuccess) return IC_ERR_OOM;
        h->defer_cap = in->n_instances;
      }
      if (!h->defer_n && cudaMalloc(&h->defer_n, 8) != cudaSuccess) return IC_ERR_OOM;
      if (cudaMemsetAsync(h->defer_n, 0, 8, (cudaStream_t)cuda_stream) != cudaSuccess) return IC_ERR_CUDA;
      p.defer_ids = h->defer_ids;
      p.defer_n = h->defer_n;
    }
    p.pad = S.pad;
    p.nq = S.nq;
    p.np2 = S.np2;
    p.kp = S.kp;
    p.discard = h->discard != 2;
    p.dec_smem = 0;
    p.dec_global = h->solo_dec;
    p.dec_slab_words = h->solo_dec_warp_words;
    p.dec_words = h->solo_dec_warp_words;
    p.ndec = 1;
    p.nslots = 1;
    p.cap = S.cap;
    p.rowbuf_stride = S.rs;
    p.solo_warp_bytes = S.bytes;
    p.off_rowbuf = S.off_rowbuf;
    p.off_dec = S.off_dec;
    p.off_rowp = S.off_rowp;
    p.off_info = S.off_info;
    p.off_task = S.off_task;
    p.off_tail = S.off_tail;
    p.off_misc = S.off_misc;
    p.off_chosen = S.off_chosen;
    p.off_sd = S.off_sd;
    p.off_sr = S.off_sr;
    p.off_sS = S.off_sS;
    p.off_key = S.off_key;
    p.off_aux = S.off_aux;
    p.off_sQ = S.off_sQ;
    p.rowp_g = nullptr;
    int64_t grid = h->solo_grid;
    const int64_t need = (in->n_instances + IC_SOLO_WPC - 1) / IC_SOLO_WPC;
    if (grid > need) grid = need;
    (state ? h->solo_state_fn : h->solo_fn)<<<(unsigned)grid, 32 * IC_SOLO_WPC, S.bytes * IC_SOLO_WPC,
                                               (cudaStream_t)cuda_stream>>>(p);
    if (cudaGetLastError() != cudaSuccess) return IC_ERR_CUDA;
    if (!h->hybrid) return IC_OK;
    // the deferred instances: the warp-specialised kernel over the listed ids (its CTAs
    // exit at once when the list is empty)
    Params q = pw;
    q.ids = h->defer_ids;
    q.nids = h->defer_n;
    h->fn<<<(unsigned)h->grid, 32 * (h->nw + 1), h->L.bytes, (cudaStream_t)cuda_stream>>>(q);
    return cudaGetLastError() == cudaSuccess ? IC_OK : IC_ERR_CUDA;
  }
  int64_t grid = h->grid;
  if (grid > in->n_instances) grid = in->n_instances;
  h->fn<<<(unsigned)grid, 32 * (h->nw + 1), h->L.bytes, (cudaStream_t)cuda_stream>>>(p);
  if (cudaGetLastError() != cudaSuccess) return IC_ERR_CUDA;
  return IC_OK;
}

extern "C" int ic_sched_reassign_impl(const ic_sched_config* cfg, int sms, const ic_batch_in* in,
                                      const ic_stage_update* upd, ic_batch_out* out, uint8_t* swapped,
                                      void* cuda_stream);

extern "C" int ic_sched_reassign_batch(ic_sched* h, const ic_batch_in* in, const ic_stage_update* upd,
                                       ic_batch_out* out, uint8_t* swapped, void* cuda_stream) {
  if (!h || !upd || !swapped) return IC_ERR_INVALID_ARG;
  int rc = check_io(in, out);
  if (rc != IC_OK) return rc;
  if (in->n_instances == 0) return IC_OK;
  if (!upd->kept || !upd->done || !upd->observed || upd->heuristic < IC_UTIL_GIVEN ||
      upd->heuristic > IC_UTIL_LIN)
    return IC_ERR_INVALID_ARG;
  if (h->cfg.max_opt_stages > 0 && (!in->opt_wcet || !in->opt_gain)) return IC_ERR_INVALID_ARG;
  if (cudaSetDevice(h->cfg.device) != cudaSuccess) return IC_ERR_CUDA;
  return ic_sched_reassign_impl(&h->cfg, h->sms, in, upd, out, swapped, cuda_stream);
}

// Host-buffer entry point: H2D of the inputs, solve, D2H of the outputs.  The batch
// is cut into instance chunks (>= 8, each <= ~256 MB staged) that cycle through a
// ring of three device staging slots over three internal streams (copy-in,
// compute, copy-out), so PCIe traffic overlaps the sweep and device memory stays
// bounded whatever the batch size.  Kernels stay serialised on the compute stream
// (they share the decision workspace).  Ordered after prior work on
// `cuda_stream`; synchronised before returning.
extern "C" int ic_sched_solve_batch_host(ic_sched* h, const ic_batch_in* in, ic_batch_out* out,
                                         void* cuda_stream) {
  if (!h) return IC_ERR_INVALID_ARG;
  int rc = check_io(in, out);
  if (rc != IC_OK) return rc;
  if (in->n_instances == 0) return IC_OK;
  if (h->cfg.max_opt_stages > 0 && (!in->opt_wcet || !in->opt_gain)) return IC_ERR_INVALID_ARG;
  if (cudaSetDevice(h->cfg.device) != cudaSuccess) return IC_ERR_CUDA;
  if (!h->s_in) {
    if (cudaStreamCreateWithFlags(&h->s_in, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&h->s_comp, cudaStreamNonBlocking) != cudaSuccess ||
        cudaStreamCreateWithFlags(&h->s_out, cudaStreamNonBlocking) != cudaSuccess)
      return IC_ERR_CUDA;
    for (cudaEvent_t& e : h->ev)
      if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) return IC_ERR_CUDA;
  }
  const int64_t B = in->n_instances;
  const int64_t* tbh = in->task_begin;
  for (int64_t b = 0; b < B; ++b)
    if (tbh[b + 1] < tbh[b]) return IC_ERR_INVALID_ARG;
  const int64_t st = h->cfg.max_opt_stages;
  const int64_t T = tbh[B] - tbh[0];
  const int64_t task_bytes = 4 * 5 + 1 + 8 * st + 9, inst_bytes = 8 * 4 + 4 + 1 + 8;
  // chunk: at least 8 per batch for overlap, at most ~256 MB of staging
  int64_t chunk = (B + 7) / 8;
  const int64_t per_inst = (T / B + 1) * task_bytes + inst_bytes;
  const int64_t lim = (256ll << 20) / per_inst;
  if (chunk > lim) chunk = lim > 64 ? lim : 64;
  if (chunk < 1) chunk = 1;
  // the largest chunk's task count bounds the slot size
  int64_t maxt = 0;
  for (int64_t b0 = 0; b0 < B; b0 += chunk) {
    const int64_t b1 = b0 + chunk < B ? b0 + chunk : B;
    if (tbh[b1] - tbh[b0] > maxt) maxt = tbh[b1] - tbh[b0];
  }
  size_t off = 0;
  auto take = [&](size_t bytes) { size_t o = off; off = (off + bytes + 255) & ~(size_t)255; return o; };
  const size_t o_tb = take((chunk + 1) * 8), o_r = take(maxt * 4), o_d = take(maxt * 4),
               o_m = take(maxt * 4), o_n = take(maxt), o_ow = take(maxt * st * 4), o_mc = take(maxt * 4),
               o_og = take(maxt * st * 4), o_k = take(maxt), o_s = take(maxt * 4), o_f = take(maxt * 4),
               o_q = take(chunk * 8), o_c = take(chunk * 8), o_ct = take(chunk * 8), o_ms = take(chunk * 4),
               o_st = take(chunk);
  const size_t slot = off;
  const size_t o_stats = 3 * slot;
  if (o_stats + 64 > h->stage_bytes) {
    if (h->stage) cudaFree(h->stage);
    h->stage = nullptr;
    h->stage_bytes = 0;
    if (cudaMalloc(&h->stage, o_stats + 64) != cudaSuccess) return IC_ERR_OOM;
    h->stage_bytes = o_stats + 64;
  }
  if (chunk + 1 > h->tb_cap) {
    if (h->tb_pinned) cudaFreeHost(h->tb_pinned);
    h->tb_pinned = nullptr;
    h->tb_cap = 0;
    if (cudaMallocHost(&h->tb_pinned, 3 * (chunk + 1) * 8) != cudaSuccess) return IC_ERR_OOM;
    h->tb_cap = chunk + 1;
  }
  char* g0 = (char*)h->stage;
  cudaStream_t user = (cudaStream_t)cuda_stream;
  // every early return first drains the three pipeline streams, so no copy still in flight
  // touches the caller's host buffers or the pinned CSR ring after the call returns
  auto fail = [&](int code) {
    cudaStreamSynchronize(h->s_in);
    cudaStreamSynchronize(h->s_comp);
    cudaStreamSynchronize(h->s_out);
    return code;
  };
  cudaEvent_t* ev = h->ev;  // [slot*4 + 0] inputs staged, +1 kernel done, +2 outputs drained; [12], [13]
  bool ok = cudaEventRecord(ev[13], user) == cudaSuccess &&
            cudaStreamWaitEvent(h->s_in, ev[13], 0) == cudaSuccess &&
            cudaStreamWaitEvent(h->s_comp, ev[13], 0) == cudaSuccess;
  if (out->stats) ok = ok && cudaMemsetAsync(g0 + o_stats, 0, 64, h->s_comp) == cudaSuccess;
  int64_t j = 0;
  for (int64_t b0 = 0; b0 < B && ok; b0 += chunk, ++j) {
    const int64_t b1 = b0 + chunk < B ? b0 + chunk : B, nbi = b1 - b0;
    const int64_t t0 = tbh[b0], nt = tbh[b1] - t0;
    const int sl = (int)(j % 3);
    char* g = g0 + sl * slot;
    if (j >= 3) {  // slot reuse: its previous chunk's outputs must be drained, its CSR copied
      if (cudaEventSynchronize(ev[sl * 4 + 2]) != cudaSuccess) return fail(IC_ERR_CUDA);
      ok = cudaStreamWaitEvent(h->s_in, ev[sl * 4 + 2], 0) == cudaSuccess;
    }
    int64_t* tbp = h->tb_pinned + sl * (chunk + 1);
    for (int64_t b = 0; b <= nbi; ++b) tbp[b] = tbh[b0 + b] - t0;  // rebase onto the slot's rows
    auto h2d = [&](size_t o, const void* src, size_t bytes) {
      return bytes == 0 || cudaMemcpyAsync(g + o, src, bytes, cudaMemcpyHostToDevice, h->s_in) == cudaSuccess;
    };
    ok = ok && h2d(o_tb, tbp, (nbi + 1) * 8) && h2d(o_r, in->release + t0, nt * 4) &&
         h2d(o_d, in->deadline + t0, nt * 4) && h2d(o_m, in->mand_wcet + t0, nt * 4) &&
         h2d(o_n, in->n_opt + t0, nt) && h2d(o_mc, in->mand_conf + t0, nt * 4);
    if (st > 0)
      ok = ok && h2d(o_ow, in->opt_wcet + t0 * st, nt * st * 4) && h2d(o_og, in->opt_gain + t0 * st, nt * st * 4);
    ok = ok && cudaEventRecord(ev[sl * 4], h->s_in) == cudaSuccess &&
         cudaStreamWaitEvent(h->s_comp, ev[sl * 4], 0) == cudaSuccess;
    if (!ok) break;
    ic_batch_in din = {nbi, (const int64_t*)(g + o_tb), (const int32_t*)(g + o_r), (const int32_t*)(g + o_d),
                       (const int32_t*)(g + o_m), (const uint8_t*)(g + o_n), (const int32_t*)(g + o_ow),
                       (const uint32_t*)(g + o_mc), (const int32_t*)(g + o_og)};
    ic_batch_out dout = {(int8_t*)(g + o_k), (int32_t*)(g + o_s), (int32_t*)(g + o_f), (int64_t*)(g + o_q),
                         (int64_t*)(g + o_c), (double*)(g + o_ct), (int32_t*)(g + o_ms), (uint8_t*)(g + o_st),
                         out->stats ? (int64_t*)(g0 + o_stats) : nullptr};
    rc = ic_sched_solve_batch(h, &din, &dout, h->s_comp);
    if (rc != IC_OK) return fail(rc);
    ok = cudaEventRecord(ev[sl * 4 + 1], h->s_comp) == cudaSuccess &&
         cudaStreamWaitEvent(h->s_out, ev[sl * 4 + 1], 0) == cudaSuccess;
    auto d2h = [&](void* dst, size_t o, size_t bytes) {
      return bytes == 0 || cudaMemcpyAsync(dst, g + o, bytes, cudaMemcpyDeviceToHost, h->s_out) == cudaSuccess;
    };
    ok = ok && d2h(out->kept + t0, o_k, nt) && d2h(out->start + t0, o_s, nt * 4) &&
         d2h(out->finish + t0, o_f, nt * 4) && d2h(out->q_total + b0, o_q, nbi * 8) &&
         d2h(out->conf_micro + b0, o_c, nbi * 8) && d2h(out->conf_total + b0, o_ct, nbi * 8) &&
         d2h(out->makespan + b0, o_ms, nbi * 4) && d2h(out->status + b0, o_st, nbi) &&
         cudaEventRecord(ev[sl * 4 + 2], h->s_out) == cudaSuccess;
  }
  int64_t stats_dev[8];
  if (ok && out->stats) {
    ok = cudaEventRecord(ev[12], h->s_comp) == cudaSuccess && cudaStreamWaitEvent(h->s_out, ev[12], 0) == cudaSuccess &&
         cudaMemcpyAsync(stats_dev, g0 + o_stats, 64, cudaMemcpyDeviceToHost, h->s_out) == cudaSuccess;
  }
  if (!ok) return fail(IC_ERR_CUDA);
  if (cudaStreamSynchronize(h->s_out) != cudaSuccess) return fail(IC_ERR_CUDA);
  if (out->stats)
    for (int i = 0; i < 8; ++i) out->stats[i] += stats_dev[i];
  return IC_OK;
}

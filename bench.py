"""Benchmark: scheduling instances solved per second on 1..8 B200s.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2|C3|C4|C5]
    python bench.py --impl reference ...     # the CPU oracle, timed on the host cores
    torchrun --nproc-per-node N bench.py --gpus N ...

One step = one pass of the whole hot path (descriptor
load, prefix/quantise, EDF sort, DP sweep, backtrack, schedule, stats) over
one batch of the configuration's instances, inputs resident in HBM, followed by
the NCCL all-reduce of the int64 stats vector when N > 1.  The default workload
is C5, the configuration BASELINE.json's metric ("instances solved/sec at
1/2/4/8 B200") is quoted on: 2^24 instances of the C3 shape in four
utilisation blocks U = 1, 2, 4, 8, split over the ranks (strong scaling; each
rank generates its own contiguous global-id shard on device).  C1-C4 are
weak-scaled (every rank solves a full batch of distinct ids).  Rank 0 prints
one JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import gen  # noqa: E402

SMEM_BYTES_PER_CLK_PER_SM = 128  # LDS crossbar (B300_MICROARCH.md "smem crossbar BW 128/N B/cyc/SM")
BYTES_PER_EVAL = 4               # one int32 DP cell read per (task, tick, option)
METRIC = "scheduling instances solved/sec"


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        return json.load(open(p))
    except Exception:
        return {}


def _sms():
    import torch
    return torch.cuda.get_device_properties(torch.cuda.current_device()).multi_processor_count


def algorithmic_evals(inputs, n_tasks, opt_stride, delta_micro=0, eps_micro=100_000, chunk=16384):
    """Algorithmic option evaluations of a batch (measurement only; torch ops on the inputs).

    Returns (W_active, W_survey).  W_survey = sum_i [(T+1) + sum_k #{t <= d_i : t - C_i(k) >= r_i}],
    T = max(0, max_i d_i).  W_active counts what this kernel evaluates on the
    axis it picks per instance: on the time axis
      sum_i [(d_i + 1)^+ + sum_k #{t <= d_i : t - C_i(k) >= r_i}]
    (columns past d_i share one value), on the reward axis (the paper's P(i, r), chosen when its
    estimate sum_i (Qpre_i + 1)(K_i + 1) is the smaller, no releases)
      sum_i [(Qpre_i + 1) + sum_{k < K_i} (Qpre_i - q_i(k) + 1)^+],
    Qpre_i = prefix over EDF order of max_k q_i(k).  Each evaluation reads one 4-byte DP cell."""
    import torch
    B = inputs["task_begin"].numel() - 1
    wa = ws = 0
    N = n_tasks
    for lo in range(0, B, chunk):
        hi = min(B, lo + chunk)
        nb = hi - lo
        sl = slice(lo * N, hi * N)
        m = inputs["mand_wcet"][sl].long()
        ow = inputs["opt_wcet"][sl].long()
        S = inputs["n_opt"][sl].long()
        w = torch.cat([m[:, None], ow], 1)
        C = torch.cumsum(w, 1)
        k = torch.arange(opt_stride + 1, device=C.device)[None, :]
        valid = k <= S[:, None]
        d = inputs["deadline"][sl].long()
        r = inputs["release"][sl].long()
        fit = (C <= (d - r)[:, None]) & valid
        K = fit.sum(1)
        opts = torch.clamp(d[:, None] - r[:, None] - C + 1, min=0) * valid
        T = torch.clamp(d.view(nb, N).max(1).values, min=0)
        ws += int(((T + 1) * N).sum() + opts.sum())
        wt_inst = (torch.clamp(d + 1, min=0) + opts.sum(1)).view(nb, N).sum(1)
        # reward axis (replicates the kernel's per-instance choice)
        R = inputs["mand_conf"][sl].long()[:, None] + torch.cat(
            [torch.zeros_like(m)[:, None], torch.cumsum(inputs["opt_gain"][sl].long(), 1)], 1)
        if delta_micro:
            dl = torch.full((nb,), delta_micro, dtype=torch.long, device=C.device)
        else:
            feas = ((r[:, None] + C) <= d[:, None]) & valid
            rmax = torch.where(feas, R, torch.zeros_like(R)).max(1).values.view(nb, N).max(1).values
            dl = torch.clamp(eps_micro * rmax // (1_000_000 * N), min=1)
        q = torch.where(valid, R // dl.repeat_interleave(N)[:, None], torch.zeros_like(R))
        qmax = torch.where(fit, q, torch.zeros_like(q)).max(1).values.view(nb, N)  # options that fit
        key = d.view(nb, N) * (N + 1) + torch.arange(N, device=C.device)[None, :]  # EDF (d, idx); r = 0 here
        order = torch.argsort(key, 1)
        qpre = torch.cumsum(torch.gather(qmax, 1, order), 1)
        Kg = torch.gather(K.view(nb, N), 1, order)
        qg = torch.gather(q.view(nb, N, -1), 1, order[:, :, None].expand(-1, -1, q.shape[1]))
        kk = torch.arange(q.shape[1], device=C.device)[None, None, :]
        ropt = (torch.clamp(qpre[:, :, None] - qg + 1, min=0) * (kk < Kg[:, :, None])).sum(2)
        wr_inst = ((qpre + 1) + ropt).sum(1)
        est_t = (torch.clamp(d + 1, min=0).view(nb, N) * (K.view(nb, N) + 1)).sum(1)
        est_r = ((qpre + 1) * (Kg + 1)).sum(1)
        norel = (r.view(nb, N) == 0).all(1)
        use_r = norel & (est_r < est_t)
        wa += int(torch.where(use_r, wr_inst, wt_inst).sum())
    return wa, ws


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index, self.rows, self.proc = index, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([x.strip() for x in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if len(r) > 5 + i and r[5 + i] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def workload_config(cw, args, n_instances):
    mode = f"Delta={args.delta_micro / 1e6:g}" if args.delta_micro else f"FPTAS eps={cw.epsilon_micro / 1e6:g}"
    return {"workload": f"{cw.name}: {n_instances} instances/GPU x {cw.n_tasks} tasks x (1 mandatory + "
                        f"{cw.n_opt} optional stages), horizon {cw.horizon} ticks, U in [{cw.u_lo},{cw.u_hi}], "
                        f"{mode}, drop allowed",
            "name": cw.name, "instances_per_gpu": n_instances, "tasks": cw.n_tasks, "optional_stages": cw.n_opt,
            "horizon": cw.horizon, "seed": hex(cw.seed)}


def sample_batch(cw, n, salt=0):
    """n instances of the workload for the CPU oracle; C5 draws equally from its U blocks."""
    if not cw.u_blocks:
        return gen.generate(cw, n, id_offset=salt)
    parts, start = [], 0
    per = max(1, n // len(cw.u_blocks))
    for _, cnt in cw.u_blocks:
        parts.append(gen.generate(cw, per, id_offset=start + salt))
        start += cnt
    return gen.concat(parts, cw.n_opt)


def cpu_model():
    try:
        for line in subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout.splitlines():
            if line.startswith("Model name:"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


def _oracle_cfg(cw, delta_micro):
    import oracle
    return oracle.OracleConfig(epsilon_micro=cw.epsilon_micro, delta_micro=delta_micro, max_tasks=cw.n_tasks,
                               max_horizon=cw.horizon)


def _native_oracle():
    """Load the oracle built -O3 -march=native for this host."""
    import oracle
    try:
        oracle.use_native_build()
        return "gcc -O3 -march=native"
    except Exception:  # no compiler on the host: the portable -O3 build
        return "gcc -O3"


def _time_oracle(cw, ocfg, algo, threads, target_s, salt=0):
    """Instances/s of the oracle (as it stands) on `threads` threads over a sample sized to run
    about target_s seconds (calibrated on a smaller sample of other ids first)."""
    import oracle
    n = max(threads * 8, 32)
    while True:
        cal = sample_batch(cw, n, salt=salt + (1 << 20))
        t0 = time.perf_counter()
        oracle.solve(cal, ocfg, algo, threads)
        dt = time.perf_counter() - t0
        if dt >= 0.5 or n >= cw.n_instances:
            break
        n *= 4
    rate = n / dt
    for _ in range(3):  # the first calibration pass pays thread start-up and page faults
        n = int(min(cw.n_instances, max(threads * 8, rate * target_s)))
        sample = sample_batch(cw, n, salt=salt)
        t0 = time.perf_counter()
        oracle.solve(sample, ocfg, algo, threads)
        el = time.perf_counter() - t0
        rate = sample.n_instances / el
        if el >= 0.6 * target_s or n >= cw.n_instances:
            break
    return rate, sample.n_instances, el


def cpu_oracle_baseline(cw, args, target_s):
    """the oracle timed on the host cores, as it stands, built -O3 -march=native
    for this host: O3 (the time-indexed DP, the scale oracle whose cost matches the GPU's) on
    every core and on one core, plus O2 (the paper's reward-indexed DP, Eqs. 1-2) at the paper's
    Delta = 0.1 beside it.  Bounded samples of the same workload."""
    import oracle
    build = _native_oracle()
    threads = os.cpu_count() or 1
    v, n, el = _time_oracle(cw, _oracle_cfg(cw, args.delta_micro), oracle.TIME, threads, target_s)
    v1, n1, el1 = _time_oracle(cw, _oracle_cfg(cw, args.delta_micro), oracle.TIME, 1, target_s / 4, salt=1 << 21)
    v2, n2, el2 = _time_oracle(cw, _oracle_cfg(cw, 100_000), oracle.PAPER, threads, target_s / 4, salt=1 << 22)
    part = "equal parts of every U block" if cw.u_blocks else "consecutive ids"
    return {"value": v, "unit": "instances/s", "cores": threads, "kind": "oracle",
            "sample": f"{n} {cw.name} instances ({part}), O3 time-indexed DP on {threads} OpenMP threads, {el:.1f} s",
            "algorithm": "O3 (oracle/ic_oracle.c solve_time) at the workload's own Delta", "build": build,
            "cpu_model": cpu_model(),
            "single_thread": {"value": v1, "unit": "instances/s", "sample": f"{n1} instances, {el1:.1f} s"},
            "paper_dp_delta_0_1": {"value": v2, "unit": "instances/s", "cores": threads,
                                   "sample": f"{n2} instances, O2 (Eqs. 1-2, Alg. 1) at Delta = 0.1, {el2:.1f} s"}}


# The paper's own figures for the method (context, not the target: different hardware, and the
# paper's solver runs on the CPU with TensorFlow inference on the GPU).  BASELINE.md §1.
PAPER_CONTEXT = {
    "hardware": "Intel i7-4770 (32 GB) + NVIDIA TITAN X Pascal, TensorFlow 1.14 (P:L251)",
    "accuracy_gain_vs_edf_lcf_rr": "+10% ~ 20% (P:L6, P:L221)",
    "deadline_misses": "(nearly) no deadline misses (P:L6)",
    "exp_vs_opt_utility": "within 2% of optimal most of the time (P:L260-261, P:L273)",
    "scheduler_overhead": "0.5% - 6% of per-request time, user-space CPU scheduler (P:L536, P:L541)",
    "solver_throughput": "not reported (BASELINE.md §1)",
}


def smem_peak(local):
    """Measured shared-memory load bandwidth of this GPU (include/ic_probe.h): the roofline
    denominator of the sweep.  The peak is the conflict-free 4-byte LDS stream, the access the
    sweep makes (one LDS.32 per option evaluation); the LDS.128 stream (the crossbar's ceiling
    with vector loads) and the LDS.32 + VIADDMNMX stream (the sweep's inner op) are beside it."""
    import paper_2011_01112_b200 as pkg
    r = {m: pkg.probe_smem(local, m, 60.0) for m in ("lds32", "lds128", "lds32_viaddmax")}
    best = r["lds32"]
    return {"gbs": best["gbs"], "bytes_per_clk_per_sm": best["bytes_per_clk_per_sm"], "mode": "lds32",
            "modes": {m: {"gbs": round(x["gbs"], 1), "bytes_per_clk_per_sm": round(x["bytes_per_clk_per_sm"], 2),
                          "sm_mhz": round(x["sm_mhz"], 1)} for m, x in r.items()}}


def run_reference(args, cw, rank, world):
    """--impl reference: the CPU oracle (O3, -O3 -march=native) on the host cores, rank 0 only."""
    if rank != 0:
        return
    import oracle
    build = _native_oracle()
    threads = os.cpu_count() or 1
    ocfg = _oracle_cfg(cw, args.delta_micro)
    # size each step so the whole K+W-step run stays near two minutes of CPU work
    per_step = min(10.0, max(1.0, 120.0 / (args.steps + args.warmup)))
    _, n, _ = _time_oracle(cw, ocfg, oracle.TIME, threads, per_step)
    sample = sample_batch(cw, n)
    n = sample.n_instances
    for _ in range(args.warmup):
        oracle.solve(sample, ocfg, oracle.TIME, threads)
    t0 = time.perf_counter()
    for _ in range(args.steps):
        oracle.solve(sample, ocfg, oracle.TIME, threads)
    el = time.perf_counter() - t0
    v = n * args.steps / el
    line = {"metric": METRIC, "value": v, "unit": "instances/s", "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": el / args.steps * 1e3, "higher_is_better": True,
            "scaling": "strong" if cw.u_blocks and not args.instances else "weak", "vs_baseline": None,
            "dtype": "int64", "data": "synthetic", "impl": "reference", "config": workload_config(cw, args, n),
            "cpu_baseline": {"value": v, "unit": "instances/s", "cores": threads, "kind": "oracle",
                             "sample": f"{n} instances of {cw.name} per step, O3 time-indexed DP ({build})",
                             "cpu_model": cpu_model()},
            "e2e": {"value": v, "unit": "instances/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def run_replan(args, cw, sched, inputs, out, stream, n_inst, world, rank, dev, strong):
    """--op replan: NEXT-2, Alg. 1 from row k.  Arrival: every instance's last task
    arrives and the rows before its EDF position come from the state of the solve without it.
    Departure: every instance loses one task (index b*7 mod N) and the rows before its
    old EDF position come from the state of the solve with it.  Both reported beside a full solve
    of the same instances (the state-keeping solve itself is not timed)."""
    import torch
    N = cw.n_tasks
    pkg = sys.modules["paper_2011_01112_b200"]

    def subset(drop):  # every instance without task drop[b] (others in order)
        keep = torch.ones(n_inst, N, dtype=torch.bool, device=dev)
        keep[torch.arange(n_inst, device=dev), drop] = False
        sub = {}
        for k, v in inputs.items():
            if k == "task_begin":
                sub[k] = torch.arange(n_inst + 1, device=dev, dtype=torch.int64) * (N - 1)
            else:
                w = v.view(torch.int32) if v.dtype == torch.uint32 else v  # no uint32 gather on CUDA
                w = (w.view(n_inst, N, -1)[keep].reshape(n_inst * (N - 1), -1) if v.dim() == 2
                     else w.view(n_inst, N)[keep]).contiguous()
                sub[k] = w.view(torch.uint32) if v.dtype == torch.uint32 else w
        return sub

    last = torch.full((n_inst,), N - 1, dtype=torch.long, device=dev)
    base = subset(last)  # before the arrival
    dropj = (torch.arange(n_inst, device=dev) * 7) % N
    after = subset(dropj)  # after the departure
    j32 = dropj.to(torch.int32)
    dl = inputs["deadline"].view(n_inst, N)[torch.arange(n_inst, device=dev), dropj].to(torch.int32).contiguous()
    rl = inputs["release"].view(n_inst, N)[torch.arange(n_inst, device=dev), dropj].to(torch.int32).contiguous()
    state = torch.empty(sched.state_bytes(n_inst), dtype=torch.uint8, device=dev)
    out2 = pkg.alloc_outputs(n_inst, n_inst * (N - 1), device=dev)
    k = args.steps or 10
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            sched.solve_batch(inputs, out, stream)
        ev[0].record(stream)
        for _ in range(k):
            sched.solve_batch(inputs, out, stream)
        ev[1].record(stream)
        ta = td = 0.0
        for _ in range(k):
            sched.solve_batch_state(base, state, None, stream)
            ev[2].record(stream)
            sched.replan_batch(inputs, state, out, stream)
            ev[3].record(stream)
            ev[3].synchronize()
            ta += ev[2].elapsed_time(ev[3])
        for _ in range(k):
            sched.solve_batch_state(inputs, state, None, stream)
            ev[2].record(stream)
            sched.depart_batch(after, j32, dl, rl, state, out2, stream)
            ev[3].record(stream)
            ev[3].synchronize()
            td += ev[2].elapsed_time(ev[3])
    stream.synchronize()
    full_ms = ev[0].elapsed_time(ev[1]) / k
    rep_ms, dep_ms = ta / k, td / k
    if rank == 0:
        total = n_inst * world
        info = sched.info()
        print(json.dumps({
            "metric": "re-plans on arrival/sec (Alg. 1 from row k)", "value": total / (rep_ms / 1e3),
            "unit": "instances/s", "n_gpus": world, "steps": k, "warmup": args.warmup, "ms_per_step": rep_ms,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int32",
            "data": "synthetic (device-generated, seeded)", "config": workload_config(cw, args, n_inst),
            "full_solve_ms": full_ms, "speedup_vs_full_solve": full_ms / rep_ms,
            "departure": {"value": total / (dep_ms / 1e3), "unit": "instances/s", "ms_per_step": dep_ms,
                          "speedup_vs_full_solve": full_ms / dep_ms},
            "kernel": info, "state_bytes_per_instance": sched.state_bytes(1),
            "gpu_launches": 3 * k * info.get("kernels_per_solve", 1)}), flush=True)


def run_reassign(args, cw, sched, inputs, out, stream, n_inst, world, rank, dev, strong):
    """--op reassign: one stage-completion update per instance of the solved batch (J_1 after its
    mandatory block with a uniformly random observed confidence, Exp re-prediction)."""
    import torch
    import torch.distributed as dist
    import paper_2011_01112_b200 as pkg
    with torch.cuda.stream(stream):
        sched.solve_batch(inputs, out, stream)
        kept = out["kept"].clone()
        g = torch.Generator(device=dev).manual_seed(cw.seed)
        done = torch.zeros(n_inst, dtype=torch.int8, device=dev)
        observed = torch.randint(0, 1_000_001, (n_inst,), generator=g, device=dev).to(torch.uint32)
        out2 = pkg.alloc_outputs(n_inst, kept.numel(), device=dev)
        sw = torch.empty(n_inst, dtype=torch.uint8, device=dev)
        for _ in range(args.warmup):
            sched.reassign_batch(inputs, kept, done, observed, pkg.IC_UTIL_EXP, out2, sw, stream)
    stream.synchronize()
    k = args.steps or 20
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        dist.barrier()
    with ClockSampler(int(os.environ.get("LOCAL_RANK", 0))) as clk, torch.cuda.stream(stream):
        e0.record(stream)
        for _ in range(k):
            sched.reassign_batch(inputs, kept, done, observed, pkg.IC_UTIL_EXP, out2, sw, stream)
        e1.record(stream)
        e1.synchronize()
    ms = torch.tensor([e0.elapsed_time(e1)], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(ms, op=dist.ReduceOp.MAX)
    ms = float(ms.item())
    if rank == 0:
        total = cw.n_instances if strong else n_inst * world
        per_ms = ms / k
        in_bytes = sum(v.numel() * v.element_size() for v in inputs.values()) / n_inst
        io = in_bytes + 9 * inputs["release"].numel() / n_inst + 32  # descriptors + plan in/out + per-instance
        achieved = io * n_inst / (per_ms / 1e3) / 1e9
        peak = _peaks().get("hbm_gbs", 6553.3)
        print(json.dumps({
            "metric": "stage-completion updates/sec (Eq. 5 greedy reassignment)", "value": total * k / (ms / 1e3),
            "unit": "updates/s", "n_gpus": world, "steps": k, "warmup": args.warmup, "ms_per_step": per_ms,
            "higher_is_better": True, "scaling": "strong" if strong else "weak", "vs_baseline": None,
            "dtype": "int64", "data": "synthetic (device-generated, seeded)",
            "config": workload_config(cw, args, n_inst),
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s", "frac": achieved / peak,
                         "traffic": None, "work": "descriptor + plan bytes per instance (one read, one write)"},
            "gpu_launches": k, "clocks": clk.summary(),
            "swapped_fraction": float(sw.float().mean().item()),
        }), flush=True)


def run_simulate(args, rank, world, local):
    """--op simulate (NEXT-4): many independent edge servers (P:L345-356 load sweep shape) in
    lockstep; every round batches all servers' re-plans into one host-buffer GPU solve.  The
    line reports the planner's throughput and the four policies' accuracy / miss rate."""
    import torch
    import torch.distributed as dist
    import paper_2011_01112_b200 as pkg
    servers = args.instances or 2048
    kw = dict(servers=servers, clients=args.sim_clients, requests_per_client=20, n_opt=7, period=args.sim_period,
              seed=0x2011011106 + rank, device=local, delta_micro=args.delta_micro or 100_000)
    with ClockSampler(local) as clk:
        pol = {p: pkg.simulate(pkg.SimConfig(policy=p, **kw)) for p in ("planner", "edf", "lcf", "rr")}
    p = pol["planner"]
    t = torch.tensor([p["sim_seconds"], p["gpu_seconds"]], dtype=torch.float64,
                     device=torch.device("cuda", local))
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    if rank == 0:
        sec = float(t[0])
        print(json.dumps({
            "metric": "simulated requests/sec (RTDeepIoT planner, edge-server simulation)",
            "value": p["requests"] * world / sec, "unit": "requests/s", "n_gpus": world, "steps": 1,
            "warmup": 0, "ms_per_step": sec * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "int64", "data": "synthetic (seeded request traces)",
            "config": {"workload": f"sim {servers} servers x {args.sim_clients} clients x 20 requests, 8 stages, "
                                   + (f"open loop period {args.sim_period}" if args.sim_period else "closed loop"),
                       "delta_micro": kw["delta_micro"]},
            "plans_per_s": p["plans"] * world / sec, "gpu_fraction": float(t[1]) / sec,
            "policies": {k: {"accuracy": v["accuracy"], "miss_rate": v["miss_rate"],
                             "mean_depth": v["mean_depth"]} for k, v in pol.items()},
            "clocks": clk.summary(),
        }), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=None, help="timed steps (default: >= 1 s of work)")
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="C5", help="C5 (default): the 2^24-instance overload sweep the metric is quoted on at 1/2/4/8 GPUs; C1-C4 are the other BASELINE.json configs")
    ap.add_argument("--instances", type=int, default=0, help="override instances per GPU")
    ap.add_argument("--delta-micro", type=int, default=0, help="fixed Delta instead of FPTAS eps")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--sim-clients", type=int, default=20, help="--op simulate: clients per server")
    ap.add_argument("--sim-period", type=int, default=600, help="--op simulate: open-loop mean gap (0: closed loop)")
    ap.add_argument("--op", default="solve", choices=["solve", "reassign", "replan", "simulate"],
                    help="reassign: the stage-completion update (NEXT-3, Eq. 5) on the solved batch; replan: "
                         "one arrival per instance re-planned from its row (NEXT-2, needs --delta-micro); simulate: "
                         "the edge-server simulator, planner vs EDF/LCF/RR (NEXT-4)")
    ap.add_argument("--cpu-seconds", type=float, default=12.0)
    ap.add_argument("--lib", default=None, help="load libicsched from this path (A/B of two builds)")
    ap.add_argument("--tune", action="append", default=[], metavar="FIELD=VALUE",
                    help="ic_sched_tuning field for the handle (A/B of launch choices), repeatable")
    ap.add_argument("--no-probe", action="store_true", help="skip the shared-memory peak probe")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local = int(os.environ.get("LOCAL_RANK", 0))
    cw = gen.CONFIGS[args.config]

    if args.impl == "reference":
        args.steps = args.steps or 3
        run_reference(args, cw, rank, world)
        return

    import torch
    import torch.distributed as dist
    import paper_2011_01112_b200 as pkg
    from paper_2011_01112_b200.multigpu import reduce_stats, shard_range, weak_shard, derived_metrics
    if args.lib:
        pkg.use_library(args.lib)
    tuning = {k: int(v) for k, v in (t.split("=", 1) for t in args.tune)} or None

    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    strong = bool(cw.u_blocks) and not args.instances  # C5: a fixed 2^24-instance sweep split over ranks
    if strong:
        id0, id1 = shard_range(cw.n_instances, rank, world)
        n_inst = id1 - id0
        hash_id0 = id0
        spans = []  # (global id lo, hi) pieces of this rank's shard
        start = 0
        for _, cnt in cw.u_blocks:
            lo, hi = max(id0, start), min(id1, start + cnt)
            spans.append((lo, hi) if lo < hi else None)
            start += cnt
    elif cw.u_blocks:  # --instances with C5: an equal slice from the start of every U block (profiling)
        per = args.instances // len(cw.u_blocks)
        n_inst = per * len(cw.u_blocks)
        hash_id0 = 0
        spans, start = [], 0
        for _, cnt in cw.u_blocks:
            spans.append((start + rank * per, start + (rank + 1) * per))
            start += cnt
    else:
        n_inst = args.instances or cw.n_instances
        id0 = weak_shard(n_inst, rank)[0]
        hash_id0 = id0
        spans = [(id0, id0 + n_inst)]
    if args.op == "simulate":
        run_simulate(args, rank, world, local)
        if world > 1:
            dist.destroy_process_group()
        return
    stream = torch.cuda.Stream(dev)

    # ---- inputs resident in HBM: this rank's global-id shard, generated on device
    with torch.cuda.stream(stream):
        N = cw.n_tasks
        inputs = pkg.alloc_inputs(n_inst, n_inst * N, cw.n_opt, dev)
        a = 0
        for bi, span in enumerate(spans):
            if span is None:
                continue
            lo, hi = span
            u = cw.u_blocks[bi][0] if cw.u_blocks else None
            g = cw.gen_config(None, u, u) if u is not None else cw.gen_config()
            z = a + hi - lo
            view = {k: (v[a:z + 1] if k == "task_begin" else v[a * N:z * N]) for k, v in inputs.items()}
            pkg.gen_batch_device(g.seed, g.n_tasks, g.n_opt, g.opt_stride, g.horizon, g.u_lo_q16,
                                 g.u_hi_q16, g.d_lo, hi - lo, lo, device=dev, stream=stream, out=view)
            a = z
        inputs["task_begin"].copy_(torch.arange(n_inst + 1, device=dev, dtype=torch.int64) * N)
    stream.synchronize()
    T = n_inst * cw.n_tasks
    in_bytes = sum(v.numel() * v.element_size() for v in inputs.values())
    W, W_survey = algorithmic_evals(inputs, cw.n_tasks, cw.n_opt, args.delta_micro, cw.epsilon_micro)

    sc = pkg.SchedConfig(device=local, max_tasks=cw.n_tasks, max_opt_stages=cw.n_opt, max_horizon=cw.horizon,
                         delta_micro=args.delta_micro, epsilon_micro=cw.epsilon_micro)
    sched = pkg.Scheduler(sc, tuning)
    info = sched.info()
    out = pkg.alloc_outputs(n_inst, T, device=dev)
    out_bytes = sum(v.numel() * v.element_size() for k, v in out.items() if k != "stats")

    def step():
        out["stats"].zero_()
        sched.solve_batch(inputs, out, stream)
        reduce_stats(out["stats"])

    if args.op == "replan":
        run_replan(args, cw, sched, inputs, out, stream, n_inst, world, rank, dev, strong)
        sched.close()
        if world > 1:
            dist.destroy_process_group()
        return
    if args.op == "reassign":
        run_reassign(args, cw, sched, inputs, out, stream, n_inst, world, rank, dev, strong)
        sched.close()
        if world > 1:
            dist.destroy_process_group()
        return

    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            step()
    stream.synchronize()
    if args.steps is None:  # default: enough steps for >= 1 s of timed work (clock samples)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        with torch.cuda.stream(stream):
            step()
        e1.record(stream)
        e1.synchronize()
        k = max(3, int(1000.0 / max(e0.elapsed_time(e1), 1e-3)) + 1)
        kt = torch.tensor([k], device=dev)
        if world > 1:
            dist.all_reduce(kt, op=dist.ReduceOp.MAX)
        args.steps = int(kt.item())
    if world > 1:
        dist.barrier()
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    t_start, t_end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize(dev)
    with ClockSampler(local) as clk, torch.cuda.stream(stream):
        t_start.record(stream)
        for i in range(args.steps):
            out["stats"].zero_()
            ev[i][0].record(stream)
            sched.solve_batch(inputs, out, stream)
            ev[i][1].record(stream)
            reduce_stats(out["stats"])
        t_end.record(stream)
        stream.synchronize()
    torch.cuda.synchronize(dev)
    ms = t_start.elapsed_time(t_end)
    kern_ms = float(np.mean([a.elapsed_time(b) for a, b in ev]))
    tmax = torch.tensor([ms], device=dev, dtype=torch.float64)
    if world > 1:
        dist.all_reduce(tmax, op=dist.ReduceOp.MAX)
    ms = float(tmax.item())
    stats = out["stats"].cpu().numpy()
    # plans fingerprint: all_reduce(SUM) of an int64 hash keyed by global id;
    # identical at any GPU count for the strong-scaled C5 sweep
    from paper_2011_01112_b200.multigpu import result_hash
    rh = result_hash(out, inputs["task_begin"], hash_id0, cw.n_tasks).reshape(1)
    if world > 1:
        dist.all_reduce(rh)
    total_inst = cw.n_instances if strong else n_inst * world
    value = total_inst * args.steps / (ms / 1e3)

    # ---- C1-sized batches are launch-bound: per-solve latency by CUDA-graph replay
    # (SURVEY.md §8(d)); the graph holds one ic_sched_solve_batch launch on `stream`
    latency = None
    if n_inst <= 64:
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(stream):
            sched.solve_batch(inputs, out, stream)  # warm the launch path outside capture
            stream.synchronize()
            with torch.cuda.graph(g, stream=stream):
                sched.solve_batch(inputs, out, stream)
            for _ in range(20):
                g.replay()
            reps = 2000
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(stream)
            for _ in range(reps):
                g.replay()
            e1.record(stream)
        e1.synchronize()
        latency = {"graph_replay_us": e0.elapsed_time(e1) * 1e3 / reps, "launch_us": kern_ms * 1e3,
                   "instances_per_solve": n_inst}

    # ---- end to end through the public host-buffer entry point (pinned H2D + solve + D2H)
    e2e = None
    if not args.no_e2e:
        hin = {k: torch.empty(v.shape, dtype=v.dtype, pin_memory=True) for k, v in inputs.items()}
        for k in hin:
            hin[k].copy_(inputs[k])
        hout = pkg.alloc_outputs(n_inst, T, host=True, pinned=True)
        for _ in range(1):
            sched.solve_batch_host(hin, hout, stream)
        if world > 1:
            dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ke = max(2, min(args.steps, 5))
        e0.record(stream)
        for _ in range(ke):
            sched.solve_batch_host(hin, hout, stream)
        e1.record(stream)
        e1.synchronize()
        ems = torch.tensor([e0.elapsed_time(e1) / ke], device=dev, dtype=torch.float64)
        if world > 1:
            dist.all_reduce(ems, op=dist.ReduceOp.MAX)
        e2e = {"value": n_inst * world / (float(ems.item()) / 1e3), "unit": "instances/s",
               "h2d_bytes_per_step": int(in_bytes), "d2h_bytes_per_step": int(out_bytes + 64)}

    if rank == 0:
        sms = _sms()
        clk_s = clk.summary()
        fmax = _peaks().get("sm_max_mhz") or clk_s.get("sm_max_mhz") or 1965.0
        nominal_gbs = SMEM_BYTES_PER_CLK_PER_SM * sms * fmax * 1e6 / 1e9
        probe = None if args.no_probe else smem_peak(local)
        peak_gbs = probe["gbs"] if probe else nominal_gbs
        peak_basis = (f"measured: ic_probe_smem conflict-free LDS.32 stream on {sms} SMs, "
                      f"{probe['bytes_per_clk_per_sm']:.1f} B/clk/SM at {probe['modes']['lds32']['sm_mhz']:.0f} MHz "
                      "(include/ic_probe.h)") if probe else \
            f"nominal 128 B/clk/SM x {sms} SMs x {fmax:.0f} MHz (probe skipped)"
        achieved = W * BYTES_PER_EVAL / (kern_ms / 1e3) / 1e9
        traffic = None
        prof = os.path.join(ROOT, "profiles", f"ncu_{cw.name}{'d01' if args.delta_micro == 100000 else ''}_summary.json")
        if os.path.exists(prof) and (not args.delta_micro or args.delta_micro == 100000):
            try:
                ps = json.load(open(prof))
                traffic = ps.get("dram_bytes_per_instance") * n_inst
                traffic_src = f"{os.path.relpath(prof, ROOT)} ({ps.get('round', '?')}, {ps.get('kernel', '')})"
            except Exception:
                traffic = None
        # issue-rate view of the same launch (the reward axis at a fixed Delta is bound by
        # per-row and per-instance instructions, not by its evaluations): warp instructions per
        # instance from the committed ncu capture of this workload, times the batch, over the
        # live kernel time, against 4 warp instructions / clk / SM
        issue = None
        iprof = os.path.join(ROOT, "profiles", f"ncu_{cw.name}{'d01' if args.delta_micro == 100000 else ''}_summary.json")
        if os.path.exists(iprof) and (not args.delta_micro or args.delta_micro == 100000):
            try:
                ps = json.load(open(iprof))
                ipi = ps["instructions"] / ps["instances_in_capture"]
                rate = ipi * n_inst / (kern_ms / 1e3)
                ipeak = 4.0 * sms * fmax * 1e6
                issue = {"achieved": rate, "peak": ipeak, "unit": "warp instructions/s", "frac": rate / ipeak,
                         "warp_instructions_per_instance": ipi,
                         "warp_instructions_per_32_evals": ipi / (W / n_inst / 32.0),
                         "ncu_issue_pct": ps.get("issue_pct_of_peak"), "ncu_smem_pct": ps.get("smem_pct_of_peak"),
                         "source": f"{os.path.relpath(iprof, ROOT)} ({ps.get('round', '?')}, {ps.get('kernel', '')})"}
            except Exception:
                issue = None
        line = {
            "metric": METRIC, "value": value, "unit": "instances/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms / args.steps, "higher_is_better": True,
            "scaling": "strong" if strong else "weak",
            "vs_baseline": None, "dtype": "int32", "data": "synthetic (device-generated, seeded)",
            "config": dict(workload_config(cw, args, n_inst),
                           l2=f"inputs {in_bytes / 1e6:.0f} MB/GPU vs L2 126 MB" +
                              (" (larger than L2)" if in_bytes > 126e6 else " (fits L2; not flushed)"),
                           parallelism=f"instance shards x{world}"),
            "roofline": {"bound": "smem", "achieved": achieved, "peak": peak_gbs, "unit": "GB/s",
                         "frac": achieved / peak_gbs, "traffic": traffic,
                         "traffic_source": traffic_src if traffic else None,
                         "peak_basis": peak_basis, "smem_probe": probe,
                         "nominal_peak": nominal_gbs, "frac_of_nominal": achieved / nominal_gbs,
                         "frac_of_lds128": achieved / probe["modes"]["lds128"]["gbs"] if probe else None,
                         "evals_per_instance": W / n_inst, "kernel_ms": kern_ms,
                         "work": "W_active evals x 4 B (DESIGN.md §5)",
                         "survey_evals_per_instance": W_survey / n_inst,
                         "achieved_at_survey_W": W_survey * BYTES_PER_EVAL / (kern_ms / 1e3) / 1e9},
            "issue": issue,
            "gpu_launches": args.steps * int(info.get("kernels_per_solve", 1)),
            "clocks": clk_s,
            "kernel": info,
            "stats": dict(zip(pkg.STATS_FIELDS, [int(x) for x in stats])),
            "accuracy_and_misses": derived_metrics(stats),
            "result_hash": hex(int(rh.item()) & ((1 << 64) - 1)),
        }
        if e2e:
            line["e2e"] = e2e
        if latency:
            line["latency"] = latency
        if world == 1 and not args.no_cpu_baseline:
            line["cpu_baseline"] = cpu_oracle_baseline(cw, args, args.cpu_seconds)
        line["paper_context"] = PAPER_CONTEXT
        print(json.dumps(line), flush=True)
    sched.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

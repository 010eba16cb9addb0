"""ctypes marshalling for libicsched.so (include/ic_sched.h, include/ic_gen.h).

Argument marshalling only.  Device memory comes from torch tensors (their
``data_ptr()``), streams from ``torch.cuda.Stream`` (``cuda_stream``).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = os.path.join(_HERE, "libicsched.so")

IC_OK, IC_ERR_INVALID_ARG, IC_ERR_LIMIT, IC_ERR_CUDA, IC_ERR_OOM = 0, -1, -2, -3, -4
IC_DROP_ALLOWED, IC_MANDATORY_ENFORCED = 0, 1
IC_INST_OK, IC_INST_INFEASIBLE, IC_INST_BAD_INPUT, IC_INST_LIMIT = 0, 1, 2, 3

# (name, numpy dtype, per "task" | "instance" | "task_opt" | "csr")
INPUT_FIELDS = (("task_begin", np.int64, "csr"), ("release", np.int32, "task"),
                ("deadline", np.int32, "task"), ("mand_wcet", np.int32, "task"),
                ("n_opt", np.uint8, "task"), ("opt_wcet", np.int32, "task_opt"),
                ("mand_conf", np.uint32, "task"), ("opt_gain", np.int32, "task_opt"))
OUTPUT_FIELDS = (("kept", np.int8, "task"), ("start", np.int32, "task"), ("finish", np.int32, "task"),
                 ("q_total", np.int64, "instance"), ("conf_micro", np.int64, "instance"),
                 ("conf_total", np.float64, "instance"), ("makespan", np.int32, "instance"),
                 ("status", np.uint8, "instance"))
STATS_FIELDS = ("instances", "tasks", "dropped", "not_ok", "opt_kept", "opt_offered", "conf_micro",
                "q_total")

_ERR = {IC_ERR_INVALID_ARG: "invalid argument", IC_ERR_LIMIT: "beyond compiled limits",
        IC_ERR_CUDA: "CUDA error", IC_ERR_OOM: "out of device memory"}


class ICSchedError(RuntimeError):
    def __init__(self, fn, rc):
        super().__init__(f"{fn} failed: {rc} ({_ERR.get(rc, 'unknown')})")
        self.rc = rc


class SchedConfig(ctypes.Structure):
    _fields_ = [("device", ctypes.c_int32), ("drop_mode", ctypes.c_int32),
                ("delta_micro", ctypes.c_uint32), ("epsilon_micro", ctypes.c_uint32),
                ("max_tasks", ctypes.c_int32), ("max_opt_stages", ctypes.c_int32),
                ("max_horizon", ctypes.c_int32)]

    def __init__(self, device=0, drop_mode=IC_DROP_ALLOWED, delta_micro=0, epsilon_micro=100_000,
                 max_tasks=64, max_opt_stages=8, max_horizon=4096):
        super().__init__(device, drop_mode, delta_micro, epsilon_micro, max_tasks, max_opt_stages,
                         max_horizon)


TUNING_FIELDS = ("dp_warps", "pad_cols", "in_place", "slots", "decisions", "option_tables", "axis", "ckpt",
                 "ctas_per_sm", "no_vec_loads", "kernel", "packed_options", "discard")


class SchedTuning(ctypes.Structure):
    """include/ic_sched.h ic_sched_tuning: launch choices fixed at create (0 = library default)."""
    _fields_ = [(n, ctypes.c_int32) for n in TUNING_FIELDS]

    def __init__(self, **kw):
        bad = set(kw) - set(TUNING_FIELDS)
        if bad:
            raise ValueError(f"unknown tuning fields {sorted(bad)}")
        super().__init__(*[int(kw.get(n, 0)) for n in TUNING_FIELDS])


class SchedInfo(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in ("threads_per_cta", "cols_per_thread", "ctas_per_sm", "grid",
                                              "smem_bytes", "decisions_in_smem", "double_buffered",
                                              "pad_cols")] + [("workspace_bytes", ctypes.c_int64)] + \
        [(n, ctypes.c_int32) for n in ("kernels_per_solve", "hybrid", "packed_options")]

    def as_dict(self):
        return {n: getattr(self, n) for n, _ in self._fields_}


class _In(ctypes.Structure):
    _fields_ = [("n_instances", ctypes.c_int64)] + [(n, ctypes.c_void_p) for n, _, _ in INPUT_FIELDS]


class _Out(ctypes.Structure):
    _fields_ = [(n, ctypes.c_void_p) for n, _, _ in OUTPUT_FIELDS] + [("stats", ctypes.c_void_p)]


class _GenCfg(ctypes.Structure):
    _fields_ = [("seed", ctypes.c_uint64), ("n_tasks", ctypes.c_int32), ("n_opt", ctypes.c_int32),
                ("opt_stride", ctypes.c_int32), ("horizon", ctypes.c_int32), ("u_lo_q16", ctypes.c_int32),
                ("u_hi_q16", ctypes.c_int32), ("d_lo", ctypes.c_int32), ("release_mode", ctypes.c_int32)]


EXPORTED = ("ic_sched_create", "ic_sched_create_tuned", "ic_sched_solve_batch", "ic_sched_solve_batch_host", "ic_sched_destroy",
            "ic_sched_get_info", "ic_gen_batch_device", "ic_sched_reassign_batch", "ic_sched_state_bytes",
            "ic_sched_solve_batch_state", "ic_sched_replan_batch", "ic_sched_depart_batch", "ic_sim_run", "ic_sim_run_dump",
            "ic_probe_smem")

IC_UTIL_GIVEN, IC_UTIL_MAX, IC_UTIL_EXP, IC_UTIL_LIN = 0, 1, 2, 3


class _Upd(ctypes.Structure):
    _fields_ = [("kept", ctypes.c_void_p), ("done", ctypes.c_void_p), ("observed", ctypes.c_void_p),
                ("heuristic", ctypes.c_int32)]

IC_SIM_PLANNER, IC_SIM_EDF, IC_SIM_LCF, IC_SIM_RR = 0, 1, 2, 3
IC_SIM_UTIL_EXP, IC_SIM_UTIL_ORACLE = 0, 1
SIM_POLICIES = {"planner": IC_SIM_PLANNER, "edf": IC_SIM_EDF, "lcf": IC_SIM_LCF, "rr": IC_SIM_RR}


class SimConfig(ctypes.Structure):
    """include/ic_sim.h ic_sim_config."""
    _fields_ = [("servers", ctypes.c_int32), ("clients", ctypes.c_int32),
                ("requests_per_client", ctypes.c_int32), ("n_opt", ctypes.c_int32),
                ("wcet_base", ctypes.c_int32), ("d_lo", ctypes.c_int32), ("d_hi", ctypes.c_int32),
                ("think", ctypes.c_int32), ("seed", ctypes.c_uint64), ("policy", ctypes.c_int32),
                ("utility", ctypes.c_int32), ("delta_micro", ctypes.c_uint32), ("prior_micro", ctypes.c_uint32),
                ("device", ctypes.c_int32), ("period", ctypes.c_int32), ("plan_cells_per_tick", ctypes.c_int32)]

    def __init__(self, servers=1, clients=20, requests_per_client=50, n_opt=7, wcet_base=10, d_lo=10,
                 d_hi=300, think=1, seed=0x2011011106, policy=IC_SIM_PLANNER, utility=IC_SIM_UTIL_EXP,
                 delta_micro=100_000, prior_micro=500_000, device=0, period=0, plan_cells_per_tick=0):
        if isinstance(policy, str):
            policy = SIM_POLICIES[policy]
        super().__init__(servers, clients, requests_per_client, n_opt, wcet_base, d_lo, d_hi, think, seed,
                         policy, utility, delta_micro, prior_micro, device, period, plan_cells_per_tick)


class SimResult(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int64) for n in ("requests", "misses", "stages_run", "plans", "rounds",
                                              "conf_micro")] + \
               [(n, ctypes.c_double) for n in ("accuracy", "miss_rate", "mean_depth", "sim_seconds",
                                               "gpu_seconds")] + \
               [(n, ctypes.c_int64) for n in ("plan_ticks", "busy_ticks")]

    def as_dict(self):
        return {n: getattr(self, n) for n, _ in self._fields_}


_DUMP_FIELDS = (("task_begin", np.int64, "csr"), ("release", np.int32, "task"), ("deadline", np.int32, "task"),
                ("mand_wcet", np.int32, "task"), ("n_opt", np.uint8, "task"), ("opt_wcet", np.int32, "task_opt"),
                ("mand_conf", np.uint32, "task"), ("opt_gain", np.int32, "task_opt"), ("kept", np.int8, "task"),
                ("start", np.int32, "task"), ("finish", np.int32, "task"), ("q_total", np.int64, "instance"),
                ("conf_micro", np.int64, "instance"), ("makespan", np.int32, "instance"),
                ("status", np.uint8, "instance"))


class _SimDump(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int64) for n in ("cap_instances", "cap_tasks", "n_instances", "n_tasks")] + \
               [(n, ctypes.c_void_p) for n, _, _ in _DUMP_FIELDS]


def simulate(cfg: SimConfig, dump_instances: int = 0, dump_tasks: int = 0):
    """ic_sim_run: event-driven edge-server simulation (include/ic_sim.h, NEXT-4).

    With dump_instances > 0 (ic_sim_run_dump) also returns the first planner batches the
    simulator sent to the solver: inputs in the ic_batch_in layout and the solver's outputs."""
    lib = load_library()
    r = SimResult()
    if not dump_instances:
        rc = lib.ic_sim_run(ctypes.byref(cfg), ctypes.byref(r))
        if rc != 0:
            raise ICSchedError("ic_sim_run", rc)
        return r.as_dict()
    cap_t = dump_tasks or dump_instances * cfg.clients * 4
    bufs = {n: np.zeros(((cap_t, cfg.n_opt) if k == "task_opt" else
                         (dump_instances + 1 if k == "csr" else cap_t if k == "task" else dump_instances)), dt)
            for n, dt, k in _DUMP_FIELDS}
    d = _SimDump(dump_instances, cap_t, 0, 0, *[_ptr(bufs[n]) if bufs[n].size else None for n, _, _ in _DUMP_FIELDS])
    rc = lib.ic_sim_run_dump(ctypes.byref(cfg), ctypes.byref(r), ctypes.byref(d))
    if rc != 0:
        raise ICSchedError("ic_sim_run_dump", rc)
    B, T = d.n_instances, d.n_tasks
    out = {n: (v[:B + 1] if n == "task_begin" else v[:B] if k == "instance" else v[:T]) for (n, _, k), v in
           zip(_DUMP_FIELDS, [bufs[n] for n, _, _ in _DUMP_FIELDS])}
    return r.as_dict(), out


PROBE_MODES = {"lds32": 0, "lds128": 1, "lds32_viaddmax": 2}


def probe_smem(device: int = 0, mode: str = "lds32", target_ms: float = 50.0) -> dict:
    """ic_probe_smem (include/ic_probe.h): measured shared-memory load bandwidth of `device`."""
    lib = load_library()
    bps, bpc, clk = ctypes.c_double(), ctypes.c_double(), ctypes.c_double()
    rc = lib.ic_probe_smem(device, PROBE_MODES[mode], target_ms, ctypes.byref(bps), ctypes.byref(bpc),
                           ctypes.byref(clk))
    if rc != 0:
        raise ICSchedError("ic_probe_smem", rc)
    return {"mode": mode, "gbs": bps.value / 1e9, "bytes_per_clk_per_sm": bpc.value, "sm_mhz": clk.value / 1e6}


_lib = None


def lib_path() -> str:
    return _LIB


def use_library(path: str) -> None:
    """Load the library from an explicit path instead of the in-tree build (A/B comparisons
    of two builds in tools/ and bench.py --lib).  Must be called before the first load."""
    global _LIB
    if _lib is not None and os.path.abspath(path) != _LIB:
        raise RuntimeError("libicsched already loaded from " + _LIB)
    _LIB = os.path.abspath(path)


def load_library():
    """Load libicsched.so; raise loudly if it was not built (no fallback exists)."""
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB):
            raise ImportError(f"{_LIB} is missing: run `python __graft_entry__.py build` "
                              "(the solver has no CPU fallback)")
        lib = ctypes.CDLL(_LIB)
        P = ctypes.POINTER
        lib.ic_sched_create.argtypes = [P(SchedConfig), P(ctypes.c_void_p)]
        lib.ic_sched_create_tuned.argtypes = [P(SchedConfig), P(SchedTuning), P(ctypes.c_void_p)]
        lib.ic_sched_solve_batch.argtypes = [ctypes.c_void_p, P(_In), P(_Out), ctypes.c_void_p]
        lib.ic_sched_solve_batch_host.argtypes = [ctypes.c_void_p, P(_In), P(_Out), ctypes.c_void_p]
        lib.ic_sched_destroy.argtypes = [ctypes.c_void_p]
        lib.ic_sched_get_info.argtypes = [ctypes.c_void_p, P(SchedInfo)]
        lib.ic_gen_batch_device.argtypes = [P(_GenCfg), ctypes.c_int64, ctypes.c_int64] + \
            [ctypes.c_void_p] * 9
        lib.ic_sched_reassign_batch.argtypes = [ctypes.c_void_p, P(_In), P(_Upd), P(_Out), ctypes.c_void_p,
                                                ctypes.c_void_p]
        lib.ic_sched_solve_batch_state.argtypes = [ctypes.c_void_p, P(_In), P(_Out), ctypes.c_void_p,
                                                   ctypes.c_void_p]
        lib.ic_sched_replan_batch.argtypes = [ctypes.c_void_p, P(_In), ctypes.c_void_p, P(_Out), ctypes.c_void_p]
        lib.ic_sched_depart_batch.argtypes = [ctypes.c_void_p, P(_In)] + [ctypes.c_void_p] * 4 + \
            [P(_Out), ctypes.c_void_p]
        lib.ic_sched_state_bytes.argtypes = [ctypes.c_void_p, ctypes.c_int64]
        lib.ic_sim_run.argtypes = [P(SimConfig), P(SimResult)]
        lib.ic_sim_run_dump.argtypes = [P(SimConfig), P(SimResult), P(_SimDump)]
        lib.ic_probe_smem.argtypes = [ctypes.c_int32, ctypes.c_int32, ctypes.c_double, P(ctypes.c_double),
                                      P(ctypes.c_double), P(ctypes.c_double)]
        for f in EXPORTED:
            getattr(lib, f).restype = ctypes.c_int
        lib.ic_sched_state_bytes.restype = ctypes.c_int64
        _lib = lib
    return _lib


def _torch_dtype(dt):
    import torch
    return torch.from_numpy(np.zeros(0, dt)).dtype


def _ptr(x):
    """Device (torch) or host (numpy) buffer -> void*."""
    if x is None:
        return None
    if hasattr(x, "data_ptr"):
        return ctypes.c_void_p(x.data_ptr()) if x.numel() else None
    return ctypes.c_void_p(x.ctypes.data) if x.size else None


def _n_instances(inputs) -> int:
    tb = inputs["task_begin"]
    return (tb.numel() if hasattr(tb, "numel") else tb.size) - 1


def alloc_outputs(n_instances: int, n_tasks: int, device="cuda", pinned: bool = False, host=False) -> dict:
    """Output buffers in the ABI layout: torch CUDA tensors, or host numpy / pinned torch."""
    import torch
    out = {}
    for name, dt, kind in OUTPUT_FIELDS:
        n = n_tasks if kind == "task" else n_instances
        tdt = torch.from_numpy(np.zeros(0, dt)).dtype
        if host:
            out[name] = torch.empty(n, dtype=tdt, pin_memory=pinned)
        else:
            out[name] = torch.empty(n, dtype=tdt, device=device)
    if host:
        out["stats"] = torch.zeros(8, dtype=torch.int64, pin_memory=pinned)
    else:
        out["stats"] = torch.zeros(8, dtype=torch.int64, device=device)
    return out


class Scheduler:
    """One ic_sched handle (bound to a device; one stream at a time)."""

    def __init__(self, cfg: SchedConfig, tuning: SchedTuning | dict | None = None):
        self._lib = load_library()
        self.cfg = cfg
        h = ctypes.c_void_p()
        if tuning is None:
            rc = self._lib.ic_sched_create(ctypes.byref(cfg), ctypes.byref(h))
        else:
            if isinstance(tuning, dict):
                tuning = SchedTuning(**tuning)
            rc = self._lib.ic_sched_create_tuned(ctypes.byref(cfg), ctypes.byref(tuning), ctypes.byref(h))
        if rc != IC_OK:
            raise ICSchedError("ic_sched_create", rc)
        self._h = h

    def info(self) -> dict:
        i = SchedInfo()
        rc = self._lib.ic_sched_get_info(self._h, ctypes.byref(i))
        if rc != IC_OK:
            raise ICSchedError("ic_sched_get_info", rc)
        return i.as_dict()

    def _check(self, inputs, outputs):
        """Layout checks the C ABI cannot make: dtype, contiguity, one device, and the
        (T, max_opt_stages) row stride of the optional-stage arrays (the kernel indexes
        row t at t * max_opt_stages, so any other stride would read the wrong stages)."""
        dev = None
        B = _n_instances(inputs)
        for fields, bufs in ((INPUT_FIELDS, inputs), (OUTPUT_FIELDS, outputs)):
            for name, dt, kind in fields:
                x = bufs[name]
                if hasattr(x, "data_ptr"):
                    ok_dt = x.dtype == _torch_dtype(dt)
                    contig = x.is_contiguous()
                    d = str(x.device)
                    shape = tuple(x.shape)
                else:
                    ok_dt = x.dtype == np.dtype(dt)
                    contig = x.flags.c_contiguous
                    d = "cpu"
                    shape = x.shape
                if not ok_dt:
                    raise TypeError(f"{name}: dtype {x.dtype}, expected {np.dtype(dt)}")
                if not contig:
                    raise ValueError(f"{name}: must be contiguous")
                if dev is None:
                    dev = d
                elif d != dev:
                    raise ValueError(f"{name}: on {d}, other buffers on {dev}")
                if kind == "task_opt" and (len(shape) != 2 or shape[1] != self.cfg.max_opt_stages):
                    raise ValueError(f"{name}: shape {shape}, expected (T, {self.cfg.max_opt_stages})")
                if kind == "instance" and shape[0] < B:
                    raise ValueError(f"{name}: {shape[0]} entries for {B} instances")
        return dev

    def _marshal(self, inputs, outputs):
        self._check(inputs, outputs)
        i = _In(_n_instances(inputs), *[_ptr(inputs[n]) for n, _, _ in INPUT_FIELDS])
        o = _Out(*[_ptr(outputs[n]) for n, _, _ in OUTPUT_FIELDS], _ptr(outputs.get("stats")))
        return i, o

    def solve_batch(self, inputs: dict, outputs: dict | None = None, stream=None) -> dict:
        """ic_sched_solve_batch on CUDA tensors; asynchronous on `stream` (torch.cuda.Stream)."""
        import torch
        if outputs is None:
            outputs = alloc_outputs(_n_instances(inputs), inputs["release"].numel(),
                                    device=inputs["release"].device)
        if stream is None:
            stream = torch.cuda.current_stream()
        i, o = self._marshal(inputs, outputs)
        rc = self._lib.ic_sched_solve_batch(self._h, ctypes.byref(i), ctypes.byref(o),
                                            ctypes.c_void_p(stream.cuda_stream))
        if rc != IC_OK:
            raise ICSchedError("ic_sched_solve_batch", rc)
        return outputs

    def solve_batch_host(self, inputs: dict, outputs: dict, stream=None) -> dict:
        """ic_sched_solve_batch_host on host buffers (numpy or pinned torch); synchronous."""
        import torch
        if stream is None:
            stream = torch.cuda.current_stream()
        i, o = self._marshal(inputs, outputs)
        rc = self._lib.ic_sched_solve_batch_host(self._h, ctypes.byref(i), ctypes.byref(o),
                                                 ctypes.c_void_p(stream.cuda_stream))
        if rc != IC_OK:
            raise ICSchedError("ic_sched_solve_batch_host", rc)
        return outputs

    def reassign_batch(self, inputs: dict, kept, done, observed, heuristic: int = IC_UTIL_EXP,
                       outputs: dict | None = None, swapped=None, stream=None):
        """ic_sched_reassign_batch (stage completion, Eq. 5) on CUDA tensors; asynchronous."""
        import torch
        if outputs is None:
            outputs = alloc_outputs(_n_instances(inputs), inputs["release"].numel(),
                                    device=inputs["release"].device)
        if swapped is None:
            swapped = torch.empty(_n_instances(inputs), dtype=torch.uint8, device=inputs["release"].device)
        if stream is None:
            stream = torch.cuda.current_stream()
        i, o = self._marshal(inputs, outputs)
        u = _Upd(_ptr(kept), _ptr(done), _ptr(observed), heuristic)
        rc = self._lib.ic_sched_reassign_batch(self._h, ctypes.byref(i), ctypes.byref(u), ctypes.byref(o),
                                               _ptr(swapped), ctypes.c_void_p(stream.cuda_stream))
        if rc != IC_OK:
            raise ICSchedError("ic_sched_reassign_batch", rc)
        outputs["swapped"] = swapped
        return outputs

    def state_bytes(self, n_instances: int) -> int:
        """Device bytes of re-plan state for n_instances (ic_sched_state_bytes)."""
        v = self._lib.ic_sched_state_bytes(self._h, n_instances)
        if v < 0:
            raise ICSchedError("ic_sched_state_bytes", int(v))
        return int(v)

    def solve_batch_state(self, inputs: dict, state, outputs: dict | None = None, stream=None) -> dict:
        """ic_sched_solve_batch_state: solve and keep every DP row in `state` (uint8 CUDA tensor)."""
        return self._state_call("ic_sched_solve_batch_state", inputs, state, outputs, stream)

    def replan_batch(self, inputs: dict, state, outputs: dict | None = None, stream=None) -> dict:
        """ic_sched_replan_batch: each instance gained one task (appended last); re-plan from its row."""
        return self._state_call("ic_sched_replan_batch", inputs, state, outputs, stream)

    def depart_batch(self, inputs: dict, removed_index, removed_deadline, removed_release, state,
                     outputs: dict | None = None, stream=None) -> dict:
        """ic_sched_depart_batch: each instance lost one task (its previous input index, deadline
        and release given per instance as int32 CUDA tensors); re-plan from its old EDF row."""
        import torch
        if outputs is None:
            outputs = alloc_outputs(_n_instances(inputs), inputs["release"].numel(),
                                    device=inputs["release"].device)
        if stream is None:
            stream = torch.cuda.current_stream()
        for x in (removed_index, removed_deadline, removed_release):
            if x.dtype != torch.int32 or not x.is_contiguous() or x.numel() < _n_instances(inputs):
                raise ValueError("removed_* must be contiguous int32 tensors with one entry per instance")
        i, o = self._marshal(inputs, outputs)
        rc = self._lib.ic_sched_depart_batch(self._h, ctypes.byref(i), _ptr(removed_index), _ptr(removed_deadline),
                                             _ptr(removed_release), _ptr(state), ctypes.byref(o),
                                             ctypes.c_void_p(stream.cuda_stream))
        if rc != IC_OK:
            raise ICSchedError("ic_sched_depart_batch", rc)
        return outputs

    def _state_call(self, fn, inputs, state, outputs, stream):
        import torch
        if outputs is None:
            outputs = alloc_outputs(_n_instances(inputs), inputs["release"].numel(),
                                    device=inputs["release"].device)
        if stream is None:
            stream = torch.cuda.current_stream()
        i, o = self._marshal(inputs, outputs)
        if fn == "ic_sched_replan_batch":
            rc = self._lib.ic_sched_replan_batch(self._h, ctypes.byref(i), _ptr(state), ctypes.byref(o),
                                                 ctypes.c_void_p(stream.cuda_stream))
        else:
            rc = self._lib.ic_sched_solve_batch_state(self._h, ctypes.byref(i), ctypes.byref(o), _ptr(state),
                                                      ctypes.c_void_p(stream.cuda_stream))
        if rc != IC_OK:
            raise ICSchedError(fn, rc)
        return outputs

    def close(self):
        if getattr(self, "_h", None):
            self._lib.ic_sched_destroy(self._h)
            self._h = None

    __del__ = close

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


def alloc_inputs(n_instances: int, n_tasks_total: int, opt_stride: int, device="cuda") -> dict:
    """Empty input buffers in the ABI layout on a CUDA device."""
    import torch
    B, T = int(n_instances), int(n_tasks_total)
    return {n: torch.empty((T, opt_stride) if k == "task_opt" else (B + 1 if k == "csr" else T),
                           dtype=torch.from_numpy(np.zeros(0, dt)).dtype, device=torch.device(device))
            for n, dt, k in INPUT_FIELDS}


def gen_batch_device(seed, n_tasks, n_opt, opt_stride, horizon, u_lo_q16, u_hi_q16, d_lo, n_instances,
                     id_offset=0, release_mode=0, device="cuda", stream=None, out: dict | None = None) -> dict:
    """ic_gen_batch_device: generate instances [id_offset, id_offset+n) on the GPU (ABI layout).

    With ``out`` (tensors or views of at least the batch's size) the rows are written there;
    its task_begin then holds offsets relative to the first generated row."""
    import torch
    lib = load_library()
    B, T = int(n_instances), int(n_instances) * int(n_tasks)
    dev = torch.device(device)
    t = out if out is not None else alloc_inputs(B, T, opt_stride, dev)
    g = _GenCfg(seed, n_tasks, n_opt, opt_stride, horizon, u_lo_q16, u_hi_q16, d_lo, release_mode)
    if stream is None:
        stream = torch.cuda.current_stream(dev)
    rc = lib.ic_gen_batch_device(ctypes.byref(g), id_offset, B, *[_ptr(t[n]) for n, _, _ in INPUT_FIELDS],
                                 ctypes.c_void_p(stream.cuda_stream))
    if rc != 0:
        raise ICSchedError("ic_gen_batch_device", rc)
    return t


def to_micro(x, dtype=None):
    """Float confidences (or gains) in [0, 1] -> integer micro-units, round half to even
    (SURVEY.md §8(b) "Wrapper": ``torch.round(x * 1e6)``; D5 / G11: q = R_µ div Δ_µ needs the
    decimal value, which binary floating point only reaches after rounding to micro-units).

    ``x``: a torch tensor or anything ``torch.as_tensor`` takes; computed in float64.
    Returns ``dtype`` (default int32, the ``opt_gain`` layout; use torch.uint32 for
    ``mand_conf``) on x's device.  Raises ValueError on NaN/inf or values that overflow dtype."""
    import torch
    t = torch.as_tensor(x)
    t = t.to(torch.float64)
    if not bool(torch.isfinite(t).all()):
        raise ValueError("to_micro: non-finite confidence")
    m = torch.round(t * 1e6)  # torch.round rounds half to even
    dt = torch.int32 if dtype is None else dtype
    lo, hi = (0, 2**32 - 1) if dt == torch.uint32 else (-2**31, 2**31 - 1)
    if m.numel() and (float(m.min()) < lo or float(m.max()) > hi):
        raise ValueError(f"to_micro: value outside the {dt} range")
    return m.to(torch.int64).to(dt)


def confidences_to_inputs(mand_conf, stage_conf):
    """Float confidence curves -> the ABI's micro-unit fields.

    ``mand_conf`` [T]: confidence after the mandatory stage; ``stage_conf`` [T, S]: confidence
    after each optional stage (cumulative, P:L48 R_i^L).  Returns (mand_conf uint32 [T],
    opt_gain int32 [T, S]) where opt_gain[:, l] = micro(conf after stage l) - micro(conf
    before it), so the prefix sums R_i(k) reproduce the rounded cumulative curve exactly."""
    import torch
    m = to_micro(mand_conf, torch.int64)
    c = to_micro(stage_conf, torch.int64)
    if c.dim() != 2 or m.dim() != 1 or c.shape[0] != m.shape[0]:
        raise ValueError("confidences_to_inputs: expected mand_conf [T] and stage_conf [T, S]")
    prev = torch.cat([m[:, None], c[:, :-1]], dim=1)
    return m.to(torch.uint32), (c - prev).to(torch.int32)

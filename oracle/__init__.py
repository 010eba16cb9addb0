"""CPU oracle for the batched depth assignment — TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package.  The
product path (``paper_2011_01112_b200``) never imports it and shares no code
with it; the one common module is the input generator ``gen/``.

Layers (each pinned in ``tests/test_oracle_*.py``):

* :mod:`oracle.definition` — the canonical problem written out in pure
  Python and solved by enumeration (tiny inputs only).
* ``oracle/ic_oracle.c`` (``liboracle.so``) — O1 brute force, O2 the paper's
  reward-indexed DP (Eqs. 1-2, Alg. 1), O3 the time-indexed dual,
  and the invariant checker.  Plain C, OpenMP over instances.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
# bench.py's CPU baseline builds a copy tuned for the host it runs on (-march=native) at run
# time; the portable build is the one the tests load (it travels to the GPU box prebuilt)
_LIB_NATIVE = os.path.join(_HERE, "liboracle_native.so")

BRUTE, PAPER, TIME = 1, 2, 3
OK, INFEASIBLE, BAD_INPUT = 0, 1, 2


@dataclass(frozen=True)
class OracleConfig:
    drop_mode: int = 0          # 0 drop allowed, 1 mandatory enforced
    delta_micro: int = 0        # > 0: fixed Delta (micro-units)
    epsilon_micro: int = 100_000  # iff delta_micro == 0: Delta = eps R / N (Theorem 1)
    max_tasks: int = 4096
    max_opt_stages: int = 14
    max_horizon: int = 1 << 20


class _Cfg(ctypes.Structure):
    _fields_ = [("drop_mode", ctypes.c_int32), ("delta_micro", ctypes.c_uint32),
                ("epsilon_micro", ctypes.c_uint32), ("max_tasks", ctypes.c_int32),
                ("max_opt_stages", ctypes.c_int32), ("max_horizon", ctypes.c_int32)]


class _In(ctypes.Structure):
    _fields_ = [("n_instances", ctypes.c_int64)] + [
        (n, ctypes.c_void_p) for n in ("task_begin", "release", "deadline", "mand_wcet", "n_opt",
                                       "opt_wcet", "mand_conf", "opt_gain")]


class _Out(ctypes.Structure):
    _fields_ = [(n, ctypes.c_void_p) for n in ("kept", "start", "finish", "q_total", "conf_micro",
                                               "makespan", "status", "delta_used")]


def build(force: bool = False, native: bool = False) -> str:
    src = os.path.join(_HERE, "ic_oracle.c")
    path = _LIB_NATIVE if native else _LIB_PATH
    if force or native or not os.path.exists(path) or os.path.getmtime(path) < os.path.getmtime(src):
        flags = ["-O3", "-march=native"] if native else ["-O3"]
        subprocess.check_call(["gcc", *flags, "-std=c11", "-fopenmp", "-shared", "-fPIC", "-o", path, src])
    return path


_lib = None


def use_native_build() -> str:
    """Rebuild the oracle for this host's CPU (-O3 -march=native) and load that copy; used by
    bench.py's CPU baseline only.  Must run before the first solve."""
    global _lib
    assert _lib is None, "oracle already loaded"
    path = build(native=True)
    _lib = _bind(ctypes.CDLL(path))
    return path


def _load():
    global _lib
    if _lib is None:
        build()
        _lib = _bind(ctypes.CDLL(_LIB_PATH))
    return _lib


def _bind(_lib):
    _lib.or_solve_batch.argtypes = [ctypes.c_int, ctypes.POINTER(_Cfg), ctypes.POINTER(_In),
                                    ctypes.POINTER(_Out), ctypes.c_int]
    _lib.or_solve_batch.restype = ctypes.c_int
    for f in (_lib.or_paper_table, _lib.or_time_table):
        f.argtypes = [ctypes.POINTER(_Cfg), ctypes.POINTER(_In), ctypes.c_int64,
                      ctypes.c_void_p, ctypes.c_int64]
        f.restype = ctypes.c_int64
    _lib.or_check.argtypes = [ctypes.POINTER(_Cfg), ctypes.POINTER(_In), ctypes.POINTER(_Out),
                              ctypes.c_int64]
    _lib.or_check.restype = ctypes.c_int
    return _lib


def _p(a):
    return ctypes.c_void_p(a.ctypes.data) if a is not None and a.size else None


def _cfg(cfg: OracleConfig, batch) -> _Cfg:
    return _Cfg(cfg.drop_mode, cfg.delta_micro, cfg.epsilon_micro, cfg.max_tasks,
                batch.opt_stride, cfg.max_horizon)


def _in(batch) -> _In:
    b = batch
    for a in (b.opt_wcet, b.opt_gain):
        assert a.flags.c_contiguous
    return _In(b.n_instances, _p(b.task_begin), _p(b.release), _p(b.deadline), _p(b.mand_wcet),
               _p(b.n_opt), _p(b.opt_wcet), _p(b.mand_conf), _p(b.opt_gain))


def _alloc_out(batch) -> dict:
    T, B = batch.n_total_tasks, batch.n_instances
    return dict(kept=np.zeros(T, np.int8), start=np.zeros(T, np.int32),
                finish=np.zeros(T, np.int32), q_total=np.zeros(B, np.int64),
                conf_micro=np.zeros(B, np.int64), makespan=np.zeros(B, np.int32),
                status=np.zeros(B, np.uint8), delta_used=np.zeros(B, np.int64))


def _out(o: dict) -> _Out:
    return _Out(*[_p(o[k]) for k in ("kept", "start", "finish", "q_total", "conf_micro", "makespan",
                                     "status", "delta_used")])


def solve(batch, cfg: OracleConfig = OracleConfig(), algo: int = PAPER, threads: int = 0) -> dict:
    """Solve every instance; returns the C-ABI outputs as numpy arrays.

    Adds ``conf_total`` = conf_micro / 1e6 (float64) like the ABI does."""
    lib = _load()
    o = _alloc_out(batch)
    c, i = _cfg(cfg, batch), _in(batch)
    rc = lib.or_solve_batch(algo, ctypes.byref(c), ctypes.byref(i), ctypes.byref(_out(o)), threads)
    if rc == -2:
        raise ValueError("brute force cap (1e7 vectors) exceeded")
    if rc != 0:
        raise ValueError(f"or_solve_batch failed ({rc})")
    o["conf_total"] = o["conf_micro"].astype(np.float64) / 1e6
    return o


def _table(fn, batch, cfg, b, cap):
    lib = _load()
    buf = np.zeros(cap, np.int64)
    cols = getattr(lib, fn)(ctypes.byref(_cfg(cfg, batch)), ctypes.byref(_in(batch)), b, _p(buf), cap)
    if cols < 0:
        raise ValueError("bad input or table too large")
    n = int(batch.task_begin[b + 1] - batch.task_begin[b])
    return buf[: cols * (n + 1)].reshape(n + 1, cols)


def paper_table(batch, cfg: OracleConfig, b: int = 0, cap: int = 1 << 24) -> np.ndarray:
    """P(i, r) of Eq. 2 (rows in EDF order, row 0 = empty prefix); INT64_MAX = infinity."""
    return _table("or_paper_table", batch, cfg, b, cap)


def time_table(batch, cfg: OracleConfig, b: int = 0, cap: int = 1 << 24) -> np.ndarray:
    """G_i(t) of the time-indexed dual (rows in EDF order); INT64_MIN/4 = infeasible."""
    return _table("or_time_table", batch, cfg, b, cap)


CHECK_BITS = {1: "start<release", 2: "finish!=start+C", 4: "finish>deadline", 8: "overlap",
              16: "processor-demand", 32: "drop-in-enforced", 64: "Q/conf/makespan mismatch",
              128: "kept encoding"}


def check(batch, result: dict, cfg: OracleConfig) -> np.ndarray:
    """Invariant-check every instance of a result (oracle's or the GPU's).

    Returns an int array of violation bit masks (0 = valid), see CHECK_BITS."""
    lib = _load()
    o = {k: np.ascontiguousarray(result[k]) for k in ("kept", "start", "finish", "q_total",
                                                       "conf_micro", "makespan", "status")}
    o["delta_used"] = None
    c, i, oo = _cfg(cfg, batch), _in(batch), _out(o)
    return np.array([lib.or_check(ctypes.byref(c), ctypes.byref(i), ctypes.byref(oo), b)
                     for b in range(batch.n_instances)], np.int64)


# ---------------------------------------------------------------- NEXT-3 (stage completion)
UTIL_GIVEN, UTIL_MAX, UTIL_EXP, UTIL_LIN = 0, 1, 2, 3


def predict_next(heuristic: int, r_cur: int, p_cur: int, p_next: int) -> int:
    """One step of the Max / Exp / Lin utility heuristics, micro-units."""
    lib = _load()
    lib.or_predict_next.argtypes = [ctypes.c_int, ctypes.c_int64, ctypes.c_int64, ctypes.c_int64]
    lib.or_predict_next.restype = ctypes.c_int64
    return int(lib.or_predict_next(heuristic, r_cur, p_cur, p_next))


def reassign(batch, kept, done, observed, heuristic: int, cfg: OracleConfig = OracleConfig()) -> dict:
    """Greedy depth reassignment of Eq. 5 after the EDF-current task's stage
    completion.  kept: current plan [T] int8; done / observed: per instance."""
    lib = _load()
    lib.or_reassign_batch.argtypes = [ctypes.POINTER(_Cfg), ctypes.POINTER(_In), ctypes.c_void_p,
                                      ctypes.c_void_p, ctypes.c_void_p, ctypes.c_int, ctypes.POINTER(_Out),
                                      ctypes.c_void_p]
    lib.or_reassign_batch.restype = ctypes.c_int
    o = _alloc_out(batch)
    sw = np.zeros(batch.n_instances, np.uint8)
    kept = np.ascontiguousarray(kept, np.int8)
    done = np.ascontiguousarray(done, np.int8)
    observed = np.ascontiguousarray(observed, np.uint32)
    rc = lib.or_reassign_batch(ctypes.byref(_cfg(cfg, batch)), ctypes.byref(_in(batch)), _p(kept), _p(done),
                               _p(observed), heuristic, ctypes.byref(_out(o)), _p(sw))
    if rc != 0:
        raise ValueError(f"or_reassign_batch failed ({rc})")
    o["conf_total"] = o["conf_micro"].astype(np.float64) / 1e6
    o["swapped"] = sw
    return o

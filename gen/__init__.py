"""Seeded synthetic inputs for the solver and the oracle (input plumbing only).

This package is the one module both sides of the parity check may use
(task brief ③): it produces task sets in the C-ABI input layout of
``include/ic_sched.h`` and holds none of the method's arithmetic.

* :func:`generate` — the paper-shaped workload through the
  integer-only Philox generator in ``gen/ic_gen_core.h`` (host build
  ``gen/libicgen.so``; the CUDA library compiles the same header for
  on-device generation, so both produce identical bytes).
* :func:`tiny_random` — small adversarial instances for oracle pins and
  parity edge cases: variable N and S_i, releases, non-monotone confidence,
  equal deadlines, infeasible tasks.
* :data:`CONFIGS` — the BASELINE.json configurations C1–C5.
"""
from __future__ import annotations

import ctypes
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libicgen.so")


class GenConfig(ctypes.Structure):
    _fields_ = [
        ("seed", ctypes.c_uint64),
        ("n_tasks", ctypes.c_int32),
        ("n_opt", ctypes.c_int32),
        ("opt_stride", ctypes.c_int32),
        ("horizon", ctypes.c_int32),
        ("u_lo_q16", ctypes.c_int32),
        ("u_hi_q16", ctypes.c_int32),
        ("d_lo", ctypes.c_int32),
        ("release_mode", ctypes.c_int32),
    ]


@dataclass(frozen=True)
class WorkloadConfig:
    """One BASELINE.json configuration."""

    name: str
    n_instances: int
    n_tasks: int
    n_opt: int
    horizon: int
    u_lo: float
    u_hi: float
    d_lo: int
    seed: int
    epsilon_micro: int = 100_000  # FPTAS eps = 0.1 (D7)
    delta_micro: int = 0
    release_mode: int = 0
    u_blocks: tuple = field(default=())  # C5: (U, count) blocks

    def gen_config(self, opt_stride: int | None = None, u_lo=None, u_hi=None) -> GenConfig:
        lo = self.u_lo if u_lo is None else u_lo
        hi = self.u_hi if u_hi is None else u_hi
        return GenConfig(
            seed=self.seed,
            n_tasks=self.n_tasks,
            n_opt=self.n_opt,
            opt_stride=self.n_opt if opt_stride is None else opt_stride,
            horizon=self.horizon,
            u_lo_q16=int(round(lo * 65536)),
            u_hi_q16=int(round(hi * 65536)),
            d_lo=self.d_lo,
            release_mode=self.release_mode,
        )


def _d_lo(H: int, dl: float, du: float) -> int:
    # ceil(H * D_l / D_u) in exact integer arithmetic on the decimal ratios
    num, den = round(dl * 1000), round(du * 1000)
    return -(-H * num // den)


CONFIGS = {
    "C1": WorkloadConfig("C1", 1, 4, 3, 64, 0.6, 1.0, _d_lo(64, 0.01, 0.3), 0x2011011101),
    "C2": WorkloadConfig("C2", 100_000, 32, 4, 1024, 0.6, 1.0, _d_lo(1024, 0.01, 0.3), 0x2011011102),
    "C3": WorkloadConfig("C3", 1_000_000, 64, 8, 4096, 1.0, 2.0, _d_lo(4096, 0.01, 0.8), 0x2011011103),
    "C4": WorkloadConfig("C4", 10_000, 512, 8, 32768, 1.0, 2.0, _d_lo(32768, 0.01, 0.8), 0x2011011104),
    "C5": WorkloadConfig("C5", 1 << 24, 64, 8, 4096, 1.0, 8.0, _d_lo(4096, 0.01, 0.8), 0x2011011105,
                         u_blocks=((1.0, 1 << 22), (2.0, 1 << 22), (4.0, 1 << 22), (8.0, 1 << 22))),
}


@dataclass
class Batch:
    """A batch of instances in the C-ABI input layout (CSR over tasks)."""

    task_begin: np.ndarray  # int64 [B+1]
    release: np.ndarray     # int32 [T]
    deadline: np.ndarray    # int32 [T]
    mand_wcet: np.ndarray   # int32 [T]
    n_opt: np.ndarray       # uint8 [T]
    opt_wcet: np.ndarray    # int32 [T, stride]
    mand_conf: np.ndarray   # uint32 [T]
    opt_gain: np.ndarray    # int32 [T, stride]

    @property
    def n_instances(self) -> int:
        return len(self.task_begin) - 1

    @property
    def n_total_tasks(self) -> int:
        return int(self.task_begin[-1])

    @property
    def opt_stride(self) -> int:
        return self.opt_wcet.shape[1]

    def instance(self, b: int) -> "Batch":
        lo, hi = int(self.task_begin[b]), int(self.task_begin[b + 1])
        return Batch(np.array([0, hi - lo], np.int64), self.release[lo:hi].copy(),
                     self.deadline[lo:hi].copy(), self.mand_wcet[lo:hi].copy(),
                     self.n_opt[lo:hi].copy(), self.opt_wcet[lo:hi].copy(),
                     self.mand_conf[lo:hi].copy(), self.opt_gain[lo:hi].copy())

    def select(self, idx) -> "Batch":
        parts = [self.instance(int(b)) for b in idx]
        return concat(parts, self.opt_stride)

    def with_stride(self, stride: int) -> "Batch":
        s = self.opt_stride
        if stride == s:
            return self
        T = self.n_total_tasks
        ow = np.zeros((T, stride), np.int32)
        og = np.zeros((T, stride), np.int32)
        m = min(s, stride)
        ow[:, :m] = self.opt_wcet[:, :m]
        og[:, :m] = self.opt_gain[:, :m]
        return Batch(self.task_begin, self.release, self.deadline, self.mand_wcet, self.n_opt,
                     ow, self.mand_conf, og)


def concat(parts, stride: int) -> Batch:
    """Concatenate batches (each may hold any number of instances) into one."""
    parts = [p.with_stride(stride) for p in parts]
    tbs, base = [np.zeros(1, np.int64)], 0
    for p in parts:
        tbs.append(p.task_begin[1:] - p.task_begin[0] + base)
        base += p.n_total_tasks
    tb = np.concatenate(tbs).astype(np.int64)
    if not parts:
        e = np.zeros(0, np.int32)
        return Batch(tb, e, e, e, np.zeros(0, np.uint8), np.zeros((0, stride), np.int32),
                     np.zeros(0, np.uint32), np.zeros((0, stride), np.int32))
    cat = lambda f: np.concatenate([getattr(p, f)[int(p.task_begin[0]):int(p.task_begin[-1])] for p in parts])
    return Batch(tb, cat("release"), cat("deadline"), cat("mand_wcet"), cat("n_opt"),
                 cat("opt_wcet").reshape(int(tb[-1]), stride), cat("mand_conf"),
                 cat("opt_gain").reshape(int(tb[-1]), stride))


def build(force: bool = False) -> str:
    src = os.path.join(_HERE, "ic_gen_host.c")
    if force or not os.path.exists(_LIB_PATH) or os.path.getmtime(_LIB_PATH) < max(
            os.path.getmtime(src), os.path.getmtime(os.path.join(_HERE, "ic_gen_core.h"))):
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-shared", "-fPIC", "-o", _LIB_PATH, src])
    return _LIB_PATH


_lib = None


def _load():
    global _lib
    if _lib is None:
        build()
        _lib = ctypes.CDLL(_LIB_PATH)
        p = ctypes.c_void_p
        _lib.ic_gen_batch_host.argtypes = [ctypes.POINTER(GenConfig), ctypes.c_int64, ctypes.c_int64,
                                           p, p, p, p, p, p, p, p]
        _lib.ic_gen_batch_host.restype = ctypes.c_int
    return _lib


def _ptr(a: np.ndarray):
    return ctypes.c_void_p(a.ctypes.data) if a.size else None


def generate_gc(gc: GenConfig, n_instances: int, id_offset: int = 0) -> Batch:
    lib = _load()
    B, N, st = int(n_instances), gc.n_tasks, gc.opt_stride
    T = B * N
    out = Batch(np.zeros(B + 1, np.int64), np.zeros(T, np.int32), np.zeros(T, np.int32),
                np.zeros(T, np.int32), np.zeros(T, np.uint8), np.zeros((T, st), np.int32),
                np.zeros(T, np.uint32), np.zeros((T, st), np.int32))
    rc = lib.ic_gen_batch_host(ctypes.byref(gc), id_offset, B, _ptr(out.task_begin), _ptr(out.release),
                               _ptr(out.deadline), _ptr(out.mand_wcet), _ptr(out.n_opt),
                               _ptr(out.opt_wcet), _ptr(out.mand_conf), _ptr(out.opt_gain))
    if rc != 0:
        raise ValueError(f"ic_gen_batch_host failed ({rc})")
    return out


def generate(cfg: WorkloadConfig | str, n_instances: int | None = None, id_offset: int = 0,
             opt_stride: int | None = None) -> Batch:
    """Paper-shaped instances [id_offset, id_offset+n) of a configuration."""
    if isinstance(cfg, str):
        cfg = CONFIGS[cfg]
    n = cfg.n_instances if n_instances is None else n_instances
    if cfg.u_blocks:
        # C5: consecutive blocks of global ids with a fixed U each
        parts, start = [], 0
        for u, cnt in cfg.u_blocks:
            lo, hi = max(id_offset, start), min(id_offset + n, start + cnt)
            if lo < hi:
                parts.append(generate_gc(cfg.gen_config(opt_stride, u, u), hi - lo, lo))
            start += cnt
        return concat(parts, opt_stride or cfg.n_opt)
    return generate_gc(cfg.gen_config(opt_stride), n, id_offset)


def tiny_random(rng: np.random.Generator, n_instances: int, max_tasks: int = 5, max_opt: int = 3,
                max_wcet: int = 4, horizon: int = 24, p_release: float = 0.25,
                p_nonmono: float = 0.3, delta_micro: int = 100_000, aligned: bool = False) -> Batch:
    """Small random instances covering the method's degenerate cases.

    Confidences are multiples of 1e-2 (so Δ=0.1 produces frequent quantised
    ties) unless ``aligned`` makes every cumulative confidence a multiple of
    ``delta_micro``.  A fraction of instances carry releases, non-monotone
    confidence curves, equal deadlines or zero-size task sets.
    """
    parts = []
    for _ in range(n_instances):
        N = int(rng.integers(0, max_tasks + 1))
        rel = np.zeros(N, np.int32)
        if rng.random() < p_release:
            rel = rng.integers(0, horizon // 2 + 1, N).astype(np.int32)
        m = rng.integers(1, max_wcet + 1, N).astype(np.int32)
        S = rng.integers(0, max_opt + 1, N).astype(np.uint8)
        ow = np.zeros((N, max_opt), np.int32)
        og = np.zeros((N, max_opt), np.int32)
        a0 = np.zeros(N, np.uint32)
        nonmono = rng.random() < p_nonmono
        for i in range(N):
            ow[i, :S[i]] = rng.integers(1, max_wcet + 1, S[i])
            if aligned:
                levels = rng.integers(0, 1_000_000 // delta_micro + 1, S[i] + 1) * delta_micro
            else:
                levels = rng.integers(0, 101, S[i] + 1) * 10_000
            if not nonmono:
                levels = np.sort(levels)
            a0[i] = levels[0]
            og[i, :S[i]] = np.diff(levels)
        dl = rng.integers(0, horizon, N).astype(np.int32)
        if N >= 2 and rng.random() < 0.3:
            dl[:] = dl[0]  # equal deadlines: tie on the EDF key
        if N >= 1 and rng.random() < 0.1:
            dl[0] = -1 - int(rng.integers(0, 3))  # infeasible task
        parts.append(Batch(np.array([0, N], np.int64), rel, dl, m, S, ow, a0, og))
    return concat(parts, max_opt)

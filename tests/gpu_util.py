"""Shared helpers for the GPU parity tests (test plumbing only)."""
from __future__ import annotations

import numpy as np

import oracle

KEYS_EXACT = ("kept", "start", "finish", "q_total", "conf_micro", "makespan", "status")


def to_device(batch):
    import torch
    import paper_2011_01112_b200 as pkg
    return {f: torch.from_numpy(np.ascontiguousarray(getattr(batch, f))).cuda() for f, _, _ in pkg.INPUT_FIELDS}


def gpu_solve(batch, *, max_tasks, max_opt, max_horizon, drop_mode=0, delta=0, eps=100_000, host=False,
              tuning=None):
    import torch
    import paper_2011_01112_b200 as pkg
    assert batch.opt_stride == max_opt
    sc = pkg.SchedConfig(max_tasks=max_tasks, max_opt_stages=max_opt, max_horizon=max_horizon,
                         drop_mode=drop_mode, delta_micro=delta, epsilon_micro=eps)
    with pkg.Scheduler(sc, tuning) as s:
        if host:
            inp = {f: np.ascontiguousarray(getattr(batch, f)) for f, _, _ in pkg.INPUT_FIELDS}
            out = pkg.alloc_outputs(batch.n_instances, batch.n_total_tasks, host=True, pinned=True)
            s.solve_batch_host(inp, out)
        else:
            out = s.solve_batch(to_device(batch))
            torch.cuda.synchronize()
        info = s.info()
    got = {k: v.cpu().numpy() for k, v in out.items()}
    got["_info"] = info
    return got


def assert_parity(got, ref, where=""):
    for k in KEYS_EXACT:
        if not np.array_equal(got[k], ref[k]):
            idx = np.nonzero(got[k] != ref[k])[0]
            raise AssertionError(f"{where}: {k} differs at {len(idx)} positions, first {idx[:8]}: "
                                 f"gpu {got[k][idx[:8]]} oracle {ref[k][idx[:8]]}")
    # total confidence: 1e-6 relative (north_star); both sides divide the same exact integer
    np.testing.assert_allclose(got["conf_total"], ref["conf_total"], rtol=1e-6, atol=0)


def stats_from(result, batch):
    st = np.zeros(8, np.int64)
    ok = result["status"] == 0
    tb = batch.task_begin
    st[0] = batch.n_instances
    st[3] = int((~ok).sum())
    for b in np.nonzero(ok)[0]:
        lo, hi = tb[b], tb[b + 1]
        k = result["kept"][lo:hi]
        st[1] += hi - lo
        st[2] += int((k < 0).sum())
        st[4] += int(k[k >= 0].sum())
        st[5] += int(batch.n_opt[lo:hi].sum())
    st[6] = int(result["conf_micro"][ok].sum())
    st[7] = int(result["q_total"][ok].sum())
    return st


def oracle_cfg(**kw):
    return oracle.OracleConfig(**kw)

"""Parity at BASELINE.json's full sizes, in the launch configuration bench.py times.

Each test generates a whole configuration on the device (the bench's inputs), solves it
with ONE ic_sched_solve_batch exactly as bench.py does, and then
  * compares a deterministic sample element by element with the CPU oracle (O3, the
    time-indexed DP, pinned to O1/O2 in tests/test_oracle_pins.py) run on the same
    instances generated independently on the host (gen/libicgen.so), and
  * checks properties that hold at any size over EVERY instance of the launch: kept tasks
    meet their deadlines and run back to back in EDF order, finish = start +
    C_i(kept), makespan / confidence / stats recomputed from the plan.
Sample sizes follow BASELINE.md §3 "Parity coverage": C2 and C4 in full, C3 1-in-16,
C5 1-in-64 (runs of 64 consecutive ids, one per 4096-id window, so every U block and the
highest task-row offsets — beyond 2^31 words of opt_wcet — are covered).
"""
import numpy as np
import pytest

import gen
import oracle
from oracle import OracleConfig, TIME
from tests.gpu_util import assert_parity

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)


def _device_batch(cw):
    """The bench's inputs: every U block of the configuration generated on device."""
    import paper_2011_01112_b200 as pkg
    B, N = cw.n_instances, cw.n_tasks
    inputs = pkg.alloc_inputs(B, B * N, cw.n_opt, "cuda")
    blocks = cw.u_blocks or ((None, B),)
    a = 0
    for u, cnt in blocks:
        g = cw.gen_config(None, u, u) if u is not None else cw.gen_config()
        view = {k: (v[a:a + cnt + 1] if k == "task_begin" else v[a * N:(a + cnt) * N]) for k, v in inputs.items()}
        pkg.gen_batch_device(g.seed, g.n_tasks, g.n_opt, g.opt_stride, g.horizon, g.u_lo_q16, g.u_hi_q16,
                             g.d_lo, cnt, a, out=view)
        a += cnt
    inputs["task_begin"].copy_(torch.arange(B + 1, device="cuda", dtype=torch.int64) * N)
    return inputs


def _solve(cw, inputs):
    import paper_2011_01112_b200 as pkg
    sc = pkg.SchedConfig(max_tasks=cw.n_tasks, max_opt_stages=cw.n_opt, max_horizon=cw.horizon,
                         epsilon_micro=cw.epsilon_micro)
    with pkg.Scheduler(sc) as s:
        out = s.solve_batch(inputs)
        torch.cuda.synchronize()
    return out


def _sample_runs(B, every, run):
    """Deterministic 1-in-`every` sample as runs of `run` consecutive ids: one run per window
    of every*run ids at a hashed offset, plus the first and the last run of the batch."""
    win = every * run
    starts = [0]
    for j in range(B // win):
        starts.append(j * win + (j * 2654435761) % (win - run + 1))
    starts.append(B - run)
    return sorted(set(starts))


def _check_sample(cw, inputs, out, starts, run):
    N = cw.n_tasks
    parts = [gen.generate(cw, run, id_offset=int(s)) for s in starts]
    host = gen.concat(parts, cw.n_opt)
    ids = torch.tensor(np.concatenate([np.arange(s, s + run) for s in starts]), device="cuda")
    rows = (ids[:, None] * N + torch.arange(N, device="cuda")[None, :]).reshape(-1)
    # the oracle's instances are the ones the GPU solved (same generator, built twice)
    for f in ("release", "deadline", "mand_wcet", "n_opt", "mand_conf", "opt_wcet", "opt_gain"):
        x = inputs[f]
        x = x.view(torch.int32) if x.dtype == torch.uint32 else x  # no uint32 gather on CUDA
        h = getattr(host, f)
        np.testing.assert_array_equal(x[rows].cpu().numpy().view(h.dtype), h, err_msg=f)
    ocfg = OracleConfig(epsilon_micro=cw.epsilon_micro, max_tasks=N, max_horizon=cw.horizon)
    ref = oracle.solve(host, ocfg, TIME)
    got = {k: (out[k][rows] if k in ("kept", "start", "finish") else out[k][ids]).cpu().numpy()
           for k in ("kept", "start", "finish", "q_total", "conf_micro", "conf_total", "makespan", "status")}
    assert_parity(got, ref, f"{cw.name} sample of {len(ids)}")
    return len(ids)


def _full_properties(cw, inputs, out, chunk=1 << 18):
    """Plan validity over every instance of the launch (device torch ops; test code only)."""
    B, N, S = cw.n_instances, cw.n_tasks, cw.n_opt
    stats = torch.zeros(8, dtype=torch.int64, device="cuda")
    for lo in range(0, B, chunk):
        hi = min(B, lo + chunk)
        nb = hi - lo
        t = slice(lo * N, hi * N)
        kept = out["kept"][t].long().view(nb, N)
        st, fi = out["start"][t].long().view(nb, N), out["finish"][t].long().view(nb, N)
        d = inputs["deadline"][t].long().view(nb, N)
        r = inputs["release"][t].long().view(nb, N)
        C = torch.cumsum(torch.cat([inputs["mand_wcet"][t].long()[:, None], inputs["opt_wcet"][t].long()], 1), 1)
        R = torch.cumsum(torch.cat([inputs["mand_conf"][t].long()[:, None], inputs["opt_gain"][t].long()], 1), 1)
        k = kept.clamp(min=0).view(-1, 1)
        Ck = torch.gather(C, 1, k).view(nb, N)
        Rk = torch.gather(R, 1, k).view(nb, N)
        on = kept >= 0
        assert (out["status"][lo:hi] == 0).all()
        assert ((kept >= -1) & (kept <= inputs["n_opt"][t].long().view(nb, N))).all()
        assert torch.where(on, (fi == st + Ck) & (fi <= d) & (st >= r), (st == -1) & (fi == -1)).all()
        # back to back in EDF order (deadline, release, index): no overlap between kept tasks
        key = (d * (1 << 20) + r) * 4096 + torch.arange(N, device="cuda")[None, :]
        order = torch.argsort(key, 1)
        so, fo, oo = torch.gather(st, 1, order), torch.gather(fi, 1, order), torch.gather(on, 1, order)
        prevf = torch.cummax(torch.where(oo, fo, torch.zeros_like(fo)), 1).values
        prevf = torch.cat([torch.zeros_like(prevf[:, :1]), prevf[:, :-1]], 1)
        assert torch.where(oo, so >= prevf, torch.ones_like(oo)).all()
        assert (out["makespan"][lo:hi].long() == torch.where(on, fi, torch.zeros_like(fi)).max(1).values).all()
        conf = torch.where(on, Rk, torch.zeros_like(Rk)).sum(1)
        assert (out["conf_micro"][lo:hi] == conf).all()
        stats[1] += nb * N
        stats[2] += int((~on).sum())
        stats[4] += int(torch.where(on, kept, torch.zeros_like(kept)).sum())
        stats[5] += int(inputs["n_opt"][t].long().sum())
    stats[0] = B
    stats[6] = out["conf_micro"].sum()
    stats[7] = out["q_total"].sum()
    assert torch.equal(out["stats"], stats), (out["stats"].tolist(), stats.tolist())


def test_c5_full_launch_one_in_64():
    """The headline launch: 2^24 C5 instances (U = 1, 2, 4, 8) in one solve, 262k sampled."""
    cw = gen.CONFIGS["C5"]
    inputs = _device_batch(cw)
    out = _solve(cw, inputs)
    _full_properties(cw, inputs, out)
    starts = _sample_runs(cw.n_instances, 64, 64)
    assert _check_sample(cw, inputs, out, starts, 64) >= cw.n_instances // 64
    assert starts[-1] + 64 == cw.n_instances  # the last instances: task rows past 2^30


@pytest.mark.parametrize("name,every,run", [("C2", 1, 100_000), ("C3", 16, 64), ("C4", 1, 10_000)])
def test_full_config_sampled(name, every, run):
    cw = gen.CONFIGS[name]
    inputs = _device_batch(cw)
    out = _solve(cw, inputs)
    _full_properties(cw, inputs, out, chunk=1 << 14 if cw.n_tasks > 64 else 1 << 18)
    starts = [0] if every == 1 else _sample_runs(cw.n_instances, every, run)
    assert _check_sample(cw, inputs, out, starts, run) >= cw.n_instances // every

"""Run small solves of every kernel family under compute-sanitizer (tests/test_sanitizer.py).

    compute-sanitizer --tool racecheck python tests/sanitize_driver.py

Each variant passes the launch tuning ic_sched_create_tuned fixes for the handle
(DP warps, in-place rows, global option tables, sweep axis, kernel), solves a few
instances and checks them against the oracle, so a hazard report is tied to a
correct run.  Exit code 1 on a parity mismatch.
"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import gen  # noqa: E402
import oracle  # noqa: E402
from tests.gpu_util import assert_parity, gpu_solve  # noqa: E402

VARIANTS = {
    # name: (tuning, config, instances, delta)
    "nw1": (dict(kernel=1), "C2", 6, 0),
    "nw4": ({}, "C3", 2, 0),
    "sb8_inplace": (dict(in_place=1, dp_warps=8), "C3", 2, 0),
    "nw16_global_tables": (dict(in_place=1, dp_warps=16, option_tables=1), "C3", 2, 0),
    "nw15_global_tables": (dict(in_place=1, dp_warps=15, option_tables=1), "C3", 2, 0),
    "solo_unpacked": (dict(packed_options=2), "C2", 6, 100_000),
    "reward_axis": (dict(axis=2, kernel=1), "C2", 6, 100_000),
    "solo": ({}, "C2", 6, 0),
    "solo_reward": ({}, "C2", 6, 100_000),
    "hybrid": ({}, "C3", 3, 100_000),
}
EXTRA = ("replan", "reassign")


def _first_tasks(batch, m):
    from gen import Batch
    parts = []
    for b in range(batch.n_instances):
        one = batch.instance(b)
        parts.append(Batch(np.array([0, m], np.int64), one.release[:m], one.deadline[:m], one.mand_wcet[:m],
                           one.n_opt[:m], one.opt_wcet[:m], one.mand_conf[:m], one.opt_gain[:m]))
    return gen.concat(parts, batch.opt_stride)


def replan():
    """NEXT-2 state path: solve 31 tasks keeping the state, re-plan with one arrival."""
    import torch
    import paper_2011_01112_b200 as pkg
    from tests.gpu_util import to_device
    cw = gen.WorkloadConfig("C2x", 0, 32, 4, 1024, 0.6, 1.0, 35, 0x2011011102)
    full = gen.generate(cw, 6)
    sc = pkg.SchedConfig(max_tasks=32, max_opt_stages=4, max_horizon=1024, delta_micro=100_000)
    with pkg.Scheduler(sc) as s:
        state = torch.zeros(s.state_bytes(full.n_instances), dtype=torch.uint8, device="cuda")
        s.solve_batch_state(to_device(_first_tasks(full, 31)), state)
        out = s.replan_batch(to_device(full), state)
        torch.cuda.synchronize()
        got = {k: v.cpu().numpy() for k, v in out.items()}
    ref = oracle.solve(full, oracle.OracleConfig(delta_micro=100_000, max_tasks=32, max_horizon=1024), oracle.TIME)
    assert_parity(got, ref, "sanitize replan")


def reassign():
    """NEXT-3 stage-completion kernel on a solved C2-shaped batch."""
    import torch
    import paper_2011_01112_b200 as pkg
    from tests.gpu_util import to_device
    cw = gen.CONFIGS["C2"]
    batch = gen.generate(cw, 16)
    ocfg = oracle.OracleConfig(delta_micro=100_000, max_tasks=32, max_horizon=1024)
    plan = oracle.solve(batch, ocfg, oracle.TIME)
    done = np.zeros(batch.n_instances, np.int8)
    obs = np.full(batch.n_instances, 300_000, np.uint32)
    ref = oracle.reassign(batch, plan["kept"], done, obs, 2, ocfg)
    sc = pkg.SchedConfig(max_tasks=32, max_opt_stages=4, max_horizon=1024, delta_micro=100_000)
    with pkg.Scheduler(sc) as s:
        out = s.reassign_batch(to_device(batch), torch.from_numpy(plan["kept"]).cuda(),
                               torch.from_numpy(done).cuda(), torch.from_numpy(obs).cuda(), 2)
        torch.cuda.synchronize()
    for k in ("kept", "start", "finish", "conf_micro", "makespan", "status", "swapped"):
        np.testing.assert_array_equal(out[k].cpu().numpy(), ref[k], err_msg=k)


def main(names):
    rng = np.random.default_rng(7)
    for name in names:
        if name in EXTRA:
            {"replan": replan, "reassign": reassign}[name]()
            print("ok", name, flush=True)
            continue
        tuning, cfg, n, delta = VARIANTS[name]
        cw = gen.CONFIGS[cfg]
        tiny = gen.tiny_random(rng, 24, max_tasks=6, max_opt=cw.n_opt, horizon=min(cw.horizon, 256))
        batch = gen.concat([gen.generate(cw, n), tiny], cw.n_opt)
        for mode in (0, 1):
            ocfg = oracle.OracleConfig(drop_mode=mode, delta_micro=delta, epsilon_micro=100_000,
                                       max_tasks=cw.n_tasks, max_horizon=cw.horizon)
            ref = oracle.solve(batch, ocfg, oracle.TIME)
            got = gpu_solve(batch, max_tasks=cw.n_tasks, max_opt=cw.n_opt, max_horizon=cw.horizon,
                            drop_mode=mode, delta=delta, tuning=tuning)
            assert_parity(got, ref, f"sanitize {name} mode={mode}")
        print("ok", name, flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or list(VARIANTS) + list(EXTRA))

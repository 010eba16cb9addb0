"""Run small solves of every kernel family under compute-sanitizer (tests/test_sanitizer.py).

    compute-sanitizer --tool racecheck python tests/sanitize_driver.py

Each variant sets the launch-geometry knobs the library reads at ic_sched_create
(DP warps, in-place rows, global option tables, sweep axis), solves a few
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
    # name: (env, config, instances, delta)
    "nw1": ({}, "C2", 6, 0),
    "nw4": ({}, "C3", 2, 0),
    "sb8_inplace": ({"IC_SCHED_SB": "1", "IC_SCHED_NW": "8"}, "C3", 2, 0),
    "nw16_global_tables": ({"IC_SCHED_SB": "1", "IC_SCHED_NW": "16", "IC_SCHED_ROWP": "global"}, "C3", 2, 0),
    "reward_axis": ({"IC_SCHED_AXIS": "2"}, "C2", 6, 100_000),
}
KNOBS = ("IC_SCHED_SB", "IC_SCHED_NW", "IC_SCHED_ROWP", "IC_SCHED_AXIS")


def main(names):
    rng = np.random.default_rng(7)
    for name in names:
        env, cfg, n, delta = VARIANTS[name]
        for k in KNOBS:
            os.environ.pop(k, None)
        os.environ.update(env)
        cw = gen.CONFIGS[cfg]
        tiny = gen.tiny_random(rng, 24, max_tasks=6, max_opt=cw.n_opt, horizon=min(cw.horizon, 256))
        batch = gen.concat([gen.generate(cw, n), tiny], cw.n_opt)
        for mode in (0, 1):
            ocfg = oracle.OracleConfig(drop_mode=mode, delta_micro=delta, epsilon_micro=100_000,
                                       max_tasks=cw.n_tasks, max_horizon=cw.horizon)
            ref = oracle.solve(batch, ocfg, oracle.TIME)
            got = gpu_solve(batch, max_tasks=cw.n_tasks, max_opt=cw.n_opt, max_horizon=cw.horizon,
                            drop_mode=mode, delta=delta)
            assert_parity(got, ref, f"sanitize {name} mode={mode}")
        print("ok", name, flush=True)


if __name__ == "__main__":
    main(sys.argv[1:] or list(VARIANTS))

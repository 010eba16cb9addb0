"""NEXT-4: the edge-server simulator (include/ic_sim.h).

CPU: the utility-insensitive baselines (EDF / LCF / RR) need no GPU.
GPU: the RTDeepIoT planner re-plans every scheduling point with the batched DP.
"""
import pytest

import paper_2011_01112_b200 as pkg

L = 8  # 1 mandatory + 7 optional stages


def _run(**kw):
    return pkg.simulate(pkg.SimConfig(**kw))


@pytest.mark.parametrize("policy", ["edf", "lcf", "rr"])
def test_baseline_conservation_and_determinism(policy):
    kw = dict(servers=3, clients=12, requests_per_client=30, policy=policy)
    a, b = _run(**kw), _run(**kw)
    for k in ("requests", "misses", "stages_run", "conf_micro"):
        assert a[k] == b[k], k
    assert a["requests"] == 3 * 12 * 30
    assert 0 <= a["misses"] <= a["requests"]
    assert a["stages_run"] <= a["requests"] * L
    assert a["plans"] == 0 and a["gpu_seconds"] == 0.0
    assert 0.0 <= a["accuracy"] <= 1.0


@pytest.mark.parametrize("policy", ["edf", "lcf", "rr"])
def test_baselines_run_full_depth_without_contention(policy):
    # one client, deadlines longer than a full-depth request (8 stages of <= 11 ticks):
    # nothing competes, so every request runs all stages and none misses
    r = _run(servers=2, clients=1, requests_per_client=40, d_lo=200, d_hi=300, policy=policy)
    assert r["misses"] == 0
    assert r["stages_run"] == r["requests"] * L


def test_single_client_policies_agree():
    # one outstanding request at a time: EDF, LCF and RR pick the same stage every time
    res = [_run(clients=1, requests_per_client=60, d_lo=20, d_hi=90, policy=p) for p in ("edf", "lcf", "rr")]
    assert res[0]["conf_micro"] == res[1]["conf_micro"] == res[2]["conf_micro"]
    assert res[0]["stages_run"] == res[1]["stages_run"] == res[2]["stages_run"]


def test_overload_ordering_of_baselines():
    # under overload EDF misses most; LCF and RR miss less
    kw = dict(servers=4, clients=20, requests_per_client=40)
    e, lc, rr = (_run(policy=p, **kw) for p in ("edf", "lcf", "rr"))
    assert e["miss_rate"] > lc["miss_rate"] and e["miss_rate"] > rr["miss_rate"]
    assert e["accuracy"] < lc["accuracy"] and e["accuracy"] < rr["accuracy"]


@pytest.mark.parametrize("policy", ["edf", "lcf", "rr"])
def test_open_loop_conservation(policy):
    kw = dict(servers=4, clients=10, requests_per_client=25, period=400, policy=policy)
    a, b = _run(**kw), _run(**kw)
    assert a == {**b, "sim_seconds": a["sim_seconds"]}
    assert a["requests"] == 4 * 10 * 25


def test_open_loop_light_load_no_misses():
    # one client, gaps >= 400 ticks > the longest deadline: requests never overlap
    for p in ("edf", "lcf", "rr"):
        r = _run(clients=1, requests_per_client=50, d_lo=200, d_hi=300, period=800, policy=p)
        assert r["misses"] == 0 and r["stages_run"] == 50 * L


def test_invalid_configs_rejected():
    for kw in (dict(servers=0), dict(n_opt=15), dict(d_hi=5, d_lo=10), dict(think=0), dict(policy=9),
               dict(period=-1),
               dict(policy="planner", delta_micro=0)):
        with pytest.raises(pkg.ICSchedError) as e:
            _run(**kw)
        assert e.value.rc == -1


@pytest.mark.gpu
def test_planner_deterministic_and_conserving():
    kw = dict(servers=16, clients=16, requests_per_client=20, policy="planner")
    a, b = _run(**kw), _run(**kw)
    for k in ("requests", "misses", "stages_run", "conf_micro", "plans", "rounds"):
        assert a[k] == b[k], k
    assert a["requests"] == 16 * 16 * 20
    assert a["plans"] > 0 and a["rounds"] > 0 and a["plans"] >= a["rounds"]


@pytest.mark.gpu
@pytest.mark.parametrize("clients", [20, 28])
def test_planner_beats_baselines_under_load(clients):
    # RTDeepIoT's accuracy exceeds EDF, LCF and RR under overload (open loop,
    # Delta = 0.1; DESIGN.md §5b NEXT-4 has the whole load sweep)
    kw = dict(servers=64, clients=clients, requests_per_client=20, period=600)
    p = _run(policy="planner", **kw)
    for pol in ("edf", "lcf", "rr"):
        assert p["accuracy"] > _run(policy=pol, **kw)["accuracy"], pol


@pytest.mark.gpu
def test_planner_oracle_utility_at_least_exp():
    # RTDeepIoT-OPT (true confidences) vs the Exp heuristic
    kw = dict(servers=32, clients=16, requests_per_client=30, policy="planner", period=600)
    exp = _run(utility=pkg.IC_SIM_UTIL_EXP, **kw)
    opt = _run(utility=pkg.IC_SIM_UTIL_ORACLE, **kw)
    assert opt["accuracy"] >= exp["accuracy"] - 0.01


def test_invalid_cost_model_rejected():
    with pytest.raises(pkg.ICSchedError) as e:
        _run(policy="planner", plan_cells_per_tick=-1)
    assert e.value.rc == -1


@pytest.mark.gpu
@pytest.mark.parametrize("utility,delta", [(0, 100_000), (1, 20_000), (0, 500_000)])
def test_simulator_plans_equal_oracle(utility, delta):
    """Parity hook: the DP instances the simulator's planner batched (sunk stages, carried
    remainders, Exp predictions) and the plans the GPU returned for them equal the CPU
    oracle's, element by element — the simulator's decisions are the paper's DP."""
    import numpy as np
    import oracle
    from gen import Batch
    from tests.gpu_util import assert_parity
    cfg = pkg.SimConfig(servers=24, clients=14, requests_per_client=12, period=500, policy="planner",
                        utility=utility, delta_micro=delta)
    res, d = pkg.simulate(cfg, dump_instances=3000, dump_tasks=60000)
    assert d["task_begin"].size - 1 >= 200
    batch = Batch(d["task_begin"], d["release"], d["deadline"], d["mand_wcet"], d["n_opt"], d["opt_wcet"],
                  d["mand_conf"], d["opt_gain"])
    ocfg = oracle.OracleConfig(delta_micro=delta, max_tasks=4096, max_horizon=cfg.d_hi + 1)
    ref = oracle.solve(batch, ocfg, oracle.TIME)
    got = dict(d, conf_total=d["conf_micro"] / 1e6)
    assert_parity(got, ref, f"simulator batches utility={utility} delta={delta}")
    assert (oracle.check(batch, got, ocfg) == 0).all()


@pytest.mark.gpu
def test_plan_cost_model():
    """with the scheduler's cost charged to the server, a finer reward step makes
    the paper's table larger and the planning time longer; free planning charges nothing."""
    kw = dict(servers=16, clients=16, requests_per_client=15, period=600, policy="planner")
    free = _run(**kw)
    assert free["plan_ticks"] == 0
    ticks = [_run(delta_micro=d, plan_cells_per_tick=200, **kw)["plan_ticks"] for d in (500_000, 100_000, 20_000)]
    assert 0 < ticks[0] < ticks[1] < ticks[2]

"""Pins of the CPU oracle against what the paper, its SPEC and mathematics fix.

Each test pins the oracle to something other than itself (task brief ③):
SPEC worked examples (tests/golden/spec_examples.json, each cited), closed
forms, Theorem 1, and brute-force enumeration of the plain definition
(oracle/definition.py, written independently of ic_oracle.c).
"""
import json
import os

import numpy as np
import pytest

import oracle
from oracle import definition
from oracle import OracleConfig, BRUTE, PAPER, TIME
from gen import tiny_random, concat
from tests._instances import batch_from_tasks, batch_from_many

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))
INF = np.iinfo(np.int64).max
ALGOS = (BRUTE, PAPER, TIME)


def _cfg(ex, **kw):
    return OracleConfig(drop_mode=ex.get("drop_mode", 0), delta_micro=ex.get("delta_micro", 0),
                        epsilon_micro=ex.get("epsilon_micro", 100_000), **kw)


# ---------------------------------------------------------------- SPEC worked examples
def test_quantize_examples():
    """S:L180-182 via single-task instances: q = floor(R / Delta) in micro-units."""
    for R, delta, q in GOLD["quantize"]["cases"]:
        b = batch_from_tasks([dict(r=0, d=5, m=1, w=[], g=[], a0=R)])
        for algo in ALGOS:
            out = oracle.solve(b, OracleConfig(delta_micro=delta, drop_mode=1), algo)
            assert out["q_total"][0] == q
    # the floating-point trap the micro-unit reading avoids (R11)
    assert int(np.floor(0.7 / 0.1)) == 6


@pytest.mark.parametrize("name", ["single_task", "two_task"])
def test_spec_table_cells(name):
    """cells of P(i, r) of Eq. 2."""
    ex = GOLD[name]
    b = batch_from_tasks(ex["tasks"])
    P = oracle.paper_table(b, _cfg(ex))
    for i, r, v in ex["P_cells"]:
        assert P[i, r] == v, (i, r, P[i])
    for i, r in ex.get("P_infinite", []):
        assert r >= P.shape[1] or P[i, r] == INF


@pytest.mark.parametrize("name", ["single_task", "two_task", "brute_single", "brute_mandatory_only",
                                  "tie_two_identical", "tie_zero_quantum_drop", "release_gap",
                                  "identical_enforced"])
@pytest.mark.parametrize("algo", ALGOS)
def test_golden_plans(name, algo):
    ex = GOLD[name]
    b = batch_from_tasks(ex["tasks"])
    out = oracle.solve(b, _cfg(ex), algo)
    assert out["status"][0] == oracle.OK
    assert list(out["kept"]) == ex["kept"]
    for key, field in (("Q", "q_total"), ("makespan", "makespan"), ("conf_micro", "conf_micro")):
        if key in ex:
            assert out[field][0] == ex[key], key
    for key in ("start", "finish"):
        if key in ex:
            assert list(out[key]) == ex[key]
    if "enforced" in ex:
        e = ex["enforced"]
        out = oracle.solve(b, _cfg(dict(ex, drop_mode=1)), algo)
        assert list(out["kept"]) == e["kept"]
        assert out["q_total"][0] == e["Q"] and out["makespan"][0] == e["makespan"]
    # the pure-Python definition agrees
    d = definition.solve(ex["tasks"], ex.get("delta_micro") or 1, enforced=ex.get("drop_mode", 0) == 1)
    assert d["kept"] == ex["kept"]


def test_choose_delta():
    """Delta = eps * R / N (Theorem 1), R = best feasible reward."""
    for c in GOLD["choose_delta"]["cases"]:
        tasks = [dict(r=0, d=10, m=1, w=[], g=[], a0=c["R"])] * c["n"]
        b = batch_from_tasks(tasks)
        out = oracle.solve(b, OracleConfig(epsilon_micro=c["epsilon_micro"]), PAPER)
        assert out["delta_used"][0] == c["delta_micro"]
        assert definition.fptas_delta(tasks, c["epsilon_micro"]) == c["delta_micro"]


def test_fptas_R_excludes_infeasible_depths():
    """Reading R8: R counts only individually feasible (task, depth) pairs."""
    tasks = [dict(r=0, d=1, m=1, w=[5], a0=100000, g=[900000])]  # depth 2 never fits
    out = oracle.solve(batch_from_tasks(tasks), OracleConfig(epsilon_micro=100000), PAPER)
    assert out["delta_used"][0] == 100000 * 100000 // 1_000_000


def test_theorem1_enforced_counterexample():
    """Reading R8: the (1-eps) bound needs DROP mode."""
    ex = GOLD["theorem1_enforced_counterexample"]
    b = batch_from_tasks(ex["tasks"])
    for algo in ALGOS:
        out = oracle.solve(b, _cfg(ex), algo)
        assert out["conf_micro"][0] == ex["conf_micro"]
    opt = oracle.solve(b, OracleConfig(drop_mode=1, delta_micro=1), BRUTE)
    assert opt["conf_micro"][0] == ex["opt_conf_micro"]
    assert ex["conf_micro"] < (1 - 0.5) * ex["opt_conf_micro"]


# ---------------------------------------------------------------- brute force of the definition
def _definition_results(batch, delta, enforced):
    res = []
    for b in range(batch.n_instances):
        res.append(definition.solve(definition.tasks_from_batch(batch, b), delta, enforced))
    return res


@pytest.mark.parametrize("enforced", [0, 1])
def test_c_brute_force_matches_python_definition(enforced):
    rng = np.random.default_rng(11 + enforced)
    batch = tiny_random(rng, 1500, max_tasks=4, max_opt=2, horizon=14)
    cfg = OracleConfig(drop_mode=enforced, delta_micro=100_000)
    out = oracle.solve(batch, cfg, BRUTE)
    ref = _definition_results(batch, 100_000, enforced)
    for b, d in enumerate(ref):
        lo, hi = batch.task_begin[b], batch.task_begin[b + 1]
        if d is None:
            assert out["status"][b] == oracle.INFEASIBLE
            continue
        assert out["status"][b] == oracle.OK
        assert list(out["kept"][lo:hi]) == d["kept"]
        assert list(out["start"][lo:hi]) == d["start"]
        assert list(out["finish"][lo:hi]) == d["finish"]
        assert out["q_total"][b] == d["Q"] and out["makespan"][b] == d["makespan"]
        assert out["conf_micro"][b] == d["conf"]


def _assert_same(a, b, keys=("kept", "start", "finish", "q_total", "conf_micro", "makespan", "status")):
    for k in keys:
        np.testing.assert_array_equal(a[k], b[k], err_msg=k)


@pytest.mark.parametrize("mode", [0, 1])
@pytest.mark.parametrize("delta", [100_000, 30_000, 0])
def test_three_algorithms_agree(mode, delta):
    """P12: O1 == O2 == O3 bit-exactly (releases, non-monotone rewards, ties, both modes)."""
    rng = np.random.default_rng(1000 + mode * 7 + delta)
    batch = tiny_random(rng, 20000, max_tasks=5, max_opt=3, horizon=20)
    cfg = OracleConfig(drop_mode=mode, delta_micro=delta, epsilon_micro=250_000)
    o1 = oracle.solve(batch, cfg, BRUTE)
    o2 = oracle.solve(batch, cfg, PAPER)
    o3 = oracle.solve(batch, cfg, TIME)
    _assert_same(o1, o2)
    _assert_same(o1, o3)
    assert (oracle.check(batch, o2, cfg) == 0).all()


# ---------------------------------------------------------------- Theorem 1 and exactness
@pytest.mark.parametrize("eps", [100_000, 250_000, 500_000])
def test_theorem1_bound_drop_mode(eps):
    """P6 / S:L492: plan reward >= (1-eps) OPT over >= 1000 instances, zero tolerance."""
    rng = np.random.default_rng(eps)
    batch = tiny_random(rng, 3000, max_tasks=6, max_opt=3, horizon=24, p_nonmono=0.0)
    plan = oracle.solve(batch, OracleConfig(epsilon_micro=eps), PAPER)
    opt = oracle.solve(batch, OracleConfig(delta_micro=1), BRUTE)  # exact OPT of sum R
    lhs = plan["conf_micro"] * 1_000_000
    rhs = (1_000_000 - eps) * opt["conf_micro"]
    assert (lhs >= rhs).all()


def test_exact_when_rewards_aligned():
    """P7 / S:L493: rewards multiples of Delta -> Q * Delta = OPT."""
    rng = np.random.default_rng(7)
    batch = tiny_random(rng, 3000, max_tasks=6, max_opt=3, horizon=24, aligned=True,
                        delta_micro=50_000)
    plan = oracle.solve(batch, OracleConfig(delta_micro=50_000), PAPER)
    opt = oracle.solve(batch, OracleConfig(delta_micro=1), BRUTE)
    np.testing.assert_array_equal(plan["q_total"] * 50_000, opt["conf_micro"])
    np.testing.assert_array_equal(plan["conf_micro"], opt["conf_micro"])


# ---------------------------------------------------------------- closed forms (P10)
def test_closed_form_loose_deadlines():
    """P10(i): all deadlines >= total full demand -> each task independently takes the smallest
    k maximising q; in drop mode a task whose best q is 0 is dropped."""
    rng = np.random.default_rng(3)
    lists = []
    for _ in range(400):
        N = int(rng.integers(1, 6))
        ts = []
        for _ in range(N):
            S = int(rng.integers(0, 4))
            lv = rng.integers(0, 101, S + 1) * 10_000
            ts.append(dict(r=0, d=0, m=int(rng.integers(1, 4)), w=[int(x) for x in rng.integers(1, 4, S)],
                           a0=int(lv[0]), g=[int(x) for x in np.diff(lv)]))
        tot = sum(t["m"] + sum(t["w"]) for t in ts)
        for t in ts:
            t["d"] = tot + int(rng.integers(0, 3))
        lists.append(ts)
    batch = batch_from_many(lists, 3)
    out = oracle.solve(batch, OracleConfig(delta_micro=100_000), PAPER)
    for b, ts in enumerate(lists):
        lo = batch.task_begin[b]
        for i, t in enumerate(ts):
            C, R = definition.derive(t)
            q = [r // 100_000 for r in R]
            kbest = int(np.argmax(q))
            expect = -1 if q[kbest] == 0 else kbest
            assert out["kept"][lo + i] == expect


def test_closed_form_single_task():
    """P10(ii): N = 1 -> smallest k with the largest q among C(k) <= d; DROP if that q is 0."""
    rng = np.random.default_rng(4)
    for _ in range(300):
        S = int(rng.integers(0, 5))
        lv = rng.integers(0, 101, S + 1) * 10_000
        t = dict(r=0, d=int(rng.integers(0, 12)), m=int(rng.integers(1, 4)),
                 w=[int(x) for x in rng.integers(1, 4, S)], a0=int(lv[0]), g=[int(x) for x in np.diff(lv)])
        out = oracle.solve(batch_from_tasks([t]), OracleConfig(delta_micro=100_000), PAPER)
        C, R = definition.derive(t)
        cands = [(R[k] // 100_000, -k) for k in range(len(C)) if C[k] <= t["d"]]
        if not cands or max(cands)[0] == 0:
            assert out["kept"][0] == -1
        else:
            assert out["kept"][0] == -max(cands)[1]


def test_closed_form_identical_tasks_enforced():
    """P10(iii): identical tasks (m, S stages of cost c each worth one quantum), common d,
    enforced: total kept = min(N S, (d - N m) // c), filled from the first EDF task."""
    for N in range(1, 6):
        for S in range(0, 4):
            for c in (1, 2):
                for m in (1, 3):
                    for slack in range(0, N * S * c + 3):
                        d = N * m + slack
                        t = dict(r=0, d=d, m=m, w=[c] * S, a0=500_000, g=[100_000] * S)
                        out = oracle.solve(batch_from_tasks([t] * N),
                                           OracleConfig(drop_mode=1, delta_micro=100_000), PAPER)
                        total = min(N * S, slack // c)
                        expect = []
                        for _ in range(N):
                            k = min(S, total)
                            expect.append(k)
                            total -= k
                        assert list(out["kept"]) == expect, (N, S, c, m, slack)


def _knapsack(values, weights, cap):
    best = [0] * (cap + 1)
    for v, w in zip(values, weights):
        for x in range(cap, w - 1, -1):
            best[x] = max(best[x], best[x - w] + v)
    return best[cap]


def test_closed_form_knapsack_reduction():
    """P10(iv): enforced, S = 1, common deadline: Q* - sum q(0) is the 0/1 knapsack optimum with
    values q(1) - q(0), weights c_1 and capacity d - sum m (textbook DP)."""
    rng = np.random.default_rng(5)
    for _ in range(500):
        N = int(rng.integers(1, 7))
        ts = []
        for _ in range(N):
            a0 = int(rng.integers(0, 60)) * 10_000
            ts.append(dict(r=0, d=0, m=int(rng.integers(1, 3)), w=[int(rng.integers(1, 5))], a0=a0,
                           g=[int(rng.integers(0, 101 - a0 // 10_000)) * 10_000]))
        cap = int(rng.integers(0, 12))
        d = sum(t["m"] for t in ts) + cap
        for t in ts:
            t["d"] = d
        out = oracle.solve(batch_from_tasks(ts), OracleConfig(drop_mode=1, delta_micro=100_000), PAPER)
        q0 = [t["a0"] // 100_000 for t in ts]
        q1 = [(t["a0"] + t["g"][0]) // 100_000 for t in ts]
        ks = _knapsack([b - a for a, b in zip(q0, q1)], [t["w"][0] for t in ts], cap)
        assert out["q_total"][0] - sum(q0) == ks


def test_closed_form_all_infeasible():
    """P10(v): every d_i < r_i + m_i -> all dropped (drop mode) / INFEASIBLE (enforced)."""
    ts = [dict(r=2, d=3, m=2, w=[1], a0=900_000, g=[50_000]), dict(r=0, d=0, m=1, w=[], a0=1, g=[])]
    for algo in ALGOS:
        out = oracle.solve(batch_from_tasks(ts), OracleConfig(delta_micro=100_000), algo)
        assert list(out["kept"]) == [-1, -1] and out["status"][0] == oracle.OK
        out = oracle.solve(batch_from_tasks(ts), OracleConfig(drop_mode=1, delta_micro=100_000), algo)
        assert list(out["kept"]) == [-1, -1] and out["status"][0] == oracle.INFEASIBLE
        assert out["q_total"][0] == 0


def test_empty_instance():
    b = concat([batch_from_tasks([])], 0)
    for algo in ALGOS:
        out = oracle.solve(b, OracleConfig(delta_micro=100_000), algo)
        assert out["status"][0] == oracle.OK and out["q_total"][0] == 0 and out["makespan"][0] == 0


# ---------------------------------------------------------------- table invariants (P9)
def test_time_table_monotone_and_skip_dominance():
    """P9 / S:L228: G_i(t) >= G_{i-1}(t) in drop mode; G_i non-decreasing in t."""
    rng = np.random.default_rng(9)
    batch = tiny_random(rng, 300, max_tasks=6, max_opt=3, horizon=30)
    for b in range(batch.n_instances):
        G = oracle.time_table(batch, OracleConfig(delta_micro=100_000), b)
        assert (np.diff(G, axis=1) >= 0).all()
        assert (np.diff(G, axis=0) >= 0).all()
        P = oracle.paper_table(batch, OracleConfig(delta_micro=100_000), b)
        # skip-dominance in the reward-indexed table: P(i, r) <= P(i-1, r)
        assert (P[1:] <= P[:-1]).all()
        # duality: G_N(t) = max{r : P(N, r) <= t}
        n = P.shape[0] - 1
        for t in range(G.shape[1]):
            fin = np.nonzero(P[n] <= t)[0]
            assert G[n, t] == fin.max()


# ---------------------------------------------------------------- validation / checker
def test_bad_input_status():
    base = dict(r=0, d=5, m=1, w=[1], a0=300_000, g=[100_000])
    bad = [dict(base, m=0), dict(base, w=[0]), dict(base, r=-1), dict(base, d=64),
           dict(base, a0=1_000_001), dict(base, g=[800_000]), dict(base, g=[-400_000])]
    for t in bad:
        out = oracle.solve(batch_from_tasks([t]), OracleConfig(delta_micro=100_000, max_horizon=64), PAPER)
        assert out["status"][0] == oracle.BAD_INPUT and out["kept"][0] == -1
    # a dip in confidence that stays within [0, 1e6] is legal (reading R17)
    ok = dict(base, a0=500_000, g=[-200_000])
    out = oracle.solve(batch_from_tasks([ok]), OracleConfig(delta_micro=100_000, max_horizon=64), PAPER)
    assert out["status"][0] == oracle.OK


def test_checker_detects_violations():
    ex = GOLD["two_task"]
    b = batch_from_tasks(ex["tasks"])
    cfg = OracleConfig(delta_micro=100_000)
    good = oracle.solve(b, cfg, PAPER)
    assert oracle.check(b, good, cfg)[0] == 0
    bad = {k: v.copy() for k, v in good.items()}
    bad["finish"][1] += 1
    assert oracle.check(b, bad, cfg)[0] & 2
    bad = {k: v.copy() for k, v in good.items()}
    bad["kept"][0] = -1
    assert oracle.check(b, bad, cfg)[0] != 0


# ---------------------------------------------------------------- checker negative pins
# Each bit of or_check (P:L48 schedule, P:L70 imprecise-computation feasibility, S:L494 EDF
# demand criterion) is provoked by a hand-built result that breaks exactly that rule, beside a
# near-miss at the boundary that must pass, so a dropped or inverted test fails here.
def _res(kept, start, finish, q, conf, makespan, status=0):
    return dict(kept=np.array(kept, np.int8), start=np.array(start, np.int32),
                finish=np.array(finish, np.int32), q_total=np.array([q], np.int64),
                conf_micro=np.array([conf], np.int64), makespan=np.array([makespan], np.int32),
                status=np.array([status], np.uint8))


CK = OracleConfig(delta_micro=100_000)
CK_ENF = OracleConfig(drop_mode=1, delta_micro=100_000)


def test_checker_bit1_start_before_release():
    """a job cannot start before it is released (reading R9: start = max(F, r))."""
    b = batch_from_tasks([dict(r=3, d=10, m=2, w=[], a0=500_000, g=[])])
    assert oracle.check(b, _res([0], [3], [5], 5, 500_000, 5), CK)[0] == 0       # start == release
    assert oracle.check(b, _res([0], [2], [4], 5, 500_000, 4), CK)[0] == 1       # one tick early


def test_checker_bit4_finish_after_deadline():
    """every kept task finishes by its (inclusive, adjusted) deadline."""
    b = batch_from_tasks([dict(r=0, d=5, m=2, w=[], a0=500_000, g=[])])
    assert oracle.check(b, _res([0], [3], [5], 5, 500_000, 5), CK)[0] == 0       # finish == deadline
    assert oracle.check(b, _res([0], [4], [6], 5, 500_000, 6), CK)[0] == 4


def test_checker_bit8_overlap():
    """one GPU, jobs back to back in EDF order - a job may not start before the previous
    kept job in that order has finished."""
    ts = [dict(r=0, d=10, m=2, w=[], a0=500_000, g=[]), dict(r=0, d=10, m=2, w=[], a0=500_000, g=[])]
    b = batch_from_tasks(ts)
    assert oracle.check(b, _res([0, 0], [0, 2], [2, 4], 10, 1_000_000, 4), CK)[0] == 0   # touching
    assert oracle.check(b, _res([0, 0], [0, 1], [2, 3], 10, 1_000_000, 3), CK)[0] == 8


def test_checker_bit16_processor_demand():
    """for all t1 < t2 the kept jobs released at or after t1 with deadline at most t2
    need at most t2 - t1 ticks.  Two jobs of 3 ticks with a common deadline 5 cannot both be
    kept (demand 6 > 5); at deadline 6 they can (demand == window)."""
    ts = [dict(r=0, d=5, m=3, w=[], a0=500_000, g=[]), dict(r=0, d=5, m=3, w=[], a0=500_000, g=[])]
    bits = oracle.check(batch_from_tasks(ts), _res([0, 0], [0, 3], [3, 6], 10, 1_000_000, 6), CK)[0]
    assert bits & 16 and bits & 4
    ok = [dict(t, d=6) for t in ts]
    assert oracle.check(batch_from_tasks(ok), _res([0, 0], [0, 3], [3, 6], 10, 1_000_000, 6), CK)[0] == 0
    # demand counted over the released window [t1, t2]: a late-released job only fits its own window
    ts = [dict(r=4, d=6, m=3, w=[], a0=500_000, g=[]), dict(r=0, d=9, m=2, w=[], a0=500_000, g=[])]
    bits = oracle.check(batch_from_tasks(ts), _res([0, 0], [4, 7], [7, 9], 10, 1_000_000, 9), CK)[0]
    assert bits & 16          # job 0 alone: demand 3 in [4, 6]
    ts[0]["d"] = 7
    assert oracle.check(batch_from_tasks(ts), _res([0, 0], [4, 7], [7, 9], 10, 1_000_000, 9), CK)[0] == 0


def test_checker_bit32_drop_when_enforced():
    """P:L70 "if dropping entire tasks is disallowed": in ENFORCED mode a dropped task is a
    violation; in DROP_ALLOWED mode the same plan is valid, and INFEASIBLE is never right there
    (the empty plan is always feasible)."""
    ts = [dict(r=0, d=10, m=2, w=[], a0=500_000, g=[]), dict(r=0, d=10, m=2, w=[], a0=300_000, g=[])]
    b = batch_from_tasks(ts)
    r = _res([0, -1], [0, -1], [2, -1], 5, 500_000, 2)
    assert oracle.check(b, r, CK)[0] == 0
    assert oracle.check(b, r, CK_ENF)[0] == 32
    inf = _res([-1, -1], [-1, -1], [-1, -1], 0, 0, 0, status=oracle.INFEASIBLE)
    assert oracle.check(b, inf, CK_ENF)[0] == 0
    assert oracle.check(b, inf, CK)[0] == 32


def test_checker_bits_64_128_bookkeeping():
    """Q, confidence and makespan must be recomputable from the plan; kept out of [-1, S_i] or
    a dropped task with times is an encoding error."""
    b = batch_from_tasks([dict(r=0, d=10, m=2, w=[1], a0=500_000, g=[200_000])])
    assert oracle.check(b, _res([1], [0], [3], 7, 700_000, 3), CK)[0] == 0
    assert oracle.check(b, _res([1], [0], [3], 6, 700_000, 3), CK)[0] == 64       # Q
    assert oracle.check(b, _res([1], [0], [3], 7, 699_999, 3), CK)[0] == 64       # confidence
    assert oracle.check(b, _res([1], [0], [3], 7, 700_000, 4), CK)[0] == 64       # makespan
    assert oracle.check(b, _res([2], [0], [3], 7, 700_000, 3), CK)[0] & 128       # kept > S_i
    assert oracle.check(b, _res([-1], [0], [-1], 0, 0, 0), CK)[0] & 128           # drop with a start

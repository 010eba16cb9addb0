"""Pins of the NEXT-3 oracle: utility heuristics and Eq. 5's greedy
reassignment, against SPEC's worked examples and brute-force enumeration
of the single-extension search."""
import numpy as np
import pytest

import gen
import oracle
from oracle import OracleConfig, UTIL_EXP, UTIL_GIVEN, UTIL_LIN, UTIL_MAX
from oracle import definition
from tests._instances import batch_from_tasks


def test_heuristic_examples():
    """S:L110-113 predict_next examples."""
    assert oracle.predict_next(UTIL_EXP, 600_000, 1, 2) == 800_000          # 0.6 -> 0.8
    assert oracle.predict_next(UTIL_MAX, 300_000, 1, 2) == 1_000_000        # -> 1.0
    assert oracle.predict_next(UTIL_LIN, 500_000, 40, 60) == 750_000        # 0.5 * 0.06/0.04
    assert oracle.predict_next(UTIL_LIN, 800_000, 40, 80) == 1_000_000      # clamp
    assert oracle.predict_next(UTIL_LIN, 420_000, 50, 50) == 420_000        # identity
    assert oracle.predict_next(UTIL_EXP, 1_000_000, 1, 2) == 1_000_000      # fixed point


def test_exp_curve_iterates():
    """Exp from 0.6 over two stages -> [0.6, 0.8, 0.9]; 1 - (1 - r)/2^k."""
    r, out = 600_000, [600_000]
    for _ in range(5):
        r = oracle.predict_next(UTIL_EXP, r, 1, 2)
        out.append(r)
    assert out[:3] == [600_000, 800_000, 900_000]
    for k, v in enumerate(out):
        assert abs(v - (1_000_000 - 400_000 / 2 ** k)) <= 1


def _j1_t2(observed, g2=300_000, w2=1):
    # J_1: mandatory (w 1, conf .5) + one optional stage (w 1, +.1) planned; T2: mandatory + one stage
    tasks = [dict(r=0, d=10, m=1, w=[1], a0=500_000, g=[100_000]),
             dict(r=0, d=10, m=1, w=[w2], a0=300_000, g=[g2])]
    return batch_from_tasks(tasks), np.array([1, 0], np.int8), np.array([0], np.int8), np.array([observed], np.uint32)


def test_spec_unchanged_when_not_lower():
    """new curve pointwise >= old -> plan unchanged."""
    b, kept, done, obs = _j1_t2(520_000)
    out = oracle.reassign(b, kept, done, obs, UTIL_GIVEN)
    assert list(out["kept"]) == [1, 0] and out["swapped"][0] == 0
    assert out["conf_micro"][0] == 620_000 + 300_000  # J_1 on its re-predicted curve


def test_spec_swap():
    """J_1's remaining stage (wcet 1, gain .1) yields to T2's extension (wcet 1, gain .3)."""
    b, kept, done, obs = _j1_t2(450_000)
    out = oracle.reassign(b, kept, done, obs, UTIL_GIVEN)
    assert list(out["kept"]) == [0, 1] and out["swapped"][0] == 1
    assert out["conf_micro"][0] == 450_000 + 600_000
    assert list(out["start"]) == [0, 1] and list(out["finish"]) == [1, 3]


def test_spec_no_candidate_fits():
    """no extension fits the released budget -> plan unchanged."""
    b, kept, done, obs = _j1_t2(450_000, w2=2)
    out = oracle.reassign(b, kept, done, obs, UTIL_GIVEN)
    assert list(out["kept"]) == [1, 0] and out["swapped"][0] == 0


def test_gain_must_beat_remaining():
    """swap only if the extension's gain exceeds J_1's remaining gain."""
    b, kept, done, obs = _j1_t2(450_000, g2=100_000)  # equal gains -> keep
    out = oracle.reassign(b, kept, done, obs, UTIL_GIVEN)
    assert out["swapped"][0] == 0


def _brute_reassign(tasks, kept, done, observed, heuristic):
    """Enumerate every single extension (i after J_1 in EDF order, depth l) by the definition."""
    order = definition.edf_order(tasks)
    p1 = next((p for p, i in enumerate(order) if kept[i] >= 0), None)
    if p1 is None:
        return list(kept), 0
    j1 = order[p1]
    C1, R1 = definition.derive(tasks[j1])
    l1, l1s = done, kept[j1]
    Rn = list(R1)
    Rn[l1] = observed
    for k in range(l1 + 1, len(R1)):
        if heuristic == UTIL_GIVEN:
            Rn[k] = Rn[k - 1] + R1[k] - R1[k - 1]
        else:
            Rn[k] = oracle.predict_next(heuristic, Rn[k - 1], C1[k - 1], C1[k])
    if all(Rn[k] >= R1[k] for k in range(l1, l1s + 1)):
        return list(kept), 0
    released, rem = C1[l1s] - C1[l1], Rn[l1s] - Rn[l1]
    best = None
    for pos in range(p1 + 1, len(order)):
        i = order[pos]
        C, R = definition.derive(tasks[i])
        ki = kept[i]
        for l in range(ki + 1, len(C)):
            cost = C[l] - (C[ki] if ki >= 0 else 0)
            gain = R[l] - (R[ki] if ki >= 0 else 0)
            if cost > released:
                continue
            plan = list(kept)
            plan[j1], plan[i] = l1, l
            choice = [None if plan[q] < 0 else plan[q] for q in order]
            ok = definition.evaluate(tasks, order, choice, 1)[0]
            if ok and (best is None or gain > best[0]):
                best = (gain, i, l)
    if best is not None and best[0] > rem:
        plan = list(kept)
        plan[j1], plan[best[1]] = l1, best[2]
        return plan, 1
    return list(kept), 0


@pytest.mark.parametrize("heuristic", [UTIL_GIVEN, UTIL_MAX, UTIL_EXP, UTIL_LIN])
def test_reassign_matches_enumeration(heuristic):
    rng = np.random.default_rng(40 + heuristic)
    batch = gen.tiny_random(rng, 1500, max_tasks=6, max_opt=3, horizon=30, p_nonmono=0.0)
    plan = oracle.solve(batch, OracleConfig(delta_micro=100_000), oracle.PAPER)
    done = np.zeros(batch.n_instances, np.int8)
    obs = np.zeros(batch.n_instances, np.uint32)
    for b in range(batch.n_instances):
        lo, hi = batch.task_begin[b], batch.task_begin[b + 1]
        k = plan["kept"][lo:hi]
        first = [i for i in definition.edf_order(definition.tasks_from_batch(batch, b)) if k[i] >= 0]
        if first:
            done[b] = rng.integers(0, k[first[0]] + 1)
            obs[b] = rng.integers(0, 101) * 10_000
    out = oracle.reassign(batch, plan["kept"], done, obs, heuristic)
    nsw = 0
    for b in range(batch.n_instances):
        lo, hi = batch.task_begin[b], batch.task_begin[b + 1]
        tasks = definition.tasks_from_batch(batch, b)
        ref, sw = _brute_reassign(tasks, [int(x) for x in plan["kept"][lo:hi]], int(done[b]), int(obs[b]),
                                  heuristic)
        assert list(out["kept"][lo:hi]) == ref, b
        assert out["swapped"][b] == sw
        nsw += sw
    if heuristic != UTIL_MAX:  # Max predicts 1.0 ahead, so J_1's remaining gain rarely loses
        assert nsw > 0
    # never breaks EDF feasibility
    bits = oracle.check(batch, out, OracleConfig(delta_micro=100_000))
    assert ((bits & ~64) == 0).all()  # Q / confidence differ by design (J_1's new curve)

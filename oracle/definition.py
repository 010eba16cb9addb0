"""The canonical depth-assignment problem, written out and enumerated.

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).  Pure Python, tiny inputs
only.  This is the plain definition the C brute force (O1) is pinned to; it is
written independently from ``ic_oracle.c`` and uses Python integers.

Definition:
  * C_i(k) = m_i + sum of the first k optional WCETs      (P_i^L)
  * R_i(k) = a_i0 + sum of the first k optional gains      (R_i^L)
  * q_i(k) = R_i(k) // Delta
  * a plan picks k_i in {DROP, 0..S_i} (no DROP when enforced)
  * the kept tasks run in EDF order by (deadline, release, index);
    each starts at max(previous finish, release) and must finish by its
    deadline (inclusive, "F_i^L <= d_i")
  * best plan: largest sum of q; then smallest makespan; then the smallest
    choice vector read from the last EDF task backwards, DROP < 0 < 1 < ...
"""
from __future__ import annotations

import itertools

DROP = None


def derive(task):
    """task = dict(r, d, m, w=[...], a0, g=[...]) -> (C list, R list)."""
    C, R = [task["m"]], [task["a0"]]
    for w, g in zip(task["w"], task["g"]):
        C.append(C[-1] + w)
        R.append(R[-1] + g)
    return C, R


def fptas_delta(tasks, eps_micro):
    """Delta = eps * R / N with R the best individually feasible reward (Theorem 1)."""
    best = 0
    for t in tasks:
        C, R = derive(t)
        for c, r in zip(C, R):
            if t["r"] + c <= t["d"]:
                best = max(best, r)
    if not tasks:
        return 1
    return max(1, eps_micro * best // (1_000_000 * len(tasks)))


def edf_order(tasks):
    return sorted(range(len(tasks)), key=lambda i: (tasks[i]["d"], tasks[i]["r"], i))


def evaluate(tasks, order, choice, delta):
    """choice[pos] for EDF position pos: DROP or k.  Returns (feasible, Q, makespan, conf, times)."""
    F, Q, conf, times = 0, 0, 0, {}
    for pos, i in enumerate(order):
        k = choice[pos]
        if k is DROP:
            continue
        C, R = derive(tasks[i])
        s = max(F, tasks[i]["r"])
        f = s + C[k]
        if f > tasks[i]["d"]:
            return False, None, None, None, None
        F = f
        Q += R[k] // delta
        conf += R[k]
        times[i] = (s, f)
    return True, Q, F, conf, times


def solve(tasks, delta, enforced=False):
    """Enumerate every plan; return dict(kept, start, finish, Q, makespan, conf) or None."""
    order = edf_order(tasks)
    ranges = []
    for i in order:
        ks = list(range(len(tasks[i]["w"]) + 1))
        ranges.append(ks if enforced else [DROP] + ks)

    def rank(k):
        return -1 if k is DROP else k

    best = None
    for choice in itertools.product(*ranges):
        ok, Q, F, conf, times = evaluate(tasks, order, choice, delta)
        if not ok:
            continue
        key = (-Q, F, tuple(rank(k) for k in reversed(choice)))
        if best is None or key < best[0]:
            best = (key, choice, Q, F, conf, times)
    if best is None:
        return None
    _, choice, Q, F, conf, times = best
    kept = [-1] * len(tasks)
    start = [-1] * len(tasks)
    finish = [-1] * len(tasks)
    for pos, i in enumerate(order):
        if choice[pos] is not DROP:
            kept[i] = choice[pos]
            start[i], finish[i] = times[i]
    return dict(kept=kept, start=start, finish=finish, Q=Q, makespan=F, conf=conf)


def tasks_from_batch(batch, b):
    lo, hi = int(batch.task_begin[b]), int(batch.task_begin[b + 1])
    out = []
    for t in range(lo, hi):
        S = int(batch.n_opt[t])
        out.append(dict(r=int(batch.release[t]), d=int(batch.deadline[t]), m=int(batch.mand_wcet[t]),
                        w=[int(x) for x in batch.opt_wcet[t, :S]], a0=int(batch.mand_conf[t]),
                        g=[int(x) for x in batch.opt_gain[t, :S]]))
    return out

"""Load sweep of the edge-server simulator (NEXT-4): accuracy / miss rate / depth per policy.

usage: PYTHONPATH=. python tools/sim_sweep.py [servers] [period]   (period 0 = closed loop)"""
import sys
import paper_2011_01112_b200 as pkg

servers = int(sys.argv[1]) if len(sys.argv) > 1 else 256
period = int(sys.argv[2]) if len(sys.argv) > 2 else 0
for clients in (2, 4, 8, 12, 16, 20, 28):
    row = []
    for name, kw in (("plan-exp", dict(policy="planner")),
                     ("plan-opt", dict(policy="planner", utility=pkg.IC_SIM_UTIL_ORACLE)),
                     ("plan-exp-d.02", dict(policy="planner", delta_micro=20_000)),
                     ("edf", dict(policy="edf")), ("lcf", dict(policy="lcf")), ("rr", dict(policy="rr"))):
        r = pkg.simulate(pkg.SimConfig(servers=servers, clients=clients, requests_per_client=20, period=period,
                                       **kw))
        row.append(f"{name} {r['accuracy']:.3f}/{r['miss_rate']:.3f}/{r['mean_depth']:.2f}")
    print(f"K={clients:2d} | " + " | ".join(row), flush=True)

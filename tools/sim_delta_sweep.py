"""Delta trade-off of the RTDeepIoT planner (NEXT-4; §IV-C "Hyper-parameter Tuning",
P:L524-530): accuracy / miss rate of the planner over the reward step Delta, with the
scheduler's cost charged to the server (ic_sim_config.plan_cells_per_tick) and without.

The cost model is calibrated so that planning takes about 3 % of the server's busy time at
the paper's Delta = 0.1 and K = 20 (the middle of the paper's measured 0.5 % - 6 % overhead,
P:L536), then held fixed while Delta varies — a finer Delta makes the paper's reward-indexed
table (N x Qmax cells) proportionally larger, so its planning time grows.

usage: PYTHONPATH=. python tools/sim_delta_sweep.py [servers] [period]
"""
import sys

import paper_2011_01112_b200 as pkg

servers = int(sys.argv[1]) if len(sys.argv) > 1 else 256
period = int(sys.argv[2]) if len(sys.argv) > 2 else 600
base = dict(servers=servers, requests_per_client=20, period=period, policy="planner")


def overhead(r):
    return r["plan_ticks"] / max(1, r["plan_ticks"] + r["busy_ticks"])


# calibrate cells per tick: ~3 % planning overhead at Delta = 0.1, K = 20
lo, hi = 1, 1 << 20
while hi / lo > 1.15:
    mid = int((lo * hi) ** 0.5)
    ov = overhead(pkg.simulate(pkg.SimConfig(clients=20, delta_micro=100_000, plan_cells_per_tick=mid,
                                             **dict(base, servers=min(servers, 64)))))
    lo, hi = (lo, mid) if ov < 0.03 else (mid, hi)
cpt = hi
print(f"# calibrated plan_cells_per_tick = {cpt} (~3% planning overhead at Delta=0.1, K=20)", flush=True)
print("# K | Delta | free planning: acc/miss/depth | costed planning: acc/miss/depth/overhead", flush=True)
for clients in (12, 20, 28):
    for d in (20_000, 50_000, 100_000, 200_000, 500_000):
        f = pkg.simulate(pkg.SimConfig(clients=clients, delta_micro=d, **base))
        c = pkg.simulate(pkg.SimConfig(clients=clients, delta_micro=d, plan_cells_per_tick=cpt, **base))
        print(f"{clients:2d} | {d / 1e6:.2f} | {f['accuracy']:.3f}/{f['miss_rate']:.3f}/{f['mean_depth']:.2f} | "
              f"{c['accuracy']:.3f}/{c['miss_rate']:.3f}/{c['mean_depth']:.2f}/{overhead(c):.3f}", flush=True)
    for pol in ("edf", "lcf", "rr"):
        r = pkg.simulate(pkg.SimConfig(clients=clients, **dict(base, policy=pol)))
        print(f"{clients:2d} | {pol} | {r['accuracy']:.3f}/{r['miss_rate']:.3f}/{r['mean_depth']:.2f}", flush=True)

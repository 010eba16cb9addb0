"""GPU parity: the sm_100a kernels (through the C ABI) against the CPU oracle.

Decisions, integer times, Q, makespan and status must match bit for bit;
total confidence to 1e-6 relative (north_star).  Inputs are seeded: the
paper-shaped generator (gen/) and small adversarial instances.
"""
import numpy as np
import pytest

import gen
import oracle
from oracle import OracleConfig, BRUTE, PAPER, TIME
from tests._instances import batch_from_tasks, batch_from_many
from tests.gpu_util import assert_parity, gpu_solve, stats_from

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("no CUDA device", allow_module_level=True)


@pytest.mark.parametrize("mode", [0, 1])
@pytest.mark.parametrize("delta,eps", [(100_000, 0), (30_000, 0), (0, 250_000), (0, 100_000)])
def test_tiny_random_vs_brute_force(mode, delta, eps):
    rng = np.random.default_rng(100 + mode + delta + eps)
    batch = gen.tiny_random(rng, 20000, max_tasks=5, max_opt=3, horizon=24)
    cfg = OracleConfig(drop_mode=mode, delta_micro=delta, epsilon_micro=eps, max_tasks=5, max_horizon=24)
    ref = oracle.solve(batch, cfg, BRUTE)
    got = gpu_solve(batch, max_tasks=5, max_opt=3, max_horizon=24, drop_mode=mode, delta=delta, eps=eps)
    assert_parity(got, ref, f"tiny mode={mode} delta={delta} eps={eps}")


@pytest.mark.parametrize("name,n,algo", [("C1", 20000, PAPER), ("C2", 3000, PAPER), ("C3", 300, TIME),
                                         ("C4", 3, TIME)])
@pytest.mark.parametrize("mode", [0, 1])
def test_paper_shaped_configs(name, n, algo, mode):
    cw = gen.CONFIGS[name]
    batch = gen.generate(cw, n)
    ocfg = OracleConfig(drop_mode=mode, epsilon_micro=cw.epsilon_micro, max_tasks=cw.n_tasks,
                        max_horizon=cw.horizon)
    ref = oracle.solve(batch, ocfg, algo)
    got = gpu_solve(batch, max_tasks=cw.n_tasks, max_opt=cw.n_opt, max_horizon=cw.horizon, drop_mode=mode,
                    eps=cw.epsilon_micro)
    assert_parity(got, ref, f"{name} mode={mode}")
    assert (oracle.check(batch, got, ocfg) == 0).all()


@pytest.mark.parametrize("name", ["C2", "C3"])
def test_paper_delta_point_one(name):
    """The paper's experimental default Delta = 0.1."""
    cw = gen.CONFIGS[name]
    batch = gen.generate(cw, 400 if name == "C2" else 100)
    ref = oracle.solve(batch, OracleConfig(delta_micro=100_000, max_tasks=cw.n_tasks, max_horizon=cw.horizon),
                       PAPER)
    got = gpu_solve(batch, max_tasks=cw.n_tasks, max_opt=cw.n_opt, max_horizon=cw.horizon, delta=100_000)
    assert_parity(got, ref, name)


def test_releases_and_variable_stages():
    """Releases (frames mode), ragged S_i, non-monotone curves at C2 scale."""
    rng = np.random.default_rng(5)
    parts = []
    for _ in range(300):
        N = int(rng.integers(1, 40))
        ts = []
        for _ in range(N):
            S = int(rng.integers(0, 5))
            lv = rng.integers(0, 101, S + 1) * 10_000
            if rng.random() < 0.5:
                lv = np.sort(lv)
            ts.append(dict(r=int(rng.integers(0, 300)) if rng.random() < 0.5 else 0,
                           d=int(rng.integers(-5, 1024)), m=int(rng.integers(1, 40)),
                           w=[int(x) for x in rng.integers(1, 40, S)], a0=int(lv[0]),
                           g=[int(x) for x in np.diff(lv)]))
        parts.append(ts)
    batch = batch_from_many(parts, 4)
    for mode in (0, 1):
        ocfg = OracleConfig(drop_mode=mode, epsilon_micro=100_000, max_tasks=40, max_horizon=1024)
        ref = oracle.solve(batch, ocfg, TIME)
        got = gpu_solve(batch, max_tasks=40, max_opt=4, max_horizon=1024, drop_mode=mode)
        assert_parity(got, ref, f"releases mode={mode}")


def test_general_path_long_tasks():
    """Options longer than the NEG pad take the clamped general path."""
    rng = np.random.default_rng(6)
    parts = []
    for _ in range(60):
        N = int(rng.integers(1, 12))
        ts = []
        for _ in range(N):
            S = int(rng.integers(0, 4))
            lv = np.sort(rng.integers(0, 101, S + 1)) * 10_000
            ts.append(dict(r=0, d=int(rng.integers(500, 4096)), m=int(rng.integers(1, 1500)),
                           w=[int(x) for x in rng.integers(1, 900, S)], a0=int(lv[0]),
                           g=[int(x) for x in np.diff(lv)]))
        parts.append(ts)
    batch = batch_from_many(parts, 3)
    ref = oracle.solve(batch, OracleConfig(delta_micro=20_000, max_tasks=16, max_horizon=4096), TIME)
    got = gpu_solve(batch, max_tasks=16, max_opt=3, max_horizon=4096, delta=20_000)
    assert_parity(got, ref, "general path")


def test_many_tasks_block_sort():
    """N > 32 uses the shared-memory bitonic sort; ragged N; equal deadlines."""
    rng = np.random.default_rng(7)
    parts = []
    for _ in range(100):
        N = int(rng.integers(0, 300))
        ts = []
        dl = rng.integers(0, 200, N)
        if rng.random() < 0.5:
            dl = dl // 20 * 20  # many equal deadlines
        for i in range(N):
            S = int(rng.integers(0, 3))
            lv = np.sort(rng.integers(0, 101, S + 1)) * 10_000
            ts.append(dict(r=0, d=int(dl[i]), m=int(rng.integers(1, 4)),
                           w=[int(x) for x in rng.integers(1, 4, S)], a0=int(lv[0]),
                           g=[int(x) for x in np.diff(lv)]))
        parts.append(ts)
    batch = batch_from_many(parts, 2)
    ref = oracle.solve(batch, OracleConfig(epsilon_micro=100_000, max_tasks=300, max_horizon=256), TIME)
    got = gpu_solve(batch, max_tasks=300, max_opt=2, max_horizon=256)
    assert_parity(got, ref, "block sort")


def test_bad_input_and_empty():
    base = dict(r=0, d=5, m=1, w=[1], a0=300_000, g=[100_000])
    lists = [[], [base], [dict(base, m=0)], [dict(base, w=[0])], [dict(base, r=-1)], [dict(base, d=64)],
             [dict(base, a0=1_000_001)], [dict(base, g=[800_000])], [base] * 9, [dict(base, g=[-200_000])]]
    batch = batch_from_many(lists, 1)
    ref = oracle.solve(batch, OracleConfig(delta_micro=100_000, max_tasks=8, max_horizon=64), PAPER)
    got = gpu_solve(batch, max_tasks=8, max_opt=1, max_horizon=64, delta=100_000)
    assert_parity(got, ref, "bad input")
    assert list(got["status"]) == [0, 0, 2, 2, 2, 2, 2, 2, 2, 0]


def test_limit_status():
    """16 * sum max q + 16 N >= 2^30 cannot be packed: IC_INST_LIMIT, everything dropped."""
    t = dict(r=0, d=10, m=1, w=[], g=[], a0=1_000_000)
    batch = batch_from_tasks([t] * 70)  # Delta = 1 -> q = 1e6 per task
    got = gpu_solve(batch, max_tasks=70, max_opt=0, max_horizon=64, delta=1)
    assert got["status"][0] == 3 and (got["kept"] == -1).all()


def test_host_entry_point_and_stats():
    cw = gen.CONFIGS["C2"]
    batch = gen.generate(cw, 500)
    a = gpu_solve(batch, max_tasks=32, max_opt=4, max_horizon=1024)
    b = gpu_solve(batch, max_tasks=32, max_opt=4, max_horizon=1024, host=True)
    assert_parity(a, b, "host vs device")
    np.testing.assert_array_equal(a["stats"], stats_from(a, batch))
    np.testing.assert_array_equal(b["stats"], stats_from(a, batch))


def test_device_generator_matches_host():
    import paper_2011_01112_b200 as pkg
    for name in ("C1", "C2", "C3"):
        cw = gen.CONFIGS[name]
        host = gen.generate(cw, 257, id_offset=1000)
        gc = cw.gen_config()
        dev = pkg.gen_batch_device(gc.seed, gc.n_tasks, gc.n_opt, gc.opt_stride, gc.horizon, gc.u_lo_q16,
                                   gc.u_hi_q16, gc.d_lo, 257, id_offset=1000)
        torch.cuda.synchronize()
        for f, _, _ in pkg.INPUT_FIELDS:
            np.testing.assert_array_equal(dev[f].cpu().numpy(), getattr(host, f), err_msg=f)


@pytest.mark.parametrize("decisions", [0, 1, 2])
def test_decision_placement(decisions):
    """Decisions in the global double buffer (default), in shared memory, or one global buffer
    give identical results."""
    cw = gen.CONFIGS["C2"]
    batch = gen.generate(cw, 300)
    ref = oracle.solve(batch, OracleConfig(epsilon_micro=100_000, max_tasks=32, max_horizon=1024), PAPER)
    got = gpu_solve(batch, max_tasks=32, max_opt=4, max_horizon=1024, tuning=dict(decisions=decisions))
    assert got["_info"]["decisions_in_smem"] == (1 if decisions == 1 else 0)
    assert_parity(got, ref, f"decisions={decisions}")


@pytest.mark.parametrize("tuning", [dict(dp_warps=1, kernel=1), dict(kernel=2), dict(kernel=2, pad_cols=32),
                                    dict(kernel=2, axis=1), dict(dp_warps=2), dict(dp_warps=4), dict(dp_warps=8),
                                    dict(dp_warps=16), dict(in_place=1, dp_warps=8), dict(in_place=1, dp_warps=16),
                                    dict(pad_cols=32), dict(slots=1, dp_warps=2),
                                    dict(slots=1, in_place=1, dp_warps=8), dict(option_tables=1, dp_warps=8),
                                    dict(option_tables=1, in_place=1, dp_warps=16),
                                    dict(in_place=1, dp_warps=15), dict(dp_warps=15), dict(option_tables=1, in_place=1, dp_warps=15),
                                    dict(option_tables=1, dp_warps=8, decisions=2), dict(no_vec_loads=1),
                                    dict(discard=1), dict(kernel=2, discard=2),
                                    dict(decisions=1, dp_warps=2)])
@pytest.mark.parametrize("mode", [0, 1])
def test_every_kernel_variant(tuning, mode):
    """Every compiled (DP warps, in-place rows, drop mode, decision placement) variant agrees."""
    rng = np.random.default_rng(11 + mode)
    parts = [gen.generate("C3", 40)]
    tiny = gen.tiny_random(rng, 400, max_tasks=6, max_opt=8, horizon=4096)
    tiny.deadline[:] = np.where(tiny.deadline >= 0, tiny.deadline * 170 % 4096, tiny.deadline)
    tiny.mand_wcet[:] = tiny.mand_wcet * 37
    tiny.opt_wcet[:] = tiny.opt_wcet * 29
    parts.append(tiny)
    batch = gen.concat(parts, 8)
    ocfg = OracleConfig(drop_mode=mode, epsilon_micro=100_000, max_tasks=64, max_horizon=4096)
    ref = oracle.solve(batch, ocfg, TIME)
    got = gpu_solve(batch, max_tasks=64, max_opt=8, max_horizon=4096, drop_mode=mode, tuning=tuning)
    assert_parity(got, ref, f"variant {tuning} mode={mode}")


def test_c5_sweep_blocks():
    """C5's utilisation blocks (U = 1, 2, 4, 8): instances straddling every block boundary."""
    cw = gen.CONFIGS["C5"]
    parts = [gen.generate(cw, 24, id_offset=(k << 22) - 12) for k in (1, 2, 3)]
    parts.append(gen.generate(cw, 12, id_offset=(4 << 22) - 12))
    batch = gen.concat(parts, cw.n_opt)
    ocfg = OracleConfig(epsilon_micro=cw.epsilon_micro, max_tasks=cw.n_tasks, max_horizon=cw.horizon)
    ref = oracle.solve(batch, ocfg, TIME)
    got = gpu_solve(batch, max_tasks=cw.n_tasks, max_opt=cw.n_opt, max_horizon=cw.horizon)
    assert_parity(got, ref, "C5 blocks")
    # overload shows up as planned misses only at the high-U blocks
    tb = batch.task_begin
    drops = [(got["kept"][tb[b]:tb[b + 1]] < 0).mean() for b in range(batch.n_instances)]
    assert np.mean(drops[-12:]) > np.mean(drops[:12])


@pytest.mark.parametrize("axis", [1, 2])
@pytest.mark.parametrize("mode", [0, 1])
@pytest.mark.parametrize("delta", [100_000, 20_000, 0])
def test_reward_axis(axis, mode, delta):
    """NEXT-1: the reward-indexed sweep (the paper's P(i, r) table, forced with tuning axis=2)
    and the time axis (axis=1) give the same canonical plans; instances with releases
    stay on the time axis."""
    rng = np.random.default_rng(31 + mode + delta)
    parts = [gen.tiny_random(rng, 6000, max_tasks=6, max_opt=3, horizon=40, p_release=0.0),
             gen.tiny_random(rng, 500, max_tasks=6, max_opt=3, horizon=40, p_release=0.5)]
    batch = gen.concat(parts, 3)
    ocfg = OracleConfig(drop_mode=mode, delta_micro=delta, epsilon_micro=300_000, max_tasks=6, max_horizon=40)
    ref = oracle.solve(batch, ocfg, BRUTE)
    got = gpu_solve(batch, max_tasks=6, max_opt=3, max_horizon=40, drop_mode=mode, delta=delta, eps=300_000,
                    tuning=dict(axis=axis))
    assert_parity(got, ref, f"axis={axis} mode={mode} delta={delta}")


@pytest.mark.parametrize("name", ["C2", "C3", "C4"])
@pytest.mark.parametrize("mode", [0, 1])
def test_reward_axis_paper_delta(name, mode):
    """At the paper's Delta = 0.1 the reward axis is the shorter sweep and is auto-selected."""
    cw = gen.CONFIGS[name]
    batch = gen.generate(cw, {"C2": 300, "C3": 60, "C4": 2}[name])
    ocfg = OracleConfig(drop_mode=mode, delta_micro=100_000, max_tasks=cw.n_tasks, max_horizon=cw.horizon)
    ref = oracle.solve(batch, ocfg, TIME)
    for axis in (0, 1, 2):
        got = gpu_solve(batch, max_tasks=cw.n_tasks, max_opt=cw.n_opt, max_horizon=cw.horizon, drop_mode=mode,
                        delta=100_000, tuning=dict(axis=axis))
        assert_parity(got, ref, f"{name} axis={axis} mode={mode}")


@pytest.mark.parametrize("heuristic", [0, 1, 2, 3])
@pytest.mark.parametrize("shape", ["tiny", "C2", "C3"])
def test_reassign_vs_oracle(heuristic, shape):
    """NEXT-3: stage-completion reassignment (Eq. 5) on the GPU against the oracle."""
    import paper_2011_01112_b200 as pkg
    from tests.gpu_util import to_device
    rng = np.random.default_rng(50 + heuristic)
    if shape == "tiny":
        batch = gen.tiny_random(rng, 4000, max_tasks=6, max_opt=3, horizon=30)
        mt, mo, H = 6, 3, 30
    else:
        cw = gen.CONFIGS[shape]
        batch = gen.generate(cw, 2000 if shape == "C2" else 300)
        mt, mo, H = cw.n_tasks, cw.n_opt, cw.horizon
    ocfg = OracleConfig(delta_micro=100_000, max_tasks=mt, max_horizon=H)
    plan = oracle.solve(batch, ocfg, TIME)
    done = np.zeros(batch.n_instances, np.int8)
    obs = np.zeros(batch.n_instances, np.uint32)
    from oracle import definition
    for b in range(batch.n_instances):
        lo, hi = batch.task_begin[b], batch.task_begin[b + 1]
        k = plan["kept"][lo:hi]
        first = [i for i in definition.edf_order(definition.tasks_from_batch(batch, b)) if k[i] >= 0]
        if first:
            done[b] = rng.integers(0, k[first[0]] + 1)
            obs[b] = rng.integers(0, 101) * 10_000
    ref = oracle.reassign(batch, plan["kept"], done, obs, heuristic, ocfg)
    sc = pkg.SchedConfig(max_tasks=mt, max_opt_stages=mo, max_horizon=H, delta_micro=100_000)
    with pkg.Scheduler(sc) as s:
        dev = to_device(batch)
        out = s.reassign_batch(dev, torch.from_numpy(plan["kept"]).cuda(), torch.from_numpy(done).cuda(),
                               torch.from_numpy(obs).cuda(), heuristic)
        torch.cuda.synchronize()
    got = {k: v.cpu().numpy() for k, v in out.items()}
    for k in ("kept", "start", "finish", "conf_micro", "makespan", "status", "swapped"):
        np.testing.assert_array_equal(got[k], ref[k], err_msg=k)
    if heuristic != 1:
        assert got["swapped"].sum() > 0


def _first_tasks(batch, counts):
    """Per instance b keep its first counts[b] tasks (a task set before later arrivals)."""
    from gen import Batch
    parts = []
    for b in range(batch.n_instances):
        one = batch.instance(b)
        m = int(counts[b])
        parts.append(Batch(np.array([0, m], np.int64), one.release[:m], one.deadline[:m], one.mand_wcet[:m],
                           one.n_opt[:m], one.opt_wcet[:m], one.mand_conf[:m], one.opt_gain[:m]))
    return gen.concat(parts, batch.opt_stride)


@pytest.mark.parametrize("ckpt", [1, 4])
@pytest.mark.parametrize("mode", [0, 1])
@pytest.mark.parametrize("shape", ["C2", "tiny"])
def test_incremental_replan(shape, mode, ckpt):
    """NEXT-2 (Alg. 1 from row k): chained arrivals re-planned from the
    state equal a full solve of the grown task set (GPU and oracle)."""
    import paper_2011_01112_b200 as pkg
    from tests.gpu_util import to_device
    rng = np.random.default_rng(70 + mode)
    if shape == "C2":
        cw = gen.WorkloadConfig("C2x", 0, 34, 4, 1024, 0.6, 1.0, 35, 0x2011011102)
        full = gen.generate(cw, 400)
        mt, mo, H = 34, 4, 1024
        base = np.full(full.n_instances, 31)
    else:
        full = gen.tiny_random(rng, 2000, max_tasks=7, max_opt=3, horizon=40)
        mt, mo, H = 7, 3, 40
        sizes = np.diff(full.task_begin)
        keep = sizes >= 3
        full = full.select(np.nonzero(keep)[0])
        base = np.diff(full.task_begin) - 3
    sc = pkg.SchedConfig(max_tasks=mt, max_opt_stages=mo, max_horizon=H, delta_micro=100_000, drop_mode=mode)
    with pkg.Scheduler(sc, dict(ckpt=ckpt)) as s:
        state = torch.zeros(s.state_bytes(full.n_instances), dtype=torch.uint8, device="cuda")
        b0 = _first_tasks(full, base)
        s.solve_batch_state(to_device(b0), state)
        for add in (1, 2, 3):
            bk = _first_tasks(full, base + add)
            out = s.replan_batch(to_device(bk), state)
            torch.cuda.synchronize()
            got = {k: v.cpu().numpy() for k, v in out.items()}
            ref = oracle.solve(bk, OracleConfig(drop_mode=mode, delta_micro=100_000, max_tasks=mt, max_horizon=H),
                               TIME)
            assert_parity(got, ref, f"{shape} arrival {add} mode={mode}")


def test_limit_counts_only_options_that_fit():
    """IC_INST_LIMIT bounds the packed keys by the depths the DP can add (r + C <= d): an
    instance whose huge-q depths can never fit is solved normally."""
    fit = dict(r=0, d=10, m=1, w=[50], g=[999_000], a0=1_000)   # the optional stage never fits
    batch = batch_from_tasks([fit] * 70)
    got = gpu_solve(batch, max_tasks=70, max_opt=1, max_horizon=64, delta=1)
    ref = oracle.solve(batch, OracleConfig(delta_micro=1, max_tasks=70, max_horizon=64), TIME)
    assert got["status"][0] == 0
    assert_parity(got, ref, "limit over fitting depths")


@pytest.mark.parametrize("S,H,lo,hi", [(8, 4096, 1024, 2048), (14, 32768, 256, 1024)])
def test_create_envelope(S, H, lo, hi):
    """include/ic_sched.h "Envelope": the largest max_tasks ic_sched_create accepts lies in the
    documented band; one task more is IC_ERR_LIMIT, and a solve at the boundary is correct."""
    import paper_2011_01112_b200 as pkg
    def ok(n):
        try:
            pkg.Scheduler(pkg.SchedConfig(max_tasks=n, max_opt_stages=S, max_horizon=H)).close()
            return True
        except pkg.ICSchedError as e:
            assert e.rc == pkg.IC_ERR_LIMIT
            return False
    a, b = 1, 4097
    while b - a > 1:
        m = (a + b) // 2
        a, b = (m, b) if ok(m) else (a, m)
    assert lo <= a < hi, a
    assert not ok(a + 1)
    rng = np.random.default_rng(3)
    tiny = gen.tiny_random(rng, 3, max_tasks=6, max_opt=S, horizon=H)
    ts = [dict(r=0, d=int(rng.integers(0, H)), m=int(rng.integers(1, 30)), w=[3] * S, a0=100_000,
               g=[10_000] * S) for _ in range(a)]
    batch = gen.concat([batch_from_tasks(ts, S), tiny], S)
    ocfg = OracleConfig(delta_micro=100_000, max_tasks=a, max_horizon=H)
    ref = oracle.solve(batch, ocfg, TIME)
    got = gpu_solve(batch, max_tasks=a, max_opt=S, max_horizon=H, delta=100_000)
    assert_parity(got, ref, f"envelope S={S} H={H} N={a}")


@pytest.mark.parametrize("name,n", [("C1", 4000), ("C2", 1500)])
@pytest.mark.parametrize("delta", [0, 100_000])
@pytest.mark.parametrize("mode", [0, 1])
def test_solo_and_warp_specialised_kernels_agree(name, n, delta, mode):
    """The one-warp-per-instance kernel (default for H <= 1024) and the warp-specialised kernel
    (tuning kernel=1) both equal the oracle on the same batch, both sweep axes, releases."""
    cw = gen.CONFIGS[name]
    rng = np.random.default_rng(90 + mode)
    rel = gen.tiny_random(rng, 300, max_tasks=cw.n_tasks, max_opt=cw.n_opt, horizon=cw.horizon, p_release=0.7)
    batch = gen.concat([gen.generate(cw, n), rel], cw.n_opt)
    ocfg = OracleConfig(drop_mode=mode, delta_micro=delta, epsilon_micro=cw.epsilon_micro, max_tasks=cw.n_tasks,
                        max_horizon=cw.horizon)
    ref = oracle.solve(batch, ocfg, TIME)
    for tuning in (dict(kernel=0), dict(kernel=1), dict(kernel=2), dict(kernel=0, packed_options=2)):
        got = gpu_solve(batch, max_tasks=cw.n_tasks, max_opt=cw.n_opt, max_horizon=cw.horizon, drop_mode=mode,
                        delta=delta, eps=cw.epsilon_micro, tuning=tuning)
        assert_parity(got, ref, f"{name} {tuning} delta={delta} mode={mode}")
        assert (got["_info"]["threads_per_cta"] == 32) == (tuning["kernel"] != 1)
        if tuning["kernel"] != 1:  # fixed Delta = 0.1: packed option entries unless turned off
            assert got["_info"]["packed_options"] == (1 if delta and "packed_options" not in tuning else 0)


@pytest.mark.parametrize("mode", [0, 1])
def test_hybrid_reward_rows(mode):
    """Fixed Delta = 0.1 at H = 4096 (C3 shape): the solo kernel sweeps the instances whose
    reward-axis rows fit it and defers the rest (releases force the time axis; a time axis
    past its row) to the warp-specialised kernel.  Every instance equals the oracle."""
    cw = gen.CONFIGS["C3"]
    rng = np.random.default_rng(120 + mode)
    rel = gen.tiny_random(rng, 400, max_tasks=12, max_opt=8, horizon=4096, p_release=0.6)
    rel.mand_wcet[:] = rel.mand_wcet * 50
    short = gen.tiny_random(rng, 400, max_tasks=12, max_opt=8, horizon=600, p_release=0.0)
    batch = gen.concat([gen.generate(cw, 300), rel, short], cw.n_opt)
    ocfg = OracleConfig(drop_mode=mode, delta_micro=100_000, max_tasks=64, max_horizon=4096)
    ref = oracle.solve(batch, ocfg, TIME)
    for tuning in (None, dict(packed_options=2)):
        got = gpu_solve(batch, max_tasks=64, max_opt=8, max_horizon=4096, drop_mode=mode, delta=100_000,
                        tuning=tuning)
        assert got["_info"]["hybrid"] == 1 and got["_info"]["kernels_per_solve"] == 2
        assert got["_info"]["packed_options"] == (0 if tuning else 1)
        assert_parity(got, ref, f"hybrid mode={mode} {tuning}")
        np.testing.assert_array_equal(got["stats"], stats_from(got, batch))


@pytest.mark.parametrize("mode", [0, 1])
def test_packed_option_fields_at_their_limits(mode):
    """Packed option entries hold 16-bit fields: the largest Delta-bounded q (Delta = 489 micro:
    q <= 2044, key up to 32703) and option lengths up to C = 4095 at H = 4096 (reward-axis addend
    C*16 + code up to 65529).  Both axes, packed and int2 tables, equal the oracle."""
    rng = np.random.default_rng(700 + mode)
    tiny = gen.tiny_random(rng, 600, max_tasks=6, max_opt=8, horizon=4096)
    tiny.deadline[:] = np.where(tiny.deadline >= 0, 4095 - (tiny.deadline * 7 % 300), tiny.deadline)
    tiny.mand_wcet[:] = np.minimum(tiny.mand_wcet * 500, 3000)
    tiny.opt_wcet[:] = tiny.opt_wcet * 90
    tiny.mand_conf[:] = (tiny.mand_conf.astype(np.int64) * 7 % 400_001).astype(np.uint32)
    tiny.opt_gain[:] = np.abs(tiny.opt_gain.astype(np.int64)) * 13 % 75_001  # R <= 1e6: q up to 2044
    for delta in (489, 100_000):
        ocfg = OracleConfig(drop_mode=mode, delta_micro=delta, max_tasks=6, max_horizon=4096)
        ref = oracle.solve(tiny, ocfg, TIME)
        for tuning in (dict(kernel=2), dict(kernel=2, packed_options=2), dict(kernel=2, axis=1),
                       dict(kernel=2, axis=2)):
            got = gpu_solve(tiny, max_tasks=6, max_opt=8, max_horizon=4096, drop_mode=mode, delta=delta,
                            tuning=tuning)
            assert got["_info"]["packed_options"] == (0 if "packed_options" in tuning else 1)
            assert_parity(got, ref, f"packed limits delta={delta} {tuning}")


def _remove_one(batch, rng):
    """Per instance, remove one random task (the others keep their order); returns the reduced
    batch and the removed task's previous input index, deadline and release."""
    from gen import Batch
    parts, idx, dl, rl = [], [], [], []
    for b in range(batch.n_instances):
        one = batch.instance(b)
        n = one.n_total_tasks
        j = int(rng.integers(0, n))
        keep = np.array([i for i in range(n) if i != j], np.int64)
        parts.append(Batch(np.array([0, n - 1], np.int64), one.release[keep], one.deadline[keep],
                           one.mand_wcet[keep], one.n_opt[keep], one.opt_wcet[keep], one.mand_conf[keep],
                           one.opt_gain[keep]))
        idx.append(j)
        dl.append(int(one.deadline[j]))
        rl.append(int(one.release[j]))
    cat = gen.concat(parts, batch.opt_stride)
    to = lambda a: torch.tensor(a, dtype=torch.int32, device="cuda")
    return cat, to(idx), to(dl), to(rl)


@pytest.mark.parametrize("kernel", [0, 1])
@pytest.mark.parametrize("mode", [0, 1])
@pytest.mark.parametrize("shape", ["C2", "tiny", "H32768", "hybrid"])
def test_departures_and_arrivals(kernel, mode, shape):
    """NEXT-2 both ways (P:L112 arrivals, P:L236 departures): chained departures and arrivals
    re-planned from the state equal full solves of the changed task sets, for the solo and the
    warp-specialised kernels, with in-place rows at H = 32768, and in the hybrid solve (C3 shape
    at Delta = 0.1: the solo kernel keeps the reward-axis instances' state, the warp-specialised
    kernel the deferred ones', and an instance that changes kernel between calls starts over)."""
    import paper_2011_01112_b200 as pkg
    from tests.gpu_util import to_device
    rng = np.random.default_rng(200 + mode + 10 * kernel)
    if shape == "C2":
        full = gen.generate("C2", 300)
        mt, mo, H = 32, 4, 1024
    elif shape == "tiny":
        full = gen.tiny_random(rng, 1500, max_tasks=7, max_opt=3, horizon=40)
        mt, mo, H = 7, 3, 40
    elif shape == "H32768":
        full = gen.tiny_random(rng, 200, max_tasks=8, max_opt=3, horizon=32768, p_release=0.3)
        full.mand_wcet[:] = full.mand_wcet * 900
        full.opt_wcet[:] = full.opt_wcet * 700
        mt, mo, H = 8, 3, 32768
    else:
        rel = gen.tiny_random(rng, 150, max_tasks=12, max_opt=8, horizon=4096, p_release=0.6)
        rel.mand_wcet[:] = rel.mand_wcet * 50
        short = gen.tiny_random(rng, 150, max_tasks=12, max_opt=8, horizon=600, p_release=0.3)
        full = gen.concat([gen.generate("C3", 60), rel, short], 8)
        mt, mo, H = 64, 8, 4096
    full = full.select(np.nonzero(np.diff(full.task_begin) >= 4)[0])
    sc = pkg.SchedConfig(max_tasks=mt, max_opt_stages=mo, max_horizon=H, delta_micro=100_000, drop_mode=mode)
    ocfg = OracleConfig(drop_mode=mode, delta_micro=100_000, max_tasks=mt, max_horizon=H)
    with pkg.Scheduler(sc, dict(kernel=kernel, ckpt=2)) as s:
        state = torch.zeros(s.state_bytes(full.n_instances), dtype=torch.uint8, device="cuda")
        s.solve_batch_state(to_device(full), state)
        cur = full
        for step in range(3):
            cur, j, dl, rl = _remove_one(cur, rng)
            out = s.depart_batch(to_device(cur), j, dl, rl, state)
            torch.cuda.synchronize()
            got = {k: v.cpu().numpy() for k, v in out.items()}
            assert_parity(got, oracle.solve(cur, ocfg, TIME), f"{shape} departure {step} mode={mode} k={kernel}")
        # an arrival after the departures: the full instance's last task is appended again
        parts = [gen.concat([cur.instance(b), _last_task(full.instance(b))], mo) for b in range(cur.n_instances)]
        grown = _merge_tasks(parts, mo)
        out = s.replan_batch(to_device(grown), state)
        torch.cuda.synchronize()
        got = {k: v.cpu().numpy() for k, v in out.items()}
        assert_parity(got, oracle.solve(grown, ocfg, TIME), f"{shape} arrival after departures mode={mode}")


def _last_task(one):
    from gen import Batch
    n = one.n_total_tasks
    return Batch(np.array([0, 1], np.int64), one.release[n - 1:], one.deadline[n - 1:], one.mand_wcet[n - 1:],
                 one.n_opt[n - 1:], one.opt_wcet[n - 1:], one.mand_conf[n - 1:], one.opt_gain[n - 1:])


def _merge_tasks(parts, stride):
    """Each part is a two-instance batch (the current tasks, one new task): one instance each."""
    from gen import Batch
    out = []
    for p in parts:
        T = p.n_total_tasks
        out.append(Batch(np.array([0, T], np.int64), p.release, p.deadline, p.mand_wcet, p.n_opt, p.opt_wcet,
                         p.mand_conf, p.opt_gain))
    return gen.concat(out, stride)

"""The seeded input generator (gen/): determinism, recipe ranges, paper shapes."""
import numpy as np

import gen
from gen import CONFIGS, generate


def test_d_lo_matches_survey():
    """d_lo = ceil(H * D_l / D_u) with the paper's D_l/D_u: 3, 35, 52, 410."""
    assert [CONFIGS[c].d_lo for c in ("C1", "C2", "C3", "C4")] == [3, 35, 52, 410]


def test_deterministic_and_shardable():
    a = generate("C2", 64)
    b = generate("C2", 64)
    for f in ("release", "deadline", "mand_wcet", "n_opt", "opt_wcet", "mand_conf", "opt_gain"):
        np.testing.assert_array_equal(getattr(a, f), getattr(b, f))
    # ids [32, 64) generated as a shard equal the tail of the full batch
    c = generate("C2", 32, id_offset=32)
    np.testing.assert_array_equal(c.deadline, a.deadline[32 * 32:])
    np.testing.assert_array_equal(c.opt_gain, a.opt_gain[32 * 32:])


def test_recipe_ranges():
    cfg = CONFIGS["C3"]
    b = generate(cfg, 200)
    S, H, N = cfg.n_opt, cfg.horizon, cfg.n_tasks
    assert (b.n_opt == S).all() and (b.release == 0).all()
    assert (b.mand_wcet >= 1).all() and (b.opt_wcet >= 1).all()
    w = np.concatenate([b.mand_wcet[:, None], b.opt_wcet], 1)
    raw = b.deadline + w.max(1)
    assert raw.min() >= cfg.d_lo and raw.max() <= H
    assert (b.deadline < H).all()
    R = b.mand_conf.astype(np.int64)[:, None] + np.concatenate(
        [np.zeros((len(w), 1), np.int64), np.cumsum(b.opt_gain, 1)], 1)
    assert (R >= 0).all() and (R <= 1_000_000).all() and (np.diff(R, axis=1) >= 0).all()
    # utilisation: full-depth demand over the horizon within [u_lo, u_hi] (+10% WCET inflation, rounding)
    U = w.sum(1).reshape(-1, N).sum(1) / H
    assert U.min() >= cfg.u_lo * 0.95 and U.max() <= cfg.u_hi * 1.12
    easy = b.mand_conf >= 800_000
    assert 0.4 < easy.mean() < 0.6


def test_exp_heuristic_curve():
    """rho = 0.5 reproduces the paper's Exp heuristic R_{k+1} = R_k + 0.5 (1 - R_k)
    (S:L129 R_k = 1 - (1 - r) / 2^k), up to the integer floor."""
    a0 = 600_000
    resid, R = 1_000_000 - a0, [a0]
    for _ in range(4):
        nr = (resid * 32768) >> 16  # the generator's step with rho_q16 = 0.5
        R.append(R[-1] + resid - nr)
        resid = nr
    assert R == [600_000, 800_000, 900_000, 950_000, 975_000]


def test_c5_blocks():
    cfg = CONFIGS["C5"]
    b = generate(cfg, 8, id_offset=(1 << 22) - 4)  # straddles the U=1 / U=2 block boundary
    N, H = cfg.n_tasks, cfg.horizon
    w = np.concatenate([b.mand_wcet[:, None], b.opt_wcet], 1).sum(1).reshape(-1, N).sum(1) / H
    assert (w[:4] < 1.15).all() and (w[4:] > 1.9).all()


def test_tiny_random_covers_edge_cases():
    rng = np.random.default_rng(0)
    b = gen.tiny_random(rng, 500)
    sizes = np.diff(b.task_begin)
    assert (sizes == 0).any() and (b.release > 0).any() and (b.deadline < 0).any()

"""Pins for oracle/tree.py, oracle/fmm.py, oracle/direct.py: brute force and identities."""
import math
import os

import numpy as np
import pytest

from workloads import CONFIGS, small_config, points_and_charges
from oracle.tree import build_level, neighbours, interaction_list, cheb
from oracle.plan import make_plan, Plan, LevelPlan, level_params
from oracle.fmm import OracleFMM
from oracle.direct import direct_sum
from oracle.resample import resample_half_batch

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def test_direct_two_particles():
    x = np.array([[0.0, 0, 0], [0.3, 0.4, 0.0]])
    q = np.array([1.0 + 0j, 1.0 + 0j])
    y = direct_sum(x, q, 7.0)
    assert np.allclose(y, np.exp(1j * 7.0 * 0.5) / 0.5, rtol=1e-15)


def test_direct_permutation_invariance():
    rng = np.random.default_rng(2)
    x = rng.uniform(size=(50, 3))
    q = rng.standard_normal(50) + 1j * rng.standard_normal(50)
    p = rng.permutation(50)
    y = direct_sum(x, q, 11.0)
    yp = direct_sum(x[p], q[p], 11.0)
    assert np.allclose(yp, y[p], rtol=1e-14)


def test_interaction_partition_exact():
    """Every ordered pair is near (leaf neighbours) or in exactly one M2L."""
    counts = dict(l.split() for l in open(os.path.join(GOLDEN, "counts.txt")) if not l.startswith("#"))
    rng = np.random.default_rng(8)
    x = rng.uniform(-1, 1, (300, 3))
    lo, a0, L = (-1.0, -1.0, -1.0), 2.0, 4
    levels = {l: build_level(x, lo, a0, l) for l in range(2, L + 1)}
    cover = np.zeros((300, 300), dtype=np.int64)
    for l in range(2, L + 1):
        lev = levels[l]
        for a, c in enumerate(lev.boxes):
            il = interaction_list(lev, c)
            assert len(il) <= int(counts["max_interaction_list"])
            for b, o in il:
                assert max(map(abs, o)) >= 2 and max(map(abs, o)) <= 3
                cover[np.ix_(lev.members[a], lev.members[b])] += 1
    lev = levels[L]
    for a, c in enumerate(lev.boxes):
        for b in neighbours(lev, c):
            cover[np.ix_(lev.members[a], lev.members[b])] += 1
    assert np.all(cover == 1)


def test_full_lattice_has_189():
    # a box deep inside a full lattice has exactly 189 interaction partners
    g = (np.arange(8) + 0.5) / 8 * 2 - 1
    X, Y, Z = np.meshgrid(g, g, g, indexing="ij")
    x = np.stack([X.ravel(), Y.ravel(), Z.ravel()], 1)
    lev = build_level(x, (-1, -1, -1), 2.0, 3)
    assert len(interaction_list(lev, (3, 4, 3))) == 189


def _plan_for(cfg):
    return make_plan(cfg.kappa, cfg.eps, cfg.size, cfg.depth, cfg.alpha)


def test_c1_policy_run_is_direct():
    cfg = CONFIGS["C1"]
    x, q = points_and_charges(cfg)
    plan = _plan_for(cfg)
    assert plan.L_f is None
    f = OracleFMM(x, cfg.lo, cfg.size, plan)
    t = np.arange(0, cfg.n, 97)
    assert np.allclose(f.matvec(q, t), direct_sum(x, q, cfg.kappa, t), rtol=1e-12)


@pytest.fixture(scope="module")
def small_case():
    cfg = small_config("small", n=400, kappa=32 * math.pi, depth=3, eps=1e-6, seed=21)
    x, q = points_and_charges(cfg)
    plan = _plan_for(cfg)
    return cfg, x, q, plan, OracleFMM(x, cfg.lo, cfg.size, plan)


def test_small_fmm_vs_direct(small_case):
    cfg, x, q, plan, f = small_case
    assert plan.L_f == 3                                      # two active levels: M2M/L2L exercised
    y = f.matvec(q)
    yd = direct_sum(x, q, cfg.kappa)
    assert np.linalg.norm(y - yd) / np.linalg.norm(yd) <= cfg.eps


def test_fmm_linearity(small_case):
    cfg, x, q, plan, f = small_case
    rng = np.random.default_rng(9)
    q2 = rng.standard_normal(len(q)) + 1j * rng.standard_normal(len(q))
    t = np.arange(0, len(q), 7)
    lhs = f.matvec(2.0 * q - 1j * q2, t)
    rhs = 2.0 * f.matvec(q, t) - 1j * f.matvec(q2, t)
    assert np.linalg.norm(lhs - rhs) / np.linalg.norm(rhs) < 1e-12


def test_m2m_translation_identity(small_case):
    """S2M at the parent centre == M2M(S2M at the children) (band-limited)."""
    cfg, x, q, plan, f = small_case
    M3 = f.s2m(q)
    M2 = f.m2m(M3, 3)
    lev2 = f.levels[2]
    S = f.grid(2)
    for p in list(M2)[:4]:
        idx = lev2.members[p]
        direct = np.exp(1j * cfg.kappa * (S @ (x[idx] - lev2.centers[p]).T)) @ q[idx]
        assert np.max(np.abs(M2[p] - direct)) < 1e-9 * np.max(np.abs(direct))


def test_single_source_at_centre():
    # S:520-style identity: a single charge at the leaf centre gives M == q on every direction
    cfg = small_config("one", n=400, kappa=32 * math.pi, depth=3, eps=1e-6, seed=21)
    x, q = points_and_charges(cfg)
    plan = _plan_for(cfg)
    f = OracleFMM(x, cfg.lo, cfg.size, plan)
    lev = f.levels[3]
    b = 0
    xs = x.copy()
    xs[lev.members[b][0]] = lev.centers[b]
    f2 = OracleFMM(xs, cfg.lo, cfg.size, plan)
    qq = np.zeros_like(q)
    qq[lev.members[b][0]] = 1.5 - 0.5j
    M = f2.s2m(qq, boxes=[b])[b]
    assert np.allclose(M, 1.5 - 0.5j, rtol=0, atol=1e-15)


def test_multilevel_corner_pair():
    """Sec. 4.2 / Fig. Error_Quad: two points at opposite box corners, M2L only at
    level 2 (a_2 = 1); adding translation levels (L = 2..5) leaves eps_I essentially unchanged."""
    kappa, eps, alpha = 30.0, 1e-6, 0.8
    a0 = 4.0
    # points at opposite corners of two level-2 boxes with offset (2, 0, 0): the pair is only
    # ever separated at level 2 (no M2L below, no near field at any leaf level)
    e = 1e-9
    x = np.array([[0.0 + e, 0.0 + e, 0.0 + e], [3.0 - e, 1.0 - e, 1.0 - e]]) - 2.0
    q = np.array([1.0 + 0j, 0.0 + 0j])
    exact = np.exp(1j * kappa * np.linalg.norm(x[0] - x[1])) / np.linalg.norm(x[0] - x[1])
    errs = {}
    for L in (2, 3, 4, 5):
        levels = {}
        for l in range(2, L + 1):
            ell, nth, nph, _ = level_params(kappa, a0 / 2 ** l, eps, alpha)
            levels[l] = LevelPlan(l, a0 / 2 ** l, ell, nth, nph, active=True)
        for l in range(L - 1, 1, -1):
            levels[l].n_theta = max(levels[l].n_theta, levels[l + 1].n_theta)
            levels[l].n_phi = max(levels[l].n_phi, levels[l + 1].n_phi)
        plan = Plan(kappa, eps, alpha, 1.0, a0, L, levels, L)
        f = OracleFMM(x, (-2.0, -2.0, -2.0), a0, plan)
        y_near, y_far = f.matvec(q, np.array([1]), parts=True)
        assert abs(y_near[0]) == 0.0
        errs[L] = y_far[0] - exact
    # corner pairs sit at |r| = sqrt3 a > alpha sqrt3 a, so eps_T itself exceeds eps;
    # what the paper checks is that the translation levels add nothing visible
    assert abs(errs[2]) < 1e-3
    for L in (3, 4, 5):
        assert abs(errs[L] - errs[2]) < 1e-12 / abs(x[0] - x[1]).max()


def test_subset_mode_equals_full_matvec():
    """Target-subset mode computes exactly the full matvec's y at the sampled
    targets: same passes restricted to the targets' ancestors (translation-only levels included)."""
    from workloads import small_config, points_and_charges
    from oracle.plan import make_plan
    from oracle.fmm import OracleFMM
    cfg = small_config("subset", n=1500, kappa=16 * math.pi, depth=4, eps=1e-6, seed=31)
    x, q = points_and_charges(cfg)
    plan = make_plan(cfg.kappa, cfg.eps, cfg.size, cfg.depth, cfg.alpha, source_level=4)
    assert plan.L_f == 2 and plan.source_level == 4
    f = OracleFMM(x, cfg.lo, cfg.size, plan)
    t = np.sort(np.random.default_rng(2).choice(cfg.n, 60, replace=False))
    y_full = f.matvec(q)
    y_sub = OracleFMM(x, cfg.lo, cfg.size, plan, workers=4).matvec_subset(q, t)
    assert np.max(np.abs(y_sub - y_full[t])) <= 1e-14 * np.max(np.abs(y_full))

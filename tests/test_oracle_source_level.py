"""Pins for the translation-only levels below L_f (reading R-14).

S2M/L2T at a source level D_s > L_f with M2M/L2L-only levels in between (added levels
"only add translation steps").  Pinned by:
  - the representation grid rule against scipy's Bessel J (independent of oracle.specfun);
  - the exact plane-wave identity: M_{L_f} obtained through the translation-only levels equals
    the direct S2M at L_f within the representation tail (eqn:PlaneWaveSpec);
  - the end-to-end matvec vs the direct sum (<= eps) and vs D_s = L_f (<= eps / 10);
  - the source-level policy against a brute-force box count.
"""
import math

import numpy as np
import pytest
from scipy.special import jv

from workloads import small_config, points_and_charges
from oracle.plan import make_plan, rep_grid, rep_tail, choose_source_level, REP_EPS_FACTOR, is_7smooth
from oracle.fmm import OracleFMM
from oracle.direct import direct_sum


def scipy_tail(z, N):
    n = np.arange(N // 2, N // 2 + 200)
    return 2.0 * float(np.sum(np.abs(jv(n, z))))


@pytest.mark.parametrize("kappa,a,eps", [(32 * math.pi, 2 / 2 ** 7, 1e-8), (128 * math.pi, 1 / 2 ** 6, 1e-6),
                                         (16 * math.pi, 2 / 2 ** 4, 1e-6), (5.0, 0.5, 1e-4)])
def test_rep_grid_is_smallest_passing(kappa, a, eps):
    z = kappa * math.sqrt(3) / 2 * a
    nth, nph = rep_grid(kappa, a, eps)
    thr = eps * REP_EPS_FACTOR
    assert nth % 2 == 0 and nph % 4 == 0 and is_7smooth(nth) and is_7smooth(nph)
    assert scipy_tail(z, nth) <= thr * (1 + 1e-9) and scipy_tail(z, nph) <= thr * (1 + 1e-9)
    assert abs(rep_tail(z, nth) - scipy_tail(z, nth)) <= 1e-12 * max(thr, 1e-300) + 1e-300
    prev_th = max([N for N in range(4, nth, 2) if is_7smooth(N)], default=None)
    prev_ph = max([N for N in range(4, nph, 4) if is_7smooth(N)], default=None)
    if prev_th:
        assert scipy_tail(z, prev_th) > thr
    if prev_ph:
        assert scipy_tail(z, prev_ph) > thr
    # the band covers the plane-wave argument (J_n decays only once n > z)
    assert nth // 2 - 1 >= z


def test_source_level_policy_brute_force():
    cfg = small_config("p", n=4000, kappa=16 * math.pi, depth=6, eps=1e-6, seed=3)
    x, _ = points_and_charges(cfg)
    lo, a0 = np.array(cfg.lo), cfg.size
    mean = {}
    for l in range(2, 7):
        keys = {tuple(np.minimum(np.floor((p - lo) / (a0 / 2 ** l)).astype(int), 2 ** l - 1)) for p in x}
        mean[l] = len(x) / len(keys)
    for L_f in (2, 3):
        want = max([l for l in range(L_f + 1, 7) if mean[l] >= 8.0], default=L_f)
        assert choose_source_level(x, cfg.lo, cfg.size, 6, L_f) == want
    assert choose_source_level(x, cfg.lo, cfg.size, 6, None) is None


@pytest.fixture(scope="module")
def deep_case():
    cfg = small_config("deep", n=3000, kappa=16 * math.pi, depth=5, eps=1e-6, seed=5)
    x, q = points_and_charges(cfg)
    p0 = make_plan(cfg.kappa, cfg.eps, cfg.size, cfg.depth, cfg.alpha)
    assert p0.L_f == 2 and p0.source_level == 2
    p1 = make_plan(cfg.kappa, cfg.eps, cfg.size, cfg.depth, cfg.alpha, source_level=4)
    return cfg, x, q, p0, p1


def test_translation_levels_reproduce_s2m(deep_case):
    """M_{L_f} through D_s -> L_f translations == direct S2M at L_f within the Jacobi-Anger tail."""
    cfg, x, q, p0, p1 = deep_case
    assert [p1.levels[l].rep for l in (2, 3, 4)] == [False, True, True]
    assert p1.levels[3].n_theta >= p1.levels[4].n_theta and p1.levels[2].n_theta >= p1.levels[3].n_theta
    f0, f1 = OracleFMM(x, cfg.lo, cfg.size, p0), OracleFMM(x, cfg.lo, cfg.size, p1)
    M0 = f0.s2m(q)
    M1, _, _ = f1.far_locals(q)
    scale = float(np.sum(np.abs(q)))
    err = max(float(np.max(np.abs(M1[2][b] - M0[b]))) for b in M0)
    assert err <= 4 * cfg.eps * REP_EPS_FACTOR * scale
    assert err >= 1e-16 * scale        # a genuinely different route (not the same computation)


def test_deep_matvec_vs_direct_and_lf(deep_case):
    cfg, x, q, p0, p1 = deep_case
    t = np.arange(0, len(x), 7)
    yd = direct_sum(x, q, cfg.kappa)[t]
    y0 = OracleFMM(x, cfg.lo, cfg.size, p0).matvec(q, t)
    y1 = OracleFMM(x, cfg.lo, cfg.size, p1).matvec(q, t)
    rel = lambda a, b: float(np.linalg.norm(a - b) / np.linalg.norm(b))
    assert rel(y1, yd) <= cfg.eps
    assert rel(y1, y0) <= cfg.eps / 10

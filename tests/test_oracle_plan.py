"""Pins for oracle/plan.py: the paper's error claims and an independent third-party derivation."""
import math

import numpy as np
import pytest

from oracle.plan import (level_params, choose_ell, collino_bound, is_7smooth, theta_spectrum_z,
                         M_index, make_plan)
from oracle.specfun import besselJ
from oracle.transfer import bmtf_table
from oracle.rig import pair_errors

# SURVEY.md §8a A-sizes / Appendix A1: (kappa a, eps) -> (ell, N_theta, N_phi) after
# 7-smooth rounding, derived by the surveyor with an independent scratch script
# (a third-party check; not paper values).
SURVEY_A1 = [
    (8 * math.pi, 1e-6, 57, 120, 120),
    (4 * math.pi, 1e-6, 44, 90, 96),
    (16 * math.pi, 1e-4, 88, 180, 180),
    (8 * math.pi, 1e-8, 66, 140, 140),
    (math.pi / 2, 1e-4, 26, 54, 56),
]


@pytest.mark.parametrize("ka,eps,ell,nth,nph", SURVEY_A1)
def test_plan_matches_independent_derivation(ka, eps, ell, nth, nph):
    got = level_params(ka, 1.0, eps, 0.8)
    assert got[0] == ell
    assert abs(got[1] - nth) <= 2 and abs(got[2] - nph) <= 4


def test_smooth_sizes():
    ell, nth, nph, ragged = level_params(16 * math.pi, 1.0, 1e-6, 0.8)
    assert nth % 2 == 0 and is_7smooth(nth) and nth >= 2 * ell
    assert nph % 4 == 0 and is_7smooth(nph)
    assert nph >= max(ragged)


def test_ell_is_smallest_passing():
    k, r, r0, eps = 40.0, 0.8 * math.sqrt(3), 2.0, 1e-7
    ell = choose_ell(k, r, r0, eps)
    assert collino_bound(ell, k, r, r0) < eps <= collino_bound(ell - 1, k, r, r0)


@pytest.mark.parametrize("kappa,eps", [(10.0, 1e-4), (30.0, 1e-8), (25.0, 1e-6)])
@pytest.mark.parametrize("axis", ["z", "x"])
def test_single_level_error_within_factor_two(kappa, eps, axis):
    """Figs. Error_R0Z / Error_R0X: a = 1, alpha = 0.8, |r| = 0.8 sqrt3,
    |r0| = 2; max over directions of |eps_T| is within a factor 2 of the target."""
    a, alpha = 1.0, 0.8
    ell, nth, nph, _ = level_params(kappa, a, eps, alpha)
    r0 = np.array([0, 0, 2.0]) if axis == "z" else np.array([2.0, 0, 0])
    T = bmtf_table(ell, kappa, r0, nth, nph)
    rng = np.random.default_rng(5)
    rn = alpha * a * math.sqrt(3)
    dirs = [np.array([0, 0, 1.0]), np.array([0, 0, -1.0]), np.array([1.0, 0, 0]), np.array([-1.0, 0, 0]),
            np.array([0, 1.0, 0])]
    v = rng.standard_normal((60, 3))
    dirs += list(v / np.linalg.norm(v, axis=1, keepdims=True))
    eT = [abs(pair_errors(kappa, rn * d, r0, ell, nth, nph, table=T)[0]) for d in dirs]
    assert max(eT) <= 2.0 * eps
    assert max(eT) >= eps / 100.0         # sharp: not a gross over-estimate


def test_alg2_bound_dominates_measured_integration_error():
    # eqn:EpsITheta: predicted bound >= |eps_I| for r, r0 along z at the chosen N_theta
    kappa, eps = 20.0, 1e-6
    ell, nth, nph, _ = level_params(kappa, 1.0, eps, 0.8)
    r0 = np.array([0, 0, 2.0])
    rn = 0.8 * math.sqrt(3)
    freqs, Tt = theta_spectrum_z(ell, kappa, 2.0, 4 * ell + 64)
    E = np.abs(besselJ(2 * (4 * ell + 64), kappa * rn))
    for N in (nth - 10, nth - 4, nth):
        bound = 4 * math.pi ** 2 * float(np.sum(Tt * E[M_index(N, freqs)]))
        T = bmtf_table(ell, kappa, r0, N, 2 * ell + 4)
        for s in (+1, -1):
            eI = abs(pair_errors(kappa, np.array([0, 0, s * rn]), r0, ell, N, 2 * ell + 4, table=T)[2])
            assert eI <= bound * 1.0001 + 1e-15


def test_quadrature_size_ratio():
    # Fig. QuadSize: ragged K / 2(ell+1)^2 approaches 2/pi ~ 0.64; in [0.6, 0.8]
    for ka in (16 * math.pi, 32 * math.pi):
        ell, nth, nph, ragged = level_params(ka, 1.0, 1e-4, 0.8)
        ratio = sum(ragged) / (2 * (ell + 1) ** 2)
        assert 0.6 <= ratio <= 0.8


def test_breakdown_levels_are_inadmissible():
    # low-frequency breakdown; F_l grows as kappa a shrinks.  C1 (kappa = 2 pi, a0 = 2)
    plan = make_plan(2 * math.pi, 1e-4, 2.0, 3)
    assert plan.L_f is None
    assert plan.levels[2].F > 1e-3                 # lambda/2 boxes

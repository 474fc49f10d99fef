"""Pins for the two oracle rules that decide L_f: F_l (oracle/plan.py level_F, R-9) and
the per-level design radius alpha (oracle/plan.py make_plan, R-13).

Each pin is something other than the oracle's own formula:
  (1) SURVEY.md Appendix A1 / P-20: the surveyor's independent derivation of F at (kappa a, eps)
      (third-party values, unrounded grids, 5 offsets) -- ours within [0.45, 2.5] of each value;
      the spread of the nine ratios (0.58 ... 2.15) means a factor-2 slip (4 pi for 8 pi, or
      16 pi) fails at least one case.
  (2) The low-frequency breakdown claim of P:833 measured directly: on the single-pair rig
      (eqn:eps_I) with a generous quadrature (N = 2 ell + 24, so the integration error
      of the bound is far below rounding), the relative error of the FP64 quadrature sum against
      the Gegenbauer partial sum is pure roundoff; its maximum over 20 random pairs must sit within
      [0.5, 3] x F (SURVEY App. A2 measured 1.0-2.3 x F).  Boxes with a != 1 (real config levels),
      so a dropped a_l factor (x4 or x8) fails, and so does a factor-2 slip.
  (3) R-13 on the BASELINE configs: at the alpha the plan selects for each active level, the
      paper's claim eps_T <= 2 eps (Figs. Error_R0Z / Error_R0X) holds for the
      worst case r = +-|r| r0hat along z and x; and every larger alpha candidate has F > tau
      (the choice is the largest admissible one, not the first in some other order).
"""
import math

import numpy as np
import pytest

from oracle.plan import (level_params, level_F, make_plan, default_tau)
from oracle.transfer import bmtf_table
from oracle.rig import pair_errors, kernel

# SURVEY.md Appendix A1 (a = 1, alpha = 0.8): (kappa a, eps, F)
SURVEY_A1_F = [
    (math.pi, 1e-4, 1.8e-2),
    (2 * math.pi, 1e-4, 1.6e-8),
    (2 * math.pi, 1e-6, 8.8),
    (4 * math.pi, 1e-4, 1.5e-13),
    (4 * math.pi, 1e-6, 1.7e-8),
    (4 * math.pi, 1e-8, 1.8e-2),
    (8 * math.pi, 1e-6, 9.9e-14),
    (8 * math.pi, 1e-8, 3.3e-11),
    (16 * math.pi, 1e-6, 1.6e-14),
]


def test_level_F_matches_survey_A1():
    ratios = []
    for ka, eps, F_ref in SURVEY_A1_F:
        ell, nth, nph, _ = level_params(ka, 1.0, eps, 0.8)
        ratios.append(level_F(ka, 1.0, ell, nth, nph) / F_ref)
    ratios = np.array(ratios)
    assert np.all(ratios >= 0.45) and np.all(ratios <= 2.5), ratios


# (kappa, a, ell): C3 level 4 (kappa a = 2 pi, ell = 40 and 28), C4 level 3 (8 pi, ell 66),
# C5-like (4 pi at a = 1/2, ell 57), C1 level 3 (pi at a = 1/4, ell 26)
RIG_CASES = [(16 * math.pi, 1 / 8, 40), (32 * math.pi, 1 / 4, 66), (16 * math.pi, 1 / 8, 28),
             (8 * math.pi, 1 / 2, 57), (4 * math.pi, 1 / 4, 26)]


@pytest.mark.parametrize("kappa,a,ell", RIG_CASES)
def test_single_pair_roundoff_tracks_F(kappa, a, ell):
    N = 2 * ell + 24
    N += (-N) % 4
    r0 = np.array([2 * a, 0.0, 0.0])                     # offset (2, 0, 0) in box units
    T = bmtf_table(ell, kappa, r0, N, N)
    F = level_F(kappa, a, ell, N, N)          # the oracle's F (max over the 34 canonical offsets)
    rng = np.random.default_rng(11)
    worst = 0.0
    for _ in range(20):
        # target and source uniform in their boxes: r = (x_t - c_t) - (x_s - c_s)
        r = rng.uniform(-a / 2, a / 2, 3) - rng.uniform(-a / 2, a / 2, 3)
        eI = pair_errors(kappa, r, r0, ell, N, N, table=T)[2]
        worst = max(worst, abs(eI) / abs(kernel(kappa, float(np.linalg.norm(r + r0)))))
    assert 0.5 <= worst / F <= 3.0, (worst, F)


@pytest.mark.parametrize("name,kappa,eps,a0,depth", [
    ("C3", 16 * math.pi, 1e-6, 2.0, 6),
    ("C4", 32 * math.pi, 1e-8, 2.0, 7),
    ("C5", 128 * math.pi, 1e-6, 1.0, 8),
])
def test_r13_alpha_selection(name, kappa, eps, a0, depth):
    plan = make_plan(kappa, eps, a0, depth)
    tau = default_tau(eps)
    assert plan.L_f is not None
    for l in range(2, plan.L_f + 1):
        lp = plan.levels[l]
        a = lp.a
        eps_l = eps / a                                     # R-1
        rn = lp.alpha * a * math.sqrt(3)
        for axis in (2, 0):
            r0 = np.zeros(3)
            r0[axis] = 2 * a
            T = bmtf_table(lp.ell, kappa, r0, lp.n_theta, lp.n_phi)
            worst = 0.0
            for s in (1.0, -1.0):
                r = np.zeros(3)
                r[axis] = s * rn
                worst = max(worst, abs(pair_errors(kappa, r, r0, lp.ell, lp.n_theta, lp.n_phi, table=T)[0]))
            assert worst <= 2.0 * eps_l, (name, l, axis, worst / eps_l)
            assert worst >= eps_l / 100.0, (name, l, axis, worst / eps_l)   # sharp, not vacuous
        assert lp.F <= tau
        for al in (1.0, 0.9):
            if al > lp.alpha + 1e-12:
                ell, nth, nph, _ = level_params(kappa, a, eps, al)
                assert level_F(kappa, a, ell, nth, nph) > tau, (name, l, al)

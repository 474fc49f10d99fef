"""Pins for the ragged quadrature (reading R-15; Alg. 3 per row).

  - the per-row rule against Alg. 3's own bound (each row passes, the previous candidate fails);
  - structure: mirror rows, <= rectangular N_phi, QuadSize ratio vs rectangular;
  - the ragged 5-step resample: identity, exact on band-limited fields, equal to the rectangular
    resample when the rows are all equal;
  - end to end: the ragged FMM vs the direct sum (<= eps) and vs the rectangular FMM (<= eps/10).
"""
import math

import numpy as np
import pytest

from workloads import small_config, points_and_charges
from oracle.plan import make_plan, nphi_row_bounds, is_7smooth
from oracle.fmm import OracleFMM
from oracle.direct import direct_sum
from oracle.resample import resample_ragged, resample_half, ragged_to_rows, rows_to_ragged
from oracle.transfer import shat


@pytest.fixture(scope="module")
def plans():
    cfg = small_config("rag", n=500, kappa=32 * math.pi, depth=3, eps=1e-6, seed=13)
    p0 = make_plan(cfg.kappa, cfg.eps, cfg.size, cfg.depth, cfg.alpha)
    p1 = make_plan(cfg.kappa, cfg.eps, cfg.size, cfg.depth, cfg.alpha, ragged=True)
    return cfg, p0, p1


def test_ragged_rows_rule(plans):
    cfg, p0, p1 = plans
    for l in (2, 3):
        lp = p1.levels[l]
        assert p0.levels[l].rows is None and lp.rows is not None
        assert (lp.n_theta, lp.n_phi) == (p0.levels[l].n_theta, p0.levels[l].n_phi)
        rows = lp.rows
        nth = lp.n_theta
        assert len(rows) == nth and all(rows[n] == rows[(nth - n) % nth] for n in range(nth))
        assert all(r % 4 == 0 and is_7smooth(r) and r <= lp.n_phi for r in rows)
        eps_l = cfg.eps / lp.a
        thr = eps_l / (4 * math.pi ** 2)
        cands = [N for N in range(4, lp.n_phi + 1, 4) if is_7smooth(N)]
        B = nphi_row_bounds(lp.ell, cfg.kappa, lp.alpha * math.sqrt(3) * lp.a, 2 * lp.a, nth, cands)
        for n in range(nth // 2 + 1):
            c = cands.index(rows[n])
            assert B[n, c] < thr or rows[n] == lp.n_phi
            assert all(B[n, j] >= thr for j in range(c))
        ratio = lp.K / (nth * lp.n_phi // 2)
        assert 0.55 < ratio < 0.85, ratio                     # Fig. QuadSize: ragged / rectangular


def _plane_wave_half(rows, nth, d, kappa):
    th = np.concatenate([np.full(r // 2, 2 * math.pi * n / nth) for n, r in enumerate(rows)])
    ph = np.concatenate([2 * math.pi * np.arange(r // 2) / r for r in rows])
    return np.exp(1j * kappa * shat(th, ph) @ d)


def test_ragged_resample_identities(plans):
    cfg, p0, p1 = plans
    rng = np.random.default_rng(0)
    lp = p1.levels[3]
    F = rng.standard_normal(lp.K) + 1j * rng.standard_normal(lp.K)
    # round trip of the row representation
    assert np.array_equal(rows_to_ragged(ragged_to_rows(F, lp.rows), lp.n_theta), F)
    # a band-limited field (plane wave of small argument) is reproduced on another quadrature
    d = np.array([0.011, -0.007, 0.005])
    up = p1.levels[2]
    Fc = _plane_wave_half(lp.rows, lp.n_theta, d, cfg.kappa)
    Fp = resample_ragged(Fc, lp.rows, up.n_theta, up.rows)
    assert np.max(np.abs(Fp - _plane_wave_half(up.rows, up.n_theta, d, cfg.kappa))) < 1e-12
    # all rows equal -> the rectangular 5-step resample
    nth, nph = 24, 28
    G = rng.standard_normal(nth * nph // 2) + 1j * rng.standard_normal(nth * nph // 2)
    a = resample_ragged(G, [nph] * nth, 36, [40] * 36)
    b = resample_half(G.reshape(nth, nph // 2), nph, 36, 40).reshape(-1)
    assert np.allclose(a, b, rtol=0, atol=1e-13)


def test_ragged_fmm_vs_direct_and_rect(plans):
    cfg, p0, p1 = plans
    x, q = points_and_charges(cfg)
    t = np.arange(0, cfg.n, 3)
    yd = direct_sum(x, q, cfg.kappa)[t]
    y0 = OracleFMM(x, cfg.lo, cfg.size, p0).matvec(q, t)
    y1 = OracleFMM(x, cfg.lo, cfg.size, p1).matvec(q, t)
    rel = lambda a, b: float(np.linalg.norm(a - b) / np.linalg.norm(b))
    assert rel(y1, yd) <= cfg.eps
    assert rel(y1, y0) <= cfg.eps / 10
    assert rel(y1, y0) > 1e-15                    # genuinely a different quadrature

"""Pins for oracle/resample.py: exactness, adjointness, Fig. InterpolateDataProfile bookkeeping."""
import math
import os

import numpy as np
import pytest

from oracle.resample import (resample_matrix, resample_half, resample_half_batch, resample_rows,
                             half_to_rows)
from oracle.transfer import shat

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def sphere_poly(nth, nph, coeffs):
    """A band-limited function of s (polynomial in s_x, s_y, s_z) on the half grid."""
    th = 2 * math.pi * np.arange(nth) / nth
    ph = 2 * math.pi * np.arange(nph // 2) / nph
    TH, PH = np.meshgrid(th, ph, indexing="ij")
    s = shat(TH, PH)
    f = np.zeros(TH.shape, dtype=complex)
    for (i, j, k), c in coeffs.items():
        f += c * s[..., 0] ** i * s[..., 1] ** j * s[..., 2] ** k
    return f


COEFFS = {(3, 0, 0): 1.0, (1, 2, 1): 0.5 - 0.2j, (0, 0, 4): -0.3j, (2, 1, 2): 0.7, (0, 0, 0): 0.1}


def test_identity_at_equal_size():
    R = resample_matrix(24, 24)
    f = np.random.default_rng(0).standard_normal(24)
    # the Nyquist mode is dropped (R-6), everything else is preserved
    F = np.fft.fft(f)
    F[12] = 0
    assert np.allclose(R @ f, np.fft.ifft(F), atol=1e-14)


@pytest.mark.parametrize("src,dst", [((12, 12), (20, 24)), ((20, 24), (12, 12)), ((16, 20), (30, 28))])
def test_exact_on_bandlimited(src, dst):
    # degree-5 polynomial in s: theta and phi bandwidth 5 <= min(N)/2 - 1
    f = sphere_poly(src[0], src[1], COEFFS)
    g = resample_half(f, src[1], dst[0], dst[1])
    assert np.max(np.abs(g - sphere_poly(dst[0], dst[1], COEFFS))) < 1e-13


def test_batch_equals_rows_version():
    rng = np.random.default_rng(3)
    F = rng.standard_normal((3, 18, 10)) + 1j * rng.standard_normal((3, 18, 10))
    for dst in ((30, 28), (12, 8), (18, 20)):
        got = resample_half_batch(F, 20, *dst)
        for b in range(3):
            assert np.max(np.abs(got[b] - resample_half(F[b], 20, *dst))) < 1e-13


def test_roundtrip_up_then_down():
    rng = np.random.default_rng(4)
    F = rng.standard_normal((1, 14, 8)) + 1j * rng.standard_normal((1, 14, 8))
    # first project onto the representable band, then up and down is the identity
    P = resample_half_batch(F, 16, 14, 16)
    U = resample_half_batch(P, 16, 30, 36)
    D = resample_half_batch(U, 36, 14, 16)
    assert np.max(np.abs(D - P)) < 1e-13


def test_adjointness():
    # <R f, g>_fine == <f, R* g>_coarse with quadrature weights 1/(N_t N_p)
    rng = np.random.default_rng(5)
    c, fn = (14, 16), (24, 28)
    f = rng.standard_normal((1, *[c[0], c[1] // 2])) + 1j * rng.standard_normal((1, c[0], c[1] // 2))
    g = rng.standard_normal((1, fn[0], fn[1] // 2)) + 1j * rng.standard_normal((1, fn[0], fn[1] // 2))
    f = resample_half_batch(f, c[1], *c)
    g = resample_half_batch(g, fn[1], *fn)
    up = resample_half_batch(f, c[1], *fn)
    down = resample_half_batch(g, fn[1], *c)
    lhs = np.vdot(g, up) / (fn[0] * fn[1])
    rhs = np.vdot(down, f) / (c[0] * c[1])
    assert abs(lhs - rhs) < 1e-13 * abs(lhs)


def test_anterpolation_contracts():
    rng = np.random.default_rng(6)
    g = rng.standard_normal((1, 30, 14)) + 1j * rng.standard_normal((1, 30, 14))
    d = resample_half_batch(g, 28, 18, 20)
    assert np.sum(np.abs(d) ** 2) / (18 * 20) <= np.sum(np.abs(g) ** 2) / (30 * 28) + 1e-12


def test_interpolate_data_profile_golden():
    # Fig. InterpolateDataProfile: N_theta 30 -> 24, calN_phi = 16, ragged rows
    vals = dict(l.split() for l in open(os.path.join(GOLDEN, "interp_profile.txt")) if not l.startswith("#"))
    nth, nthp, calN = int(vals["ntheta_in"]), int(vals["ntheta_out"]), int(vals["calN_phi"])
    rng = np.random.default_rng(7)
    # ragged input rows (pole rows short), row n = 0..15
    lens = [4, 8, 8, 12, 12, 16, 16, 16, 16, 16, 16, 12, 12, 8, 8, 4]
    rows = [rng.standard_normal(L) + 0j for L in lens]
    out_lens = [4, 4, 8, 8, 12, 16, 16, 16, 12, 8, 8, 4, 4]
    trace = []
    out = resample_rows(rows, nth, nthp, out_lens, trace=trace)
    steps = dict(trace)
    assert len(steps["input"]) == int(vals["rows_in"])
    assert steps["I_phi"] == [calN] * int(vals["rows_in"])
    assert steps["W"] == (int(vals["cols"]), nth)
    assert steps["A_theta"] == (int(vals["cols"]), nthp)
    assert steps["W2"] == [calN] * int(vals["rows_out"])
    assert steps["A_phi"] == out_lens and len(out) == int(vals["rows_out"])


# ---- NEXT 4: coefficient-domain symmetric resampling (eqn:FourierSphereSym P:277-280) ----
def full_doubled_grid(nth, nph, coeffs):
    """f(theta_n, phi_m) on the whole doubled grid n < N_theta, m < N_phi (no half storage)."""
    th = 2 * math.pi * np.arange(nth) / nth
    ph = 2 * math.pi * np.arange(nph) / nph
    TH, PH = np.meshgrid(th, ph, indexing="ij")
    s = shat(TH, PH)
    f = np.zeros(TH.shape, dtype=complex)
    for (i, j, k), c in coeffs.items():
        f += c * s[..., 0] ** i * s[..., 1] ** j * s[..., 2] ** k
    return f


@pytest.mark.parametrize("nth,nph", [(16, 16), (14, 20), (24, 12)])
def test_fourier_sphere_symmetry_holds(nth, nph):
    """eqn:FourierSphereSym: the 2-D Fourier coefficients of a function of s sampled on
    the doubled sphere satisfy f~_{n,m} = (-1)^m f~_{-n,m} (to rounding), for every (n, m)."""
    f = full_doubled_grid(nth, nph, COEFFS)
    Ft = np.fft.fft2(f) / (nth * nph)                        # f~[n, m], n mod N_theta, m mod N_phi
    n = np.arange(nth)[:, None]
    m = np.arange(nph)[None, :]
    msigned = np.where(m <= nph // 2, m, m - nph)
    lhs = Ft
    rhs = ((-1.0) ** np.abs(msigned)) * Ft[(-n) % nth, m]
    assert np.max(np.abs(lhs - rhs)) < 1e-14 * np.max(np.abs(Ft)) * 10
    # and it is not vacuous: both parities carry weight
    assert np.max(np.abs(Ft[:, 1::2])) > 1e-3 and np.max(np.abs(Ft[:, 0::2])) > 1e-3


@pytest.mark.parametrize("src,dst", [((16, 16), (32, 32)), ((32, 32), (16, 16)), ((24, 24), (32, 32)),
                                     ((32, 32), (42, 48)), ((42, 48), (60, 60)), ((60, 60), (42, 48)),
                                     ((54, 56), (40, 40)), ((18, 20), (30, 28))])
def test_coeff_sym_equals_five_step(src, dst):
    """NEXT 4 is the same operator as the 5-step procedure: random data."""
    from oracle.resample import resample_coeff_sym
    rng = np.random.default_rng(src[0] + 100 * dst[0])
    F = rng.standard_normal((3, src[0], src[1] // 2)) + 1j * rng.standard_normal((3, src[0], src[1] // 2))
    a = resample_coeff_sym(F, src[1], dst[0], dst[1])
    b = resample_half_batch(F, src[1], dst[0], dst[1])
    assert np.max(np.abs(a - b)) <= 1e-13 * np.max(np.abs(b))


def test_coeff_sym_exact_on_bandlimited():
    from oracle.resample import resample_coeff_sym
    f = sphere_poly(12, 12, COEFFS)
    g = resample_coeff_sym(f[None], 12, 20, 24)[0]
    assert np.max(np.abs(g - sphere_poly(20, 24, COEFFS))) < 1e-13

"""Pins for oracle/specfun.py against closed forms and independent library routines."""
import math

import numpy as np
import pytest
import scipy.special as sp

from oracle.specfun import sph_jn, sph_yn, sph_hn, besselJ, legendre_all, legendre_series

XS = [0.01, 0.7, 3.0, 17.5, 60.0, 150.0]


@pytest.mark.parametrize("x", XS)
def test_sph_jn_vs_scipy(x):
    n = np.arange(200)
    ref = sp.spherical_jn(n, x)
    got = sph_jn(199, x)
    m = np.abs(ref) > 1e-280
    assert np.max(np.abs(got[m] - ref[m]) / np.abs(ref[m])) < 1e-11


@pytest.mark.parametrize("x", XS)
def test_sph_yn_vs_scipy(x):
    n = np.arange(120)
    ref = sp.spherical_yn(n, x)
    got = sph_yn(119, x)
    m = np.isfinite(ref) & np.isfinite(got)
    assert np.max(np.abs(got[m] - ref[m]) / np.abs(ref[m])) < 1e-12


@pytest.mark.parametrize("x", XS[1:])
def test_besselJ_vs_scipy(x):
    n = np.arange(300)
    ref = sp.jv(n, x)
    got = besselJ(299, x)
    assert np.max(np.abs(got - ref)) < 1e-13 * max(1.0, x)
    m = np.abs(ref) > 1e-250
    big = n > x + 5               # tail (what Algs 2-3 need) to high relative accuracy
    assert np.max(np.abs(got[m & big] - ref[m & big]) / np.abs(ref[m & big])) < 1e-11


def test_hankel_closed_forms():
    for x in (0.3, 2.0, 40.0):
        h = sph_hn(1, x)
        e = np.exp(1j * x)
        assert abs(h[0] - (-1j * e / x)) < 1e-15 * abs(h[0])
        assert abs(h[1] - (-e * (x + 1j) / x ** 2)) < 1e-14 * abs(h[1])
        j = sph_jn(0, x)
        assert abs(j[0] - math.sin(x) / x) < 1e-15


def test_wronskian():
    # j_n y_{n-1} - j_{n-1} y_n = 1/x^2
    for x in (0.5, 5.0, 50.0):
        j = sph_jn(60, x)
        y = sph_yn(60, x)
        n = np.arange(1, 40)
        w = j[n] * y[n - 1] - j[n - 1] * y[n]
        assert np.max(np.abs(w * x * x - 1.0)) < 1e-10


def test_jacobi_anger_resummation():
    # eqn:PlaneWaveSpec: e^{i z cos phi} = sum_n i^n J_n(z) e^{i n phi}
    z = 23.7
    J = besselJ(120, z)
    for phi in (0.0, 0.4, 2.1, math.pi):
        n = np.arange(1, 121)
        s = J[0] + np.sum((1j ** n) * J[1:] * (np.exp(1j * n * phi) + np.exp(-1j * n * phi)))
        assert abs(s - np.exp(1j * z * math.cos(phi))) < 1e-12


def test_legendre():
    t = np.linspace(-1, 1, 101)
    P = legendre_all(50, t)
    for n in (0, 1, 2, 7, 31, 50):
        assert np.max(np.abs(P[n] - sp.eval_legendre(n, t))) < 1e-12
    c = np.random.default_rng(0).standard_normal(30) + 0j
    ref = sum(c[n] * sp.eval_legendre(n, t) for n in range(30))
    assert np.max(np.abs(legendre_series(c, t) - ref)) < 1e-12

"""Special functions for the oracle (TEST INFRASTRUCTURE; see oracle/__init__.py).

Notation table: j_n, y_n spherical Bessel of the 1st/2nd kind,
h_n^(1) = j_n + i y_n, P_n Legendre.  J_n (cylindrical Bessel) enters through
the Jacobi-Anger plane-wave spectrum eqn:PlaneWaveSpec.

Algorithms (textbook):
  j_n : Miller downward recurrence j_{n-1} = (2n+1)/x j_n - j_{n+1},
        normalised with sum_n (2n+1) j_n^2 = 1, sign fixed by j_0 or j_1.
  y_n : upward recurrence y_{n+1} = (2n+1)/x y_n - y_{n-1} (stable upward).
  J_n : Miller downward recurrence J_{n-1} = 2n/x J_n - J_{n+1},
        normalised with J_0 + 2 sum_k J_{2k} = 1.
  P_n : three-term recurrence (n+1)P_{n+1} = (2n+1) t P_n - n P_{n-1}.
Pinned by tests/test_oracle_specfun.py against scipy.special / mpmath and the
closed forms j_0 = sin x / x, h_0 = -i e^{ix}/x, h_1 = -e^{ix}(x+i)/x^2.
"""
from __future__ import annotations

import math

import numpy as np


def _miller_start(nmax: int, x: float) -> int:
    return int(max(nmax, x) + 30 + 2.0 * math.sqrt(40.0 * max(nmax, x, 1.0)))


def sph_jn(nmax: int, x: float) -> np.ndarray:
    """j_0..j_nmax at scalar x > 0 (Miller downward recurrence)."""
    assert x > 0.0
    top = _miller_start(nmax, x)
    f = np.zeros(top + 2)
    f[top + 1] = 0.0
    f[top] = 1.0
    for n in range(top, 0, -1):
        f[n - 1] = (2 * n + 1) / x * f[n] - f[n + 1]
        if abs(f[n - 1]) > 1e120:           # rescale to avoid overflow
            f[n - 1:] *= 1e-120
    norm = math.sqrt(float(np.sum((2 * np.arange(top + 2) + 1) * f * f)))
    f /= norm
    j0 = math.sin(x) / x
    j1 = math.sin(x) / (x * x) - math.cos(x) / x
    ref, got = (j0, f[0]) if abs(j0) > abs(j1) else (j1, f[1])
    if (ref < 0) != (got < 0):
        f = -f
    return f[: nmax + 1].copy()


def sph_yn(nmax: int, x: float) -> np.ndarray:
    """y_0..y_nmax at scalar x > 0 (upward recurrence, may overflow to -inf)."""
    assert x > 0.0
    y = np.zeros(nmax + 1)
    y[0] = -math.cos(x) / x
    if nmax >= 1:
        y[1] = -math.cos(x) / (x * x) - math.sin(x) / x
    with np.errstate(over="ignore", invalid="ignore"):
        for n in range(1, nmax):
            y[n + 1] = (2 * n + 1) / x * y[n] - y[n - 1]
    return y


def sph_hn(nmax: int, x: float) -> np.ndarray:
    """Spherical Hankel h_n^(1)(x) = j_n(x) + i y_n(x), n = 0..nmax."""
    return sph_jn(nmax, x) + 1j * sph_yn(nmax, x)


def besselJ(nmax: int, x: float) -> np.ndarray:
    """Cylindrical Bessel J_0..J_nmax at scalar x >= 0 (Miller)."""
    out = np.zeros(nmax + 1)
    if x == 0.0:
        out[0] = 1.0
        return out
    top = _miller_start(nmax, x)
    if top % 2:
        top += 1
    f = np.zeros(top + 2)
    f[top] = 1.0
    for n in range(top, 0, -1):
        f[n - 1] = 2.0 * n / x * f[n] - f[n + 1]
        if abs(f[n - 1]) > 1e120:
            f[n - 1:] *= 1e-120
    norm = f[0] + 2.0 * np.sum(f[2:top + 1:2])
    f /= norm
    out[:] = f[: nmax + 1]
    return out


def legendre_all(nmax: int, t: np.ndarray) -> np.ndarray:
    """P_0..P_nmax at points t (array), shape (nmax+1,) + t.shape."""
    t = np.asarray(t, dtype=np.float64)
    P = np.empty((nmax + 1,) + t.shape)
    P[0] = 1.0
    if nmax >= 1:
        P[1] = t
    for n in range(1, nmax):
        P[n + 1] = ((2 * n + 1) * t * P[n] - n * P[n - 1]) / (n + 1)
    return P


def legendre_series(coef: np.ndarray, t: np.ndarray) -> np.ndarray:
    """sum_n coef[n] P_n(t) by the three-term recurrence (complex coef)."""
    t = np.asarray(t, dtype=np.float64)
    p_prev = np.ones_like(t)
    acc = coef[0] * p_prev
    if len(coef) == 1:
        return acc
    p = t.copy()
    acc = acc + coef[1] * p
    for n in range(1, len(coef) - 1):
        p_next = ((2 * n + 1) * t * p - n * p_prev) / (n + 1)
        p_prev, p = p, p_next
        acc = acc + coef[n + 1] * p
    return acc

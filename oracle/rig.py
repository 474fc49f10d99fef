"""Single-pair error rig (TEST INFRASTRUCTURE; see oracle/__init__.py).

eqn:eps_T  eps_T = e^{i k |r + r0|}/|r + r0| - sum_n (4 pi^2 / (N_theta N_phi)) sum_m E_r T^{s,L}_{r0}
eqn:eps_G  eps_G = e^{i k |r + r0|}/|r + r0| - i k sum_{n<=l} (-1)^n (2n+1) h_n(k|r0|) j_n(k|r|) P_n(rhat.r0hat)
eqn:eps_I  eps_I = eps_T - eps_G
Rectangular quadrature on the stored half grid (weight 8 pi^2 / (N_theta N_phi)).
"""
from __future__ import annotations

import math

import numpy as np

from .specfun import sph_hn, sph_jn, legendre_series
from .transfer import shat, bmtf_table


def kernel(kappa: float, R: float) -> complex:
    return complex(np.exp(1j * kappa * R) / R)


def gegenbauer_partial(kappa: float, r, r0, ell: int) -> complex:
    """eqn:Gegenbauer truncated at ell."""
    r = np.asarray(r, dtype=np.float64)
    r0 = np.asarray(r0, dtype=np.float64)
    rn, r0n = float(np.linalg.norm(r)), float(np.linalg.norm(r0))
    h = sph_hn(ell, kappa * r0n)
    j = sph_jn(ell, kappa * rn)
    n = np.arange(ell + 1)
    c = 1j * kappa * ((-1.0) ** n) * (2 * n + 1) * h * j
    t = float(np.clip(r @ r0 / (rn * r0n), -1, 1))
    return complex(legendre_series(c, np.array(t)))


def quadrature_sum(kappa: float, r, table: np.ndarray, n_theta: int, n_phi: int) -> complex:
    """(8 pi^2 / (N_theta N_phi)) sum_{stored} e^{i kappa s.r} T^{s,LL}(s) (eqn:EpsI)."""
    th = 2 * math.pi * np.arange(n_theta) / n_theta
    ph = 2 * math.pi * np.arange(n_phi // 2) / n_phi
    TH, PH = np.meshgrid(th, ph, indexing="ij")
    S = shat(TH, PH)
    E = np.exp(1j * kappa * (S @ np.asarray(r, dtype=np.float64)))
    return complex(8 * math.pi ** 2 / (n_theta * n_phi) * np.sum(E * table))


def pair_errors(kappa: float, r, r0, ell: int, n_theta: int, n_phi: int, table=None):
    """(eps_T, eps_G, eps_I) for one (r, r0)."""
    r = np.asarray(r, dtype=np.float64)
    r0 = np.asarray(r0, dtype=np.float64)
    if table is None:
        table = bmtf_table(ell, kappa, r0, n_theta, n_phi)
    exact = kernel(kappa, float(np.linalg.norm(r + r0)))
    eT = exact - quadrature_sum(kappa, r, table, n_theta, n_phi)
    eG = exact - gegenbauer_partial(kappa, r, r0, ell)
    return eT, eG, eT - eG

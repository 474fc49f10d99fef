"""Transfer function and Alg. 1 bandlimited modified transfer function (TEST INFRASTRUCTURE).

P:108-112  eqn:TransferFn
    T_{l,r0}(s) = (i kappa / 4 pi) sum_{n=0}^{l} i^n (2n+1) h_n(kappa |r0|) P_n(s . r0hat)
P:250-256  T^s = 1/2 T |sin theta|,  s = (cos phi sin theta, sin phi sin theta, cos theta)
P:386-393  F_n[|sin theta|] = ((-1)^n + 1) / (pi (1 - n^2))
P:508-530  Alg. 1: keep theta-frequencies |n| <= N_theta/2 - 1 of T^s, computed exactly
           by convolving the (2l+1)-point spectrum of T with the spectrum of |sin|.
P:651-660  T^{s,LL}: additionally truncate phi-frequencies to |m| <= N_phi/2 - 1.
P:532      equivalent real-space route (interpolate, multiply by bandlimited |sin|,
           anterpolate) -- implemented separately as a pin.

Grid convention: theta_p = 2 pi p / N_theta (0 <= p < N_theta),
phi_q = 2 pi q / N_phi; half storage keeps q < N_phi/2.
"""
from __future__ import annotations

import math

import numpy as np

from .specfun import sph_hn, legendre_series


def shat(theta, phi):
    """Unit vector s(theta, phi) of P:256 (broadcasting)."""
    theta = np.asarray(theta, dtype=np.float64)
    phi = np.asarray(phi, dtype=np.float64)
    st = np.sin(theta)
    return np.stack(np.broadcast_arrays(np.cos(phi) * st, np.sin(phi) * st, np.cos(theta)), axis=-1)


def transfer_coeffs(ell: int, kappa: float, r0norm: float) -> np.ndarray:
    """c_n = (i kappa / 4 pi) i^n (2n+1) h_n(kappa |r0|), n = 0..ell."""
    h = sph_hn(ell, kappa * r0norm)
    n = np.arange(ell + 1)
    return (1j * kappa / (4 * math.pi)) * (1j ** n) * (2 * n + 1) * h


def transfer_eval(ell: int, kappa: float, r0vec, svec: np.ndarray) -> np.ndarray:
    """T_{ell, r0}(s) at unit vectors svec[..., 3]."""
    r0vec = np.asarray(r0vec, dtype=np.float64)
    r0n = float(np.linalg.norm(r0vec))
    c = transfer_coeffs(ell, kappa, r0n)
    t = np.clip(svec @ (r0vec / r0n), -1.0, 1.0)
    return legendre_series(c, t)


def s_tilde(n) -> np.ndarray:
    """Fourier coefficients of |sin theta|."""
    n = np.asarray(n)
    out = np.zeros(n.shape, dtype=np.float64)
    even = (n % 2) == 0
    out[even] = 2.0 / (math.pi * (1.0 - n[even].astype(np.float64) ** 2))
    return out


def _dft_rows(freqs: np.ndarray, npts: int) -> np.ndarray:
    """Matrix F[f, a] = exp(-i f 2 pi a / npts) / npts (forward coefficient extraction)."""
    a = np.arange(npts)
    return np.exp(-2j * math.pi * np.outer(freqs, a) / npts) / npts


def bmtf_coeffs(ell: int, kappa: float, r0vec, n_theta: int) -> np.ndarray:
    """2-D Fourier coefficients C[n, m] of T^{s,L} (Alg. 1).

    Rows n = -(N_theta/2 - 1) .. N_theta/2 - 1, columns m = -ell .. ell.
    Step 1: sample (1/2) T on the (2l+1) x (2l+1) grid (exact: T is a trig
            polynomial of degree <= l in theta and in phi).
    Step 2: 2-D spectrum T~[j, m].
    Step 3: (T^s)~[n, m] = sum_j T~[j, m] s~_{n-j}  (convolution),
            n truncated to |n| <= N_theta/2 - 1.
    """
    P = 2 * ell + 1
    g = 2 * math.pi * np.arange(P) / P
    th, ph = np.meshgrid(g, g, indexing="ij")
    samples = 0.5 * transfer_eval(ell, kappa, r0vec, shat(th, ph))      # [a (theta), b (phi)]
    j = np.arange(-ell, ell + 1)
    F = _dft_rows(j, P)                                                  # [freq, pt]
    Tt = F @ samples @ F.T                                               # [j, m]
    nmax = n_theta // 2 - 1
    n = np.arange(-nmax, nmax + 1)
    S = s_tilde(n[:, None] - j[None, :])                                 # [n, j]
    return S @ Tt                                                        # [n, m]


def eval_coeffs(C: np.ndarray, n_freqs: np.ndarray, m_freqs: np.ndarray, theta, phi) -> np.ndarray:
    """sum_{n,m} C[n,m] e^{i(n theta + m phi)} on the tensor grid theta x phi."""
    Et = np.exp(1j * np.outer(np.asarray(theta), n_freqs))
    Ep = np.exp(1j * np.outer(m_freqs, np.asarray(phi)))
    return Et @ C @ Ep


def bmtf_table(ell: int, kappa: float, r0vec, n_theta: int, n_phi: int) -> np.ndarray:
    """T^{s,LL} on the stored half grid [N_theta][N_phi/2]."""
    C = bmtf_coeffs(ell, kappa, r0vec, n_theta)
    nmax = n_theta // 2 - 1
    n = np.arange(-nmax, nmax + 1)
    mcut = min(ell, n_phi // 2 - 1)
    m_all = np.arange(-ell, ell + 1)
    keep = np.abs(m_all) <= mcut
    theta = 2 * math.pi * np.arange(n_theta) / n_theta
    phi = 2 * math.pi * np.arange(n_phi // 2) / n_phi
    return eval_coeffs(C[:, keep], n, m_all[keep], theta, phi)


def bmtf_table_rows(ell: int, kappa: float, r0vec, n_theta: int, rows) -> np.ndarray:
    """T^{s,LL} on a ragged stored half (R-15): row n keeps |m| <= N_phi(theta_n)/2 - 1
    and is sampled at phi = 2 pi q / N_phi(theta_n), q < N_phi(theta_n)/2; rows concatenated.
    (Rows of equal N_phi are evaluated together; the values are per row.)"""
    C = bmtf_coeffs(ell, kappa, r0vec, n_theta)
    nmax = n_theta // 2 - 1
    nf = np.arange(-nmax, nmax + 1)
    m_all = np.arange(-ell, ell + 1)
    rows = [int(r) for r in rows]
    out = [None] * n_theta
    for nph in sorted(set(rows)):
        ns = [n for n in range(n_theta) if rows[n] == nph]
        keep = np.abs(m_all) <= min(ell, nph // 2 - 1)
        theta = 2 * math.pi * np.asarray(ns) / n_theta
        phi = 2 * math.pi * np.arange(nph // 2) / nph
        vals = eval_coeffs(C[:, keep], nf, m_all[keep], theta, phi)          # [len(ns), nph/2]
        for i, n in enumerate(ns):
            out[n] = vals[i]
    return np.concatenate(out)


def bmtf_realspace_column(ell: int, kappa: float, r0vec, n_theta: int, phi: float) -> np.ndarray:
    """Real-space route of P:532 / Fig. SarvasDiag for one phi column.

    Sample (1/2)T at 2l+1 thetas, Fourier-interpolate to M = N_theta + 2l - 1
    points, multiply by |sin theta| bandlimited to |n| <= N_theta/2 + l - 1
    (sampled on the same M points), Fourier-anterpolate to N_theta points
    keeping |n| <= N_theta/2 - 1.  Returns T^{s,L}(theta_p, phi), p < N_theta.
    """
    P = 2 * ell + 1
    th = 2 * math.pi * np.arange(P) / P
    col = 0.5 * transfer_eval(ell, kappa, r0vec, shat(th, np.full(P, phi)))
    j = np.arange(-ell, ell + 1)
    Tt = _dft_rows(j, P) @ col
    M = n_theta + 2 * ell - 1
    thM = 2 * math.pi * np.arange(M) / M
    T_M = np.exp(1j * np.outer(thM, j)) @ Tt                               # interpolate
    kb = np.arange(-(n_theta // 2 + ell - 1), n_theta // 2 + ell)
    sin_band = (np.exp(1j * np.outer(thM, kb)) @ s_tilde(kb)).real          # bandlimited |sin|
    prod = T_M * sin_band
    nmax = n_theta // 2 - 1
    n = np.arange(-nmax, nmax + 1)
    coef = _dft_rows(n, M) @ prod                                          # anterpolate
    thN = 2 * math.pi * np.arange(n_theta) / n_theta
    return np.exp(1j * np.outer(thN, n)) @ coef


# The 316 transfer vectors of a level: o in [-3,3]^3 minus [-1,1]^3.
def offsets316() -> np.ndarray:
    r = range(-3, 4)
    out = [(x, y, z) for x in r for y in r for z in r if max(abs(x), abs(y), abs(z)) >= 2]
    return np.array(out, dtype=np.int64)


def offsets_canonical() -> np.ndarray:
    """Transfer vectors with x >= y >= 0, z >= 0 (Fig. SemiOctant)."""
    o = offsets316()
    keep = (o[:, 0] >= o[:, 1]) & (o[:, 1] >= 0) & (o[:, 2] >= 0)
    return o[keep]


def offset_id(o) -> int:
    """Index of offset o in offsets316() order (lexicographic x, y, z)."""
    table = {tuple(v): i for i, v in enumerate(offsets316())}
    return table[tuple(int(t) for t in o)]

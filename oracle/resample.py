"""Fourier interpolation / anterpolation on the sphere (TEST INFRASTRUCTURE).

P:373-378  interpolation pads Fourier coefficients with zeros, anterpolation truncates.
P:44       f(x) = sum_n F_n e^{inx}; forward coefficients carry 1/N.
P:512      kept band |n| <= N/2 - 1 (Nyquist bin dropped) -- reading R-6, applied to
           every 1-D resample in both directions.
P:729-748  the 5-step procedure between quadratures K and K' with
           calN_phi = max over both quadratures of N_phi(theta_n):
           (1) interpolate rows n <= N_theta/2 from N_phi(theta_n) to calN_phi
           (2) build theta-periodic columns m < calN_phi/2 with eqn:NumSphereSym
           (3) resample columns N_theta -> N'_theta
           (4) rebuild full phi-rows n <= N'_theta/2 with eqn:NumSphereSym
           (5) anterpolate rows calN_phi -> N'_phi(theta_n)
P:296      eqn:NumSphereSym  f(theta_n, phi_m) = f(theta_{N_theta - n}, phi_{N_phi/2 + m})

Representations
  "rows": list over n = 0..N_theta/2 of full phi-rows (ragged lengths allowed) --
          the paper's own layout
  "half": array [N_theta][N_phi/2] (theta over [0, 2pi), phi over [0, pi)) --
          Alg. 1's output domain, used by the FMM passes (reading R-7).
Every resample here is an explicit dense matrix built from the definition.

P:749      "A slightly more efficient algorithm uses the symmetry eqn:FourierSphereSym rather than
           eqn:NumSphereSym": resample_coeff_sym does the same operator in
           the phi-coefficient domain -- phi-DFT of the rows n <= N_theta/2, the theta sequence of
           each phi-frequency m extended by f~_{n,m} = (-1)^m f~_{-n,m} (eqn:FourierSphereSym,
           P:277-280, i.e. c_m(theta_{N_theta - n}) = (-1)^m c_m(theta_n)), resampled in theta,
           inverse phi-DFT of the rows n' <= N'_theta/2.
"""
from __future__ import annotations

import math
from functools import lru_cache
from typing import List, Sequence

import numpy as np


def band(N: int, Np: int) -> np.ndarray:
    """Kept frequencies |k| <= floor((min(N, N') - 1) / 2) (Nyquist dropped for even sizes)."""
    K = (min(N, Np) - 1) // 2
    return np.arange(-K, K + 1)


@lru_cache(maxsize=256)
def resample_matrix(N: int, Np: int) -> np.ndarray:
    """Dense R[p, j] = sum_{k in band} (1/N) e^{-2 pi i j k / N} e^{2 pi i k p / N'} (cached; read-only)."""
    k = band(N, Np)
    # e^{-2 pi i j k / N} is periodic in j k with period N: the integer product is reduced mod N
    # exactly before it becomes a phase, so every entry is within an ulp or two (an unreduced
    # phase of size ~pi N would carry ~u pi N / 2 of its own error)
    fwd = np.exp(-2j * math.pi * (np.outer(k, np.arange(N)) % N) / N) / N     # [k, j]
    inv = np.exp(2j * math.pi * (np.outer(np.arange(Np), k) % Np) / Np)       # [p, k]
    return inv @ fwd


def resample_1d(f: np.ndarray, Np: int, axis: int = -1) -> np.ndarray:
    """1-D Fourier resample of f along axis from its length N to N'."""
    f = np.moveaxis(np.asarray(f), axis, -1)
    R = resample_matrix(f.shape[-1], Np)
    return np.moveaxis(f @ R.T, -1, axis)


def half_to_rows(F: np.ndarray) -> List[np.ndarray]:
    """[N_theta][N_phi/2] -> full phi-rows for n = 0..N_theta/2 (eqn:NumSphereSym)."""
    nth = F.shape[0]
    return [np.concatenate([F[n], F[(nth - n) % nth]]) for n in range(nth // 2 + 1)]


def rows_to_half(rows: Sequence[np.ndarray], nth: int) -> np.ndarray:
    """Inverse of half_to_rows for a rectangular quadrature."""
    nph = len(rows[0])
    out = np.empty((nth, nph // 2), dtype=np.complex128)
    for n in range(nth):
        if n <= nth // 2:
            out[n] = rows[n][: nph // 2]
        else:
            out[n] = rows[nth - n][nph // 2:]
    return out


def resample_rows(rows: Sequence[np.ndarray], nth: int, nth_p: int,
                  nphi_p: Sequence[int], trace: list = None) -> List[np.ndarray]:
    """The 5-step procedure of P:738-748 on the paper's row layout.

    rows[n] (n = 0..N_theta/2) are full phi-rows of length N_phi(theta_n);
    nphi_p[n] (n = 0..N'_theta/2) are the target row lengths (multiples of 2).
    trace (optional list) receives the data profile after each step (Fig. 9).
    """
    if trace is not None:
        trace.append(("input", [len(r) for r in rows]))
    calN = max(max(len(r) for r in rows), max(nphi_p))
    # step 1: interpolate every row to calN_phi
    R1 = [resample_1d(r, calN) for r in rows]
    if trace is not None:
        trace.append(("I_phi", [len(r) for r in R1]))
    # step 2: theta-periodic columns m < calN/2 via eqn:NumSphereSym
    cols = np.empty((calN // 2, nth), dtype=np.complex128)
    for m in range(calN // 2):
        for n in range(nth):
            if n <= nth // 2:
                cols[m, n] = R1[n][m]
            else:
                cols[m, n] = R1[nth - n][m + calN // 2]
    if trace is not None:
        trace.append(("W", cols.shape))
    # step 3: resample columns N_theta -> N'_theta
    cols = resample_1d(cols, nth_p, axis=1)
    if trace is not None:
        trace.append(("A_theta", cols.shape))
    # step 4: full phi-rows n <= N'_theta/2 via eqn:NumSphereSym
    R4 = []
    for n in range(nth_p // 2 + 1):
        row = np.empty(calN, dtype=np.complex128)
        for m in range(calN):
            if m < calN // 2:
                row[m] = cols[m, n]
            else:
                row[m] = cols[m - calN // 2, (nth_p - n) % nth_p]
        R4.append(row)
    if trace is not None:
        trace.append(("W2", [len(r) for r in R4]))
    # step 5: anterpolate rows calN_phi -> N'_phi(theta_n)
    out = [resample_1d(R4[n], nphi_p[n]) for n in range(nth_p // 2 + 1)]
    if trace is not None:
        trace.append(("A_phi", [len(r) for r in out]))
    return out


def ragged_to_rows(F: np.ndarray, rows_n) -> List[np.ndarray]:
    """Ragged stored half (rows n < N_theta of N_phi(theta_n)/2 values, concatenated) -> full
    phi-rows for n = 0..N_theta/2 (eqn:NumSphereSym; N_phi(theta_{N_theta-n}) = N_phi(theta_n))."""
    nth = len(rows_n)
    off = np.concatenate([[0], np.cumsum(np.asarray(rows_n) // 2)])
    half = [F[off[n]: off[n + 1]] for n in range(nth)]
    return [np.concatenate([half[n], half[(nth - n) % nth]]) for n in range(nth // 2 + 1)]


def rows_to_ragged(rows: Sequence[np.ndarray], nth: int) -> np.ndarray:
    """Inverse of ragged_to_rows: full rows n <= N_theta/2 -> ragged stored half."""
    out = []
    for n in range(nth):
        if n <= nth // 2:
            r = rows[n]
            out.append(r[: len(r) // 2])
        else:
            r = rows[nth - n]
            out.append(r[len(r) // 2:])
    return np.concatenate(out)


def resample_ragged(F: np.ndarray, rows_n, nth_p: int, rows_p) -> np.ndarray:
    """5-step resample between two (possibly ragged) stored halves."""
    nth = len(rows_n)
    rows = ragged_to_rows(F, rows_n)
    out = resample_rows(rows, nth, nth_p, [int(rows_p[n]) for n in range(nth_p // 2 + 1)])
    return rows_to_ragged(out, nth_p)


def resample_half(F: np.ndarray, nph: int, nth_p: int, nph_p: int) -> np.ndarray:
    """5-step resample of a half-stored rectangular field [N_theta][N_phi/2] -> [N'_theta][N'_phi/2]."""
    nth = F.shape[0]
    assert F.shape[1] == nph // 2
    rows = half_to_rows(F)
    out = resample_rows(rows, nth, nth_p, [nph_p] * (nth_p // 2 + 1))
    return rows_to_half(out, nth_p)


def resample_half_batch(F: np.ndarray, nph: int, nth_p: int, nph_p: int) -> np.ndarray:
    """Same operator as resample_half, vectorised over a leading batch axis.

    F: [B][N_theta][N_phi/2].  Steps and index maps exactly as resample_rows
    (rectangular case); pinned equal to resample_half by a test.
    """
    F = np.asarray(F, dtype=np.complex128)
    B, nth, h = F.shape
    assert h == nph // 2
    calN = max(nph, nph_p)
    n_up = np.arange(nth // 2 + 1)
    # step 1: full rows n <= N_theta/2 (row n then row (N_theta - n) mod N_theta), resample
    rows = np.concatenate([F[:, n_up, :], F[:, (nth - n_up) % nth, :]], axis=2)   # [B, nth/2+1, nph]
    rows = rows @ resample_matrix(nph, calN).T                                   # [B, nth/2+1, calN]
    # step 2: columns m < calN/2 over n < N_theta
    n_all = np.arange(nth)
    lower = n_all <= nth // 2
    src_row = np.where(lower, n_all, nth - n_all)
    cols = np.where(lower[None, :, None],
                    rows[:, src_row, : calN // 2],
                    rows[:, src_row, calN // 2:])                              # [B, nth, calN/2]
    # step 3: resample columns N_theta -> N'_theta
    cols = np.einsum("pn,bnm->bpm", resample_matrix(nth, nth_p), cols)         # [B, nth', calN/2]
    # step 4: full rows n <= N'_theta/2
    n_up2 = np.arange(nth_p // 2 + 1)
    rows2 = np.concatenate([cols[:, n_up2, :], cols[:, (nth_p - n_up2) % nth_p, :]], axis=2)
    # step 5: resample rows calN -> N'_phi
    rows2 = rows2 @ resample_matrix(calN, nph_p).T                              # [B, nth'/2+1, nph']
    # back to half storage
    n_allp = np.arange(nth_p)
    lowp = n_allp <= nth_p // 2
    srcp = np.where(lowp, n_allp, nth_p - n_allp)
    return np.where(lowp[None, :, None],
                    rows2[:, srcp, : nph_p // 2],
                    rows2[:, srcp, nph_p // 2:])


def resample_coeff_sym(F: np.ndarray, nph: int, nth_p: int, nph_p: int) -> np.ndarray:
    """NEXT 4 (eqn:FourierSphereSym P:277-280): half-stored [B][N_theta][N_phi/2] ->
    [B][N'_theta][N'_phi/2], the same operator as resample_half_batch, computed in the
    phi-coefficient domain (module docstring).  Dense DFT matrices, literal steps."""
    F = np.asarray(F, dtype=np.complex128)
    B, nth, h = F.shape
    assert h == nph // 2
    n_up = np.arange(nth // 2 + 1)
    rows = np.concatenate([F[:, n_up, :], F[:, (nth - n_up) % nth, :]], axis=2)      # full rows n <= N_theta/2
    m = band(nph, nph_p)                                                            # kept phi band
    fwd = np.exp(-2j * math.pi * (np.outer(np.arange(nph), m) % nph) / nph) / nph    # [j, m]
    C = rows @ fwd                                                                  # c_m(theta_n), n <= N_theta/2
    # theta sequence of every m over n < N_theta: c_m(theta_{N_theta - n}) = (-1)^m c_m(theta_n)
    n_all = np.arange(nth)
    lower = n_all <= nth // 2
    src = np.where(lower, n_all, nth - n_all)
    sign = np.where(lower[:, None], 1.0, ((-1.0) ** np.abs(m))[None, :])            # [n, m]
    Cfull = C[:, src, :] * sign[None]                                               # [B, nth, m]
    Cp = np.einsum("pn,bnm->bpm", resample_matrix(nth, nth_p), Cfull)               # [B, nth', m]
    n_up2 = np.arange(nth_p // 2 + 1)
    inv = np.exp(2j * math.pi * (np.outer(m, np.arange(nph_p)) % nph_p) / nph_p)     # [m, t]
    rows2 = Cp[:, n_up2, :] @ inv                                                   # full rows n' <= N'_theta/2
    n_allp = np.arange(nth_p)
    lowp = n_allp <= nth_p // 2
    srcp = np.where(lowp, n_allp, nth_p - n_allp)
    return np.where(lowp[None, :, None], rows2[:, srcp, : nph_p // 2], rows2[:, srcp, nph_p // 2:])

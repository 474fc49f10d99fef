"""Per-level plan: ell, N_theta, N_phi, F_l, L_f (TEST INFRASTRUCTURE; see oracle/__init__.py).

Follows, in order:
  P:692-701   worst-case radii |r0| = 2 a_l, |r| = alpha a_l sqrt(3)
  P:146-165   ell: EBF initial guess (eqn:EBF, C = 1.8 d0^{2/3}) refined with the
              Carayol-Collino closed form eqn:CollinoError (max over the +/- cases)
  P:596-635   Alg. 2 (N_theta) with eqn:EpsITheta, M(N,n)
  P:637-686   Alg. 3 (N_phi(theta_n)) with eqn:EpsIPhi
  P:833       low-frequency breakdown -> admissibility F_l <= tau (R-9)

Readings of silent/ambiguous points are listed in DESIGN.md ("Readings"):
  R-1 eps_l = eps / a_l (per-level absolute target; = the paper at a = 1)
  R-2 d0 = -log10(eps_l); ell = smallest ell >= max(1, ceil(kappa r)) with the
      Collino bound < eps_l; EBF alone when kappa r <= 1
  R-3 N^max = 4 ell + 64 (doubled on failure); threshold eps_l / (4 pi^2) in both
      Algs
  R-4 grid sizes restricted to FFT-friendly 7-smooth values: N_theta = smallest even
      7-smooth N >= 2 ell passing Alg. 2; rectangular N_phi = smallest 7-smooth
      multiple of 4 for which EVERY row n <= N_theta/2 passes Alg. 3's test
  R-5 monotone grids on the active chain: N^{l-1} >= N^l per dimension
  R-9 F_l = 8 pi u a_l max |T^{s,LL}_l| over the 34 canonical offsets, u = 2^-53;
      active iff F_l <= tau; L_f = deepest l with 2..l all active.
  R-13 design radius per level: the largest alpha in {1, 0.9, 0.8} (>= the caller's alpha)
      whose quadrature keeps F_l <= tau (the paper uses alpha = 1 for its volume timing runs,
      P:1161, and 0.8 in its error studies; pairs beyond alpha sqrt3 a are not covered
      by the bound).  alpha_fixed=True: the caller's alpha at every level.
  R-14 source level ("additional translation steps"): S2M and L2T
      run at a source level D_s in [L_f, depth]; the levels L_f < l <= D_s are translation-only
      (M2M up, L2L down with I = 0, no M2L).  Their grid represents the outgoing field of a box,
      a sum of plane waves e^{i kappa s.(x - c)} with |x - c| <= rho_l = (sqrt3/2) a_l, whose
      Fourier series in theta (and phi) is the Jacobi-Anger series of eqn:PlaneWaveSpec
       with argument <= kappa rho_l: N_theta = smallest even 7-smooth N >= 4 and
      N_phi = smallest 7-smooth multiple of 4 whose dropped band |n| >= N/2 has
      2 sum_{n >= N/2} |J_n(kappa rho_l)| <= eps / 100.  R-5 (monotone grids) holds on the
      whole chain 2..D_s.  Policy for D_s (choose_source_level): the deepest level <= depth whose
      occupied boxes hold >= 8 points on average (L_f if none); D_s = L_f is the paper's setup.
  R-15 ragged quadrature (Alg. 3's per-row result): with ragged=True
      every active level stores N_phi(theta_n) points on row n, N_phi(theta_n) = the smallest
      7-smooth multiple of 4 at which row n passes Alg. 3's test (eqn:EpsIPhi, threshold
      eps_l / 4 pi^2) at the level's final N_theta (after R-5); rows n > N_theta/2 mirror
      N_theta - n, rows n and N_theta/2 - n take the larger of the two (exact theta -> pi - theta
      symmetry for the 34-table permutations).  Never above the rectangular N_phi.  F_l, L_f and R-5 use the rectangular grid;
      translation-only levels stay rectangular.  The 5-step resample maps between any
      two quadratures; the stored half keeps N_phi(theta_n)/2 points per row.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field
from typing import List, Optional

import numpy as np

from .specfun import sph_jn, sph_hn, besselJ
from .transfer import bmtf_coeffs, eval_coeffs, bmtf_table, offsets_canonical

U_ROUND = 2.0 ** -53


def is_7smooth(n: int) -> bool:
    if n <= 0:
        return False
    for p in (2, 3, 5, 7):
        while n % p == 0:
            n //= p
    return n == 1


def ebf_ell(kappa_r: float, eps: float) -> int:
    """eqn:EBF: ell ~ kappa r + 1.8 d0^{2/3} (kappa r)^{1/3}."""
    d0 = -math.log10(eps)
    return int(math.ceil(kappa_r + 1.8 * d0 ** (2.0 / 3.0) * kappa_r ** (1.0 / 3.0)))


def collino_bound(ell: int, kappa: float, r: float, r0: float) -> float:
    """eqn:CollinoError, maximised over the two sign cases."""
    h = sph_hn(ell + 1, kappa * r0)
    j = sph_jn(ell + 1, kappa * r)
    best = 0.0
    for s in (+1.0, -1.0):
        val = kappa ** 2 * (r * r0 / (r0 + s * r)) * abs(h[ell + 1] * j[ell] + s * h[ell] * j[ell + 1])
        if not np.isfinite(val):
            return math.inf
        best = max(best, val)
    return best


def choose_ell(kappa: float, r: float, r0: float, eps: float, ell_max: int = 4000) -> int:
    """Sec. 2.1: EBF guess refined by the closed form (reading R-2)."""
    kr = kappa * r
    if kr <= 1.0:
        return max(1, ebf_ell(kr, eps))
    lo = max(1, int(math.ceil(kr)))
    for ell in range(lo, ell_max):
        if collino_bound(ell, kappa, r, r0) < eps:
            return ell
    raise RuntimeError("choose_ell: search failed")


def M_index(N: int, n: np.ndarray) -> np.ndarray:
    """M(N, n) of P:613-619."""
    a = np.abs(n)
    return np.where(a < N / 2.0, N - a, a)


def theta_spectrum_z(ell: int, kappa: float, r0: float, nmax_pts: int) -> np.ndarray:
    """Alg. 2 lines 1-3: |F_n[T^{s,L}_{ell,|r0| z}(2 pi n / N^max, 0)]|, n = -N^max/2 .. N^max/2-1."""
    C = bmtf_coeffs(ell, kappa, (0.0, 0.0, r0), nmax_pts)
    nlim = nmax_pts // 2 - 1
    nf = np.arange(-nlim, nlim + 1)
    mf = np.arange(-ell, ell + 1)
    theta = 2 * math.pi * np.arange(nmax_pts) / nmax_pts
    samples = eval_coeffs(C, nf, mf, theta, np.array([0.0]))[:, 0]
    freqs = np.arange(-(nmax_pts // 2), nmax_pts // 2)
    F = np.exp(-2j * math.pi * np.outer(freqs, np.arange(nmax_pts)) / nmax_pts) / nmax_pts
    return freqs, np.abs(F @ samples)


def choose_ntheta(ell: int, kappa: float, r: float, r0: float, eps: float) -> int:
    """Alg. 2, candidates restricted to even 7-smooth N (R-4)."""
    nmax = 4 * ell + 64
    for _ in range(4):
        freqs, Tt = theta_spectrum_z(ell, kappa, r0, nmax)
        E = np.abs(besselJ(2 * nmax, kappa * r))
        thr = eps / (4 * math.pi ** 2)
        for N in range(2 * ell, nmax, 2):
            if not is_7smooth(N):
                continue
            bound = float(np.sum(Tt * E[M_index(N, freqs)]))
            if bound < thr:
                return N
        nmax *= 2
    raise RuntimeError("choose_ntheta: search failed")


def phi_spectra_x(ell: int, kappa: float, r0: float, n_theta: int) -> np.ndarray:
    """Alg. 3 lines 3-4 for every row n <= N_theta/2: |F_m[T^{s,L}_{ell,|r0| x}(theta_n, .)]|."""
    C = bmtf_coeffs(ell, kappa, (r0, 0.0, 0.0), n_theta)
    nlim = n_theta // 2 - 1
    nf = np.arange(-nlim, nlim + 1)
    mf = np.arange(-ell, ell + 1)
    theta = 2 * math.pi * np.arange(n_theta // 2 + 1) / n_theta
    P = 2 * ell + 1
    phi = 2 * math.pi * np.arange(P) / P
    S = eval_coeffs(C, nf, mf, theta, phi)                                 # [row, m-sample]
    F = np.exp(-2j * math.pi * np.outer(mf, np.arange(P)) / P) / P
    return mf, np.abs(S @ F.T), theta                                     # [row, m]


def nphi_row_bounds(ell, kappa, r, r0, n_theta, candidates):
    """eqn:EpsIPhi bound for every row and every candidate N."""
    mf, Tt, theta = phi_spectra_x(ell, kappa, r0, n_theta)
    Nmax = max(candidates)
    out = np.empty((len(theta), len(candidates)))
    for i, th in enumerate(theta):
        E = np.abs(besselJ(2 * Nmax, kappa * r * abs(math.sin(th))))
        for c, N in enumerate(candidates):
            out[i, c] = float(np.sum(Tt[i] * E[M_index(N, mf)]))
    return out


def choose_nphi(ell: int, kappa: float, r: float, r0: float, eps: float, n_theta: int):
    """Alg. 3.

    Returns (rectangular N_phi, ragged per-row N_phi(theta_n) list).
    Ragged rows: first multiple of 4 passing.  Rectangular (R-4):
    smallest 7-smooth multiple of 4 at which every row passes.
    """
    thr = eps / (4 * math.pi ** 2)
    Nmax = 4 * ell + 64
    Nmax -= Nmax % 4
    cands = list(range(4, Nmax + 1, 4))
    B = nphi_row_bounds(ell, kappa, r, r0, n_theta, cands)
    ragged = []
    for i in range(B.shape[0]):
        ok = np.nonzero(B[i] < thr)[0]
        if len(ok) == 0:
            raise RuntimeError("choose_nphi: row search failed")
        ragged.append(cands[ok[0]])
    allok = np.all(B < thr, axis=0)
    for c, N in enumerate(cands):
        if allok[c] and is_7smooth(N):
            return N, ragged
    raise RuntimeError("choose_nphi: rectangular search failed")


@dataclass
class LevelPlan:
    level: int
    a: float
    ell: int
    n_theta: int
    n_phi: int
    ragged: List[int] = field(default_factory=list)
    F: float = float("nan")
    active: bool = False
    alpha: float = 0.8
    rep: bool = False        # translation-only level below L_f (R-14): no ell, no M2L
    rows: Optional[List[int]] = None   # R-15: N_phi(theta_n) for n < N_theta (None: rectangular)

    @property
    def K(self) -> int:
        if self.rows is not None:
            return sum(self.rows) // 2
        return self.n_theta * self.n_phi // 2

    def row_nphi(self) -> List[int]:
        """N_phi of every stored row n < N_theta (constant for a rectangular grid)."""
        return list(self.rows) if self.rows is not None else [self.n_phi] * self.n_theta


@dataclass
class Plan:
    kappa: float
    eps: float
    alpha: float
    tau: float
    a0: float
    depth: int
    levels: dict            # level -> LevelPlan
    L_f: Optional[int]      # None: no admissible level -> P2P over all pairs
    source_level: Optional[int] = None   # S2M / L2T level D_s (R-14); None iff L_f is None
    ragged: bool = False                 # R-15: ragged rows on the active levels
    eps_absolute: bool = False


def level_params(kappa: float, a: float, eps: float, alpha: float, eps_absolute: bool = False):
    """(ell, N_theta, N_phi, ragged) for one level of box size a."""
    eps_l = eps if eps_absolute else eps / a
    r = alpha * a * math.sqrt(3.0)
    r0 = 2.0 * a
    ell = choose_ell(kappa, r, r0, eps_l)
    nth = choose_ntheta(ell, kappa, r, r0, eps_l)
    nph, ragged = choose_nphi(ell, kappa, r, r0, eps_l, nth)
    return ell, nth, nph, ragged


def level_F(kappa: float, a: float, ell: int, nth: int, nph: int) -> float:
    """F_l = 8 pi u a max |T_l| over the 34 canonical transfer vectors (R-9)."""
    mx = 0.0
    for o in offsets_canonical():
        T = bmtf_table(ell, kappa, o.astype(np.float64) * a, nth, nph)
        mx = max(mx, float(np.max(np.abs(T))))
    return 8 * math.pi * U_ROUND * a * mx


REP_EPS_FACTOR = 1e-2       # R-14: representation tail <= eps / 100
MIN_MEAN_POINTS = 8.0       # R-14: source-level policy


def rep_tail(z: float, N: int) -> float:
    """Jacobi-Anger mass dropped by keeping |n| <= N/2 - 1 (eqn:PlaneWaveSpec)."""
    J = np.abs(besselJ(N + 2 * int(math.ceil(z)) + 40, z))
    return 2.0 * float(np.sum(J[N // 2:]))


def rep_grid(kappa: float, a: float, eps: float):
    """(N_theta, N_phi) of a translation-only level of box size a (R-14)."""
    z = kappa * math.sqrt(3.0) / 2.0 * a
    thr = eps * REP_EPS_FACTOR
    nth = next(N for N in range(4, 100000, 2) if is_7smooth(N) and rep_tail(z, N) <= thr)
    nph = next(N for N in range(4, 100000, 4) if is_7smooth(N) and rep_tail(z, N) <= thr)
    return nth, nph


def ragged_rows(lp: "LevelPlan", kappa: float, eps: float, eps_absolute: bool = False) -> List[int]:
    """R-15: per-row N_phi(theta_n) of an active level at its final N_theta (Alg. 3)."""
    a = lp.a
    eps_l = eps if eps_absolute else eps / a
    r, r0 = lp.alpha * a * math.sqrt(3.0), 2.0 * a
    thr = eps_l / (4 * math.pi ** 2)
    cands = [N for N in range(4, lp.n_phi + 1, 4) if is_7smooth(N)]
    B = nphi_row_bounds(lp.ell, kappa, r, r0, lp.n_theta, cands)       # rows n <= N_theta / 2
    half = []
    for i in range(B.shape[0]):
        ok = np.nonzero(B[i] < thr)[0]
        half.append(cands[ok[0]] if len(ok) else lp.n_phi)
    nth = lp.n_theta
    # exact reflection symmetry theta -> pi - theta (rows n and N_theta/2 - n), required by the
    # 34-table permutations; the two bounds agree up to rounding, take the larger row
    half = [max(half[n], half[nth // 2 - n]) for n in range(nth // 2 + 1)]
    return [half[n] if n <= nth // 2 else half[nth - n] for n in range(nth)]


def choose_source_level(x: np.ndarray, lo, a0: float, depth: int, L_f: Optional[int],
                        min_mean: float = MIN_MEAN_POINTS) -> Optional[int]:
    """R-14 policy: deepest l in [L_f, depth] whose occupied boxes hold >= min_mean points on average."""
    if L_f is None:
        return None
    from .tree import box_coords
    for l in range(depth, L_f, -1):
        b = box_coords(np.asarray(x), lo, a0, l)
        nocc = len(np.unique(b[:, 0] * 4 ** l + b[:, 1] * 2 ** l + b[:, 2]))
        if len(x) / nocc >= min_mean:
            return l
    return L_f


def default_tau(eps: float) -> float:
    return min(eps / 10.0, 1e-9)


def alpha_candidates(alpha: float, fixed: bool):
    """Design radii tried per level, largest first (R-13): {1, 0.9, 0.8} above the caller's alpha."""
    if fixed:
        return [alpha]
    return [c for c in (1.0, 0.9, 0.8) if c > alpha + 1e-12] + [alpha]


def make_plan(kappa: float, eps: float, a0: float, depth: int, alpha: float = 0.8,
              tau: Optional[float] = None, force_all: bool = False,
              eps_absolute: bool = False, alpha_fixed: bool = False,
              source_level: Optional[int] = None, ragged: bool = False) -> Plan:
    """Plan for levels 2..depth (P:140-722 + admissibility R-9, design radius R-13, monotone R-5).

    Shallowest level first: for each candidate design radius alpha (R-13, largest first) take
    the quadrature of P:140-722 and F_l; the level is active with the first alpha whose
    F_l <= tau.  The first level with no admissible alpha ends the chain (L_f = l - 1); deeper
    levels are reported with the caller's alpha and no F."""
    if tau is None or tau <= 0:
        tau = default_tau(eps)
    ragged_grids = bool(ragged)        # (the loop below rebinds `ragged` to Alg. 3's row lists)
    levels = {}
    L_f = None
    cands = alpha_candidates(alpha, alpha_fixed or force_all)
    stop = None
    for l in range(2, depth + 1):
        a = a0 / 2 ** l
        if stop is not None:
            ell, nth, nph, ragged = level_params(kappa, a, eps, alpha, eps_absolute)
            levels[l] = LevelPlan(l, a, ell, nth, nph, ragged, alpha=alpha)
            continue
        for al in cands:
            ell, nth, nph, ragged = level_params(kappa, a, eps, al, eps_absolute)
            lp = LevelPlan(l, a, ell, nth, nph, ragged, alpha=al)
            lp.F = level_F(kappa, a, ell, nth, nph)
            lp.active = force_all or lp.F <= tau
            if lp.active:
                break
        levels[l] = lp
        if lp.active:
            L_f = l
        else:
            stop = l
    plan = Plan(kappa, eps, alpha, tau, a0, depth, levels, L_f, L_f, ragged_grids, eps_absolute)
    if L_f is not None:
        set_source_level(plan, L_f if source_level is None else source_level)
    return plan


def set_source_level(plan: Plan, source_level: int) -> Plan:
    """Translation-only levels L_f < l <= D_s (R-14) and monotone grids on the chain 2..D_s (R-5)."""
    L_f, kappa, eps, a0, levels = plan.L_f, plan.kappa, plan.eps, plan.a0, plan.levels
    D_s = max(L_f, min(int(source_level), plan.depth))
    for l in range(L_f + 1, D_s + 1):
        a = a0 / 2 ** l
        nth, nph = rep_grid(kappa, a, eps)
        levels[l] = LevelPlan(l, a, 0, nth, nph, [], alpha=plan.alpha, rep=True)
    for l in range(D_s - 1, 1, -1):
        up, dn = levels[l], levels[l + 1]
        nth = max(up.n_theta, dn.n_theta)
        nph = max(up.n_phi, dn.n_phi)
        if (nth, nph) != (up.n_theta, up.n_phi):
            up.n_theta, up.n_phi = nth, nph
            if not up.rep:
                up.F = level_F(kappa, up.a, up.ell, nth, nph)
    plan.source_level = D_s
    for l in range(2, L_f + 1):          # R-15 at the final N_theta of every active level
        levels[l].rows = ragged_rows(levels[l], kappa, eps, plan.eps_absolute) if plan.ragged else None
    return plan

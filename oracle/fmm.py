"""FMM passes of Sec. 2 for the oracle (TEST INFRASTRUCTURE; see oracle/__init__.py).

  S2M  M^L_a(s) = sum_{x_i in B_a} psi_i e^{i kappa s.(x_i - c_a)}
  M2M  M^{l-1}_a = sum_{children b} M^l_b e^{i kappa s.(c_b - c_a)}, preceded by
                    Fourier interpolation to the parent quadrature (R-10)
  M2L  I^l_a = sum_{b in I(B_a)} M^l_b T_{l, c_b - c_a}   (T = T^{s,LL}, Alg. 1)
  L2L  L^{l+1}_a = L^l_b e^{i kappa s.(c_b - c_a)} + I^{l+1}_a, the product
                    anterpolated to the child quadrature before adding I (R-10)
  L2T  sigma_i = int L e^{i kappa s.(c - x_i)} dS
                    = (4 pi^2 / (N_theta N_phi)) sum over the doubled grid
                    = (8 pi^2 / (N_theta N_phi)) sum over the stored half
  P2P  sum over j != i in the neighbour list N(B^L_a) of e^{i kappa R}/R psi_j
If no level is admissible (L_f is None) the near field is every pair (direct sum).
Highest M2L level is l = 2; no work at levels 0-1.
Source level D_s = plan.source_level (reading R-14): S2M and L2T at D_s; the levels
L_f < l <= D_s are translation-only (M2M up, L2L down with I = 0); M2L at 2..L_f and the
near field (P2P) over the neighbour lists of L_f, exactly as for D_s = L_f.
"""
from __future__ import annotations

import math
from typing import Dict, Optional

import numpy as np

from .plan import Plan
from .resample import resample_half_batch, resample_ragged
from .transfer import shat, bmtf_table, bmtf_table_rows
from .tree import build_level, neighbours, interaction_list, parent


class OracleFMM:
    def __init__(self, x: np.ndarray, lo, a0: float, plan: Plan):
        self.x = np.asarray(x, dtype=np.float64)
        self.lo = np.asarray(lo, dtype=np.float64)
        self.a0 = float(a0)
        self.plan = plan
        self.kappa = plan.kappa
        self.L = plan.L_f
        self.S = plan.source_level if plan.source_level is not None else plan.L_f
        self.levels = {}
        if self.L is not None:
            for l in range(2, self.S + 1):
                self.levels[l] = build_level(self.x, self.lo, self.a0, l)
        self._tables: Dict[tuple, np.ndarray] = {}

    # ---- quadrature of level l (half storage) -----------------------
    def grid(self, l: int):
        """Stored directions, row by row: theta_n = 2 pi n / N_theta, phi = 2 pi m / N_phi(theta_n),
        m < N_phi(theta_n)/2 (rectangular: k = n * (N_phi/2) + m; ragged rows R-15)."""
        lp = self.plan.levels[l]
        th, ph = self.grid_angles(l)
        return shat(th, ph)                                      # [K, 3]

    def grid_angles(self, l: int):
        lp = self.plan.levels[l]
        rows = lp.row_nphi()
        th = np.concatenate([np.full(r // 2, 2 * math.pi * n / lp.n_theta) for n, r in enumerate(rows)])
        ph = np.concatenate([2 * math.pi * np.arange(r // 2) / r for r in rows])
        return th, ph

    def ragged(self, l: int) -> bool:
        return self.plan.levels[l].rows is not None

    def resample(self, F: np.ndarray, l_from: int, l_to: int) -> np.ndarray:
        """5-step resample of one stored field between the quadratures of two levels."""
        a, b = self.plan.levels[l_from], self.plan.levels[l_to]
        if a.rows is None and b.rows is None:
            return resample_half_batch(F.reshape(1, a.n_theta, a.n_phi // 2), a.n_phi, b.n_theta,
                                       b.n_phi).reshape(-1)
        return resample_ragged(F, a.row_nphi(), b.n_theta, b.row_nphi())

    def table(self, l: int, o) -> np.ndarray:
        key = (l, tuple(int(v) for v in o))
        if key not in self._tables:
            lp = self.plan.levels[l]
            r0 = np.asarray(o, dtype=np.float64) * lp.a
            if lp.rows is not None:
                self._tables[key] = bmtf_table_rows(lp.ell, self.kappa, r0, lp.n_theta, lp.rows)
            else:
                self._tables[key] = bmtf_table(lp.ell, self.kappa, r0, lp.n_theta, lp.n_phi).reshape(-1)
        return self._tables[key]

    # ---- passes ---------------------------------------------------------------
    def s2m(self, q: np.ndarray, boxes=None) -> Dict[int, np.ndarray]:
        lev = self.levels[self.S]
        S = self.grid(self.S)
        out = {}
        for b in (range(len(lev.boxes)) if boxes is None else boxes):
            idx = lev.members[b]
            d = self.x[idx] - lev.centers[b]                                    # x_i - c_a
            E = np.exp(1j * self.kappa * (S @ d.T))                             # [K, n]
            out[b] = E @ q[idx]
        return out

    def m2m(self, Ml: Dict[int, np.ndarray], l: int) -> Dict[int, np.ndarray]:
        """Level l -> l-1: interpolate, multiply by e^{i kappa s.(c_b - c_a)}, accumulate."""
        ch, pa = self.levels[l], self.levels[l - 1]
        Sp = self.grid(l - 1)
        out = {}
        for b, M in Ml.items():
            Mi = self.resample(M, l, l - 1)
            p = pa.index[parent(ch.boxes[b])]
            shift = np.exp(1j * self.kappa * (Sp @ (ch.centers[b] - pa.centers[p])))
            out[p] = out.get(p, 0) + shift * Mi
        return out

    def m2l(self, Ml: Dict[int, np.ndarray], l: int, targets=None) -> Dict[int, np.ndarray]:
        lev = self.levels[l]
        K = self.plan.levels[l].K
        out = {}
        for a in (range(len(lev.boxes)) if targets is None else targets):
            acc = np.zeros(K, dtype=np.complex128)
            for b, o in interaction_list(lev, lev.boxes[a]):
                acc += self.table(l, o) * Ml[b]                                  # T_{c_b - c_a}
            out[a] = acc
        return out

    def l2l(self, Ll: Dict[int, np.ndarray], I_next: Dict[int, np.ndarray], l: int):
        """Level l -> l+1: multiply by e^{i kappa s.(c_parent - c_child)}, anterpolate, add I."""
        pa, ch = self.levels[l], self.levels[l + 1]
        Sp = self.grid(l)
        out = {}
        for c, I in I_next.items():
            p = pa.index[parent(ch.boxes[c])]
            shift = np.exp(1j * self.kappa * (Sp @ (pa.centers[p] - ch.centers[c])))
            out[c] = self.resample(shift * Ll[p], l, l + 1) + I
        return out

    def l2t(self, Lf: Dict[int, np.ndarray], targets: np.ndarray) -> np.ndarray:
        lev = self.levels[self.S]
        lp = self.plan.levels[self.S]
        S = self.grid(self.S)
        # doubled-grid weight 4 pi^2 / (N_theta N_phi(theta_n)) x 2 for half storage
        w = np.concatenate([np.full(r // 2, 8 * math.pi ** 2 / (lp.n_theta * r)) for r in lp.row_nphi()])
        y = np.zeros(len(targets), dtype=np.complex128)
        box_of = self._box_of_points(targets, self.S)
        for a in np.unique(box_of):
            sel = np.nonzero(box_of == a)[0]
            d = lev.centers[a] - self.x[targets[sel]]                            # c_a - x_i
            E = np.exp(1j * self.kappa * (d @ S.T))                              # [n, K]
            y[sel] = E @ (w * Lf[a])
        return y

    def p2p(self, q: np.ndarray, targets: np.ndarray) -> np.ndarray:
        y = np.zeros(len(targets), dtype=np.complex128)
        if self.L is None:                                   # every pair is near
            src_sets = {None: np.arange(len(self.x))}
            groups = {None: np.arange(len(targets))}
        else:
            lev = self.levels[self.L]
            box_of = self._box_of_points(targets, self.L)
            groups, src_sets = {}, {}
            for a in np.unique(box_of):
                groups[a] = np.nonzero(box_of == a)[0]
                src_sets[a] = np.concatenate([lev.members[b] for b in neighbours(lev, lev.boxes[a])])
        for a, sel in groups.items():
            src = src_sets[a]
            ti = targets[sel]
            d = self.x[ti][:, None, :] - self.x[src][None, :, :]
            R = np.sqrt(np.sum(d * d, axis=2))
            self_pair = ti[:, None] == src[None, :]
            if np.any((R == 0) & ~self_pair):
                raise ValueError("coincident points")
            with np.errstate(divide="ignore", invalid="ignore"):
                G = np.where(self_pair, 0.0, np.exp(1j * self.kappa * R) / np.where(self_pair, 1.0, R))
            y[sel] = G @ q[src]
        return y

    def _box_of_points(self, idx: np.ndarray, level: int) -> np.ndarray:
        lev = self.levels[level]
        n = 2 ** level
        b = np.minimum(np.floor((self.x[idx] - self.lo) / lev.a).astype(np.int64), n - 1)
        return np.array([lev.index[tuple(v)] for v in b], dtype=np.int64)

    # ---- the matvec ------------------------------------------------------------
    def far_locals(self, q: np.ndarray):
        """Run S2M, M2M, M2L, L2L; return (M per level, I per level, L per level down to D_s)."""
        L, S = self.L, self.S
        M = {S: self.s2m(q)}
        for l in range(S, 2, -1):
            M[l - 1] = self.m2m(M[l], l)
        I = {l: self.m2l(M[l], l) for l in range(2, L + 1)}
        for l in range(L + 1, S + 1):                 # translation-only levels: no M2L (R-14)
            K = self.plan.levels[l].K
            I[l] = {b: np.zeros(K, dtype=np.complex128) for b in range(len(self.levels[l].boxes))}
        Lloc = {2: I[2]}
        for l in range(2, S):
            Lloc[l + 1] = self.l2l(Lloc[l], I[l + 1], l)
        return M, I, Lloc

    def matvec(self, q: np.ndarray, targets: Optional[np.ndarray] = None, parts: bool = False):
        """y_i for i in targets (default: all), eqn:FMM_FinalStep."""
        q = np.asarray(q, dtype=np.complex128)
        if targets is None:
            targets = np.arange(len(self.x))
        y_near = self.p2p(q, targets)
        if self.L is None:
            y_far = np.zeros_like(y_near)
        else:
            _, _, Lloc = self.far_locals(q)
            y_far = self.l2t(Lloc[self.S], targets)
        if parts:
            return y_near, y_far
        return y_near + y_far

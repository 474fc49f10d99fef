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

Target-subset mode (`matvec_subset`): the same passes restricted to what a
sample of targets needs -- S2M for every source box and M2M at every box (every M is a potential
M2L partner), M2L and L2L only on the ancestors of the targets' source-level boxes, L2T and P2P
only for the targets.  Each restricted pass computes exactly the values the full pass computes for
those boxes (same functions, same summation order), so y at the sampled targets is the full
matvec's y there.  `workers` > 1 runs the independent per-box loops (S2M, M2L, P2P and L2T groups)
on a thread pool (numpy releases the GIL); every box is still computed by the same code.
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


def _pmap(fn, items, workers: int):
    """[fn(i) for i in items], on a thread pool when workers > 1 (order preserved)."""
    items = list(items)
    if workers <= 1 or len(items) < 2:
        return [fn(i) for i in items]
    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(workers) as ex:
        return list(ex.map(fn, items, chunksize=max(1, len(items) // (8 * workers))))


class OracleFMM:
    def __init__(self, x: np.ndarray, lo, a0: float, plan: Plan, workers: int = 1):
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
        self.workers = int(workers)

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
        def one(b):
            idx = lev.members[b]
            d = self.x[idx] - lev.centers[b]                                    # x_i - c_a
            E = np.exp(1j * self.kappa * (S @ d.T))                             # [K, n]
            return E @ q[idx]
        bs = list(range(len(lev.boxes)) if boxes is None else boxes)
        return dict(zip(bs, _pmap(one, bs, self.workers)))

    def m2m(self, Ml: Dict[int, np.ndarray], l: int) -> Dict[int, np.ndarray]:
        """Level l -> l-1: interpolate, multiply by e^{i kappa s.(c_b - c_a)}, accumulate."""
        ch, pa = self.levels[l], self.levels[l - 1]
        Sp = self.grid(l - 1)
        out = {}
        for b, Mi in self._resample_all(Ml, l, l - 1):
            p = pa.index[parent(ch.boxes[b])]
            shift = np.exp(1j * self.kappa * (Sp @ (ch.centers[b] - pa.centers[p])))
            out[p] = out.get(p, 0) + shift * Mi
        return out

    def m2l(self, Ml: Dict[int, np.ndarray], l: int, targets=None) -> Dict[int, np.ndarray]:
        lev = self.levels[l]
        K = self.plan.levels[l].K
        as_ = list(range(len(lev.boxes)) if targets is None else targets)
        lists = [interaction_list(lev, lev.boxes[a]) for a in as_]
        for lst in lists:                          # tables built once, before any threads run
            for _, o in lst:
                self.table(l, o)

        def one(i):
            acc = np.zeros(K, dtype=np.complex128)
            for b, o in lists[i]:
                acc += self.table(l, o) * Ml[b]                                  # T_{c_b - c_a}
            return acc
        return dict(zip(as_, _pmap(one, range(len(as_)), self.workers)))

    def l2l(self, Ll: Dict[int, np.ndarray], I_next: Dict[int, np.ndarray], l: int):
        """Level l -> l+1: multiply by e^{i kappa s.(c_parent - c_child)}, anterpolate, add I."""
        pa, ch = self.levels[l], self.levels[l + 1]
        Sp = self.grid(l)
        shifted = {}
        for c in I_next:
            p = pa.index[parent(ch.boxes[c])]
            shifted[c] = np.exp(1j * self.kappa * (Sp @ (pa.centers[p] - ch.centers[c]))) * Ll[p]
        return {c: R + I_next[c] for c, R in self._resample_all(shifted, l, l + 1)}

    def _resample_all(self, fields: Dict[int, np.ndarray], l_from: int, l_to: int, chunk: int = 512):
        """(key, resample(field)) for every field; rectangular grids go through the batched 5-step
        (resample_half_batch, pinned equal to the literal procedure) in bounded chunks."""
        a, b = self.plan.levels[l_from], self.plan.levels[l_to]
        keys = list(fields)
        if a.rows is not None or b.rows is not None:
            for k in keys:
                yield k, self.resample(fields[k], l_from, l_to)
            return
        for i in range(0, len(keys), chunk):
            ks = keys[i:i + chunk]
            F = np.stack([fields[k].reshape(a.n_theta, a.n_phi // 2) for k in ks])
            R = resample_half_batch(F, a.n_phi, b.n_theta, b.n_phi).reshape(len(ks), -1)
            for j, k in enumerate(ks):
                yield k, R[j]

    def l2t(self, Lf: Dict[int, np.ndarray], targets: np.ndarray) -> np.ndarray:
        lev = self.levels[self.S]
        lp = self.plan.levels[self.S]
        S = self.grid(self.S)
        # doubled-grid weight 4 pi^2 / (N_theta N_phi(theta_n)) x 2 for half storage
        w = np.concatenate([np.full(r // 2, 8 * math.pi ** 2 / (lp.n_theta * r)) for r in lp.row_nphi()])
        y = np.zeros(len(targets), dtype=np.complex128)
        box_of = self._box_of_points(targets, self.S)

        def one(a):
            sel = np.nonzero(box_of == a)[0]
            d = lev.centers[a] - self.x[targets[sel]]                            # c_a - x_i
            E = np.exp(1j * self.kappa * (d @ S.T))                              # [n, K]
            return sel, E @ (w * Lf[a])
        for sel, v in _pmap(one, np.unique(box_of), self.workers):
            y[sel] = v
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
        def one(a, sel):
            src = src_sets[a]
            ti = targets[sel]
            d = self.x[ti][:, None, :] - self.x[src][None, :, :]
            R = np.sqrt(np.sum(d * d, axis=2))
            self_pair = ti[:, None] == src[None, :]
            if np.any((R == 0) & ~self_pair):
                raise ValueError("coincident points")
            with np.errstate(divide="ignore", invalid="ignore"):
                G = np.where(self_pair, 0.0, np.exp(1j * self.kappa * R) / np.where(self_pair, 1.0, R))
            return G @ q[src]
        # bounded target chunks (the [targets x sources] matrix of one chunk stays small; enough
        # chunks to keep every worker busy)
        step = max(16, min(256, -(-len(targets) // (4 * self.workers))))
        chunks = [(a, sel[i:i + step]) for a, sel in groups.items() for i in range(0, len(sel), step)]
        for (a, sel), v in zip(chunks, _pmap(lambda c: one(*c), chunks, self.workers)):
            y[sel] = v
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

    def ancestors(self, targets: np.ndarray) -> Dict[int, list]:
        """Box indices, per level 2..D_s, of the targets' source-level boxes and their ancestors."""
        need = {self.S: sorted(set(int(b) for b in self._box_of_points(targets, self.S)))}
        for l in range(self.S, 2, -1):
            ch, pa = self.levels[l], self.levels[l - 1]
            need[l - 1] = sorted({pa.index[parent(ch.boxes[b])] for b in need[l]})
        return need

    def matvec_subset(self, q: np.ndarray, targets: np.ndarray, parts: bool = False):
        """y_i for the sampled targets only (module docstring): the full upward
        pass, then M2L / L2L restricted to the targets' ancestors, L2T and P2P for the targets."""
        q = np.asarray(q, dtype=np.complex128)
        targets = np.asarray(targets, dtype=np.int64)
        y_near = self.p2p(q, targets)
        if self.L is None:
            return (y_near, np.zeros_like(y_near)) if parts else y_near
        L, S = self.L, self.S
        need = self.ancestors(targets)
        M = {S: self.s2m(q)}
        for l in range(S, 2, -1):
            M[l - 1] = self.m2m(M[l], l)
            if l > L:
                del M[l]                         # translation-only level: no M2L partner reads it
        I = {l: self.m2l(M[l], l, targets=need[l]) for l in range(2, L + 1)}
        del M
        for l in range(L + 1, S + 1):            # translation-only levels: no M2L (R-14)
            K = self.plan.levels[l].K
            I[l] = {b: np.zeros(K, dtype=np.complex128) for b in need[l]}
        Lloc = I[2]
        for l in range(2, S):
            Lloc = self.l2l(Lloc, I[l + 1], l)
        y_far = self.l2t(Lloc, targets)
        return (y_near, y_far) if parts else y_near + y_far

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

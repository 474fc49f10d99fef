"""Direct O(N^2) sum, eqn:HelmholtzMatrixVector (TEST INFRASTRUCTURE).

sigma_i = sum_{j != i} e^{i kappa |x_i - x_j|} / |x_i - x_j| psi_j  (no 1/4pi; reading R-11)
Accumulation with math.fsum (exactly rounded sum of the rounded terms).
"""
from __future__ import annotations

import math

import numpy as np


def direct_sum(x: np.ndarray, q: np.ndarray, kappa: float, targets=None, block: int = 65536) -> np.ndarray:
    x = np.asarray(x, dtype=np.float64)
    q = np.asarray(q, dtype=np.complex128)
    if targets is None:
        targets = np.arange(len(x))
    out = np.empty(len(targets), dtype=np.complex128)
    for t, i in enumerate(targets):
        re_terms, im_terms = [], []
        for s in range(0, len(x), block):
            d = x[s:s + block] - x[i]
            R = np.sqrt(np.sum(d * d, axis=1))
            js = np.arange(s, min(s + block, len(x)))
            keep = js != i
            if np.any(R[keep] == 0.0):
                raise ValueError("coincident points")
            term = np.exp(1j * kappa * R[keep]) / R[keep] * q[js[keep]]
            re_terms.append(term.real)
            im_terms.append(term.imag)
        out[t] = complex(math.fsum(np.concatenate(re_terms)), math.fsum(np.concatenate(im_terms)))
    return out

"""Diagnostics: FMM accuracy vs direct summation on sampled targets, split into near and far parts,
for several (alpha, tau) settings.  Usage: python tools/diag_accuracy.py C5 [ntargets]"""
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np
import torch

import paper_0911_4114_b200 as hf
from workloads import CONFIGS, points_and_charges, sample_indices

name = sys.argv[1] if len(sys.argv) > 1 else "C5"
nt = int(sys.argv[2]) if len(sys.argv) > 2 else 24
cfg = CONFIGS[name]
x, q = points_and_charges(cfg)
t = sample_indices(cfg.n, nt, seed=100 + cfg.seed)


def direct(ti):
    d = x - x[ti]
    R = np.sqrt(np.sum(d * d, axis=1))
    R[ti] = 1.0
    g = np.exp(1j * cfg.kappa * R) / R
    g[ti] = 0.0
    return np.sum(g * q), R


yd = np.empty(nt, complex)
Rs = []
t0 = time.time()
for k, ti in enumerate(t):
    yd[k], R = direct(ti)
    Rs.append(R)
print("direct", time.time() - t0, flush=True)

for alpha, tau, flags in [(0.8, 0.0, 0), (0.9, 0.0, 0), (1.0, 0.0, 0), (0.8, 1e-14, 0)]:
    g = hf.HFMM(0)
    g.build_tree(x, cfg.depth, cfg.lo, cfg.size)
    g.precompute(cfg.kappa, cfg.eps, alpha, tau, flags)
    info = g.info()
    y = g.matvec(torch.from_numpy(q).cuda()).cpu().numpy()
    perm = g.debug(6)
    inv = np.empty_like(perm)
    inv[perm] = np.arange(len(perm))
    yn = g.debug(4)[inv[t]]
    L = info["L_f"]
    a = cfg.size / 2 ** L
    # exact near field: sources in neighbouring leaves at L_f
    ynx = np.empty(nt, complex)
    bx = np.minimum(np.floor((x - np.array(cfg.lo)) / a).astype(np.int64), 2 ** L - 1)
    for k, ti in enumerate(t):
        near = np.all(np.abs(bx - bx[ti]) <= 1, axis=1)
        R = Rs[k]
        gk = np.where(near, np.exp(1j * cfg.kappa * R) / R, 0)
        gk[ti] = 0
        ynx[k] = np.sum(gk * q)
    far_err = (y - g.debug(4)[inv] * 0)[t] - yn - (yd - ynx)
    rel = np.linalg.norm(y[t] - yd) / np.linalg.norm(yd)
    print(f"alpha={alpha} tau={tau} L_f={L} levels={[(l['level'], l['ell'], l['n_theta'], l['n_phi']) for l in info['levels'] if l['active']]}"
          f" relL2={rel:.3e} near_err={np.linalg.norm(yn - ynx) / np.linalg.norm(yd):.3e}"
          f" far_err={np.linalg.norm(far_err) / np.linalg.norm(yd):.3e} |far|/|y|={np.linalg.norm(yd - ynx) / np.linalg.norm(yd):.3f}"
          f" max_pt={np.max(np.abs(y[t] - yd) / np.abs(yd)):.3e}", flush=True)
    g.close()

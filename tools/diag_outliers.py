"""Diagnostics: distribution of pointwise FMM errors vs direct sum on many sampled targets,
with the target's normalised position inside its box at each active level."""
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
nt = int(sys.argv[2]) if len(sys.argv) > 2 else 200
alpha = float(sys.argv[3]) if len(sys.argv) > 3 else 0.8
cfg = CONFIGS[name]
x, q = points_and_charges(cfg)
t = sample_indices(cfg.n, nt, seed=100 + cfg.seed)
xt = torch.from_numpy(x).cuda()
qt = torch.from_numpy(q).cuda()
yd = np.empty(nt, complex)
t0 = time.time()
for k, ti in enumerate(t):           # direct sum on the GPU with torch (diagnostic only)
    d = xt - xt[ti]
    R = torch.sqrt((d * d).sum(1))
    R[ti] = 1.0
    g = torch.exp(1j * cfg.kappa * R) / R
    g[ti] = 0
    yd[k] = (g * qt).sum().item()
print("direct", time.time() - t0, flush=True)
g = hf.HFMM(0)
g.build_tree(x, cfg.depth, cfg.lo, cfg.size)
g.precompute(cfg.kappa, cfg.eps, alpha)
info = g.info()
y = g.matvec(qt).cpu().numpy()[t]
err = np.abs(y - yd) / np.abs(yd)
print("L_f", info["L_f"], [(l["level"], l["alpha"], l["ell"]) for l in info["levels"] if l["active"]], "relL2", np.linalg.norm(y - yd) / np.linalg.norm(yd), "median", np.median(err),
      "p99", np.quantile(err, 0.99), "max", err.max())
order = np.argsort(-np.abs(y - yd))
for k in order[:12]:
    pos = []
    for l in range(2, info["L_f"] + 1):
        a = cfg.size / 2 ** l
        u = (x[t[k]] - np.array(cfg.lo)) / a
        pos.append(np.round(u - np.floor(u), 2).tolist())
    print(f"abs {abs(y[k] - yd[k]):.3e} rel {err[k]:.3e} |y| {abs(yd[k]):.3e} x {np.round(x[t[k]], 4).tolist()} inbox {pos}")

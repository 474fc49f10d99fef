"""Diagnostics: run one config through the C-ABI and print per-stage buffer norms."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np
import torch

import paper_0911_4114_b200 as hf
from workloads import CONFIGS, points_and_charges

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
mode = sys.argv[2] if len(sys.argv) > 2 else "device"
cfg = CONFIGS[name]
x, q = points_and_charges(cfg)
g = hf.HFMM(0)
g.build_tree(x, cfg.depth, cfg.lo, cfg.size)
rc = g.precompute(cfg.kappa, cfg.eps, cfg.alpha)
info = g.info()
print("rc", rc, "L_f", info["L_f"], "pairs", info["p2p_pairs"], "owned", info["owned_points"])
if mode == "device":
    y = g.matvec(torch.from_numpy(q).cuda()).cpu().numpy()
else:
    y = g.matvec(q)
print("y norm", np.linalg.norm(y), "zeros", int(np.sum(y == 0)), "nan", int(np.sum(~np.isfinite(y))))
yn, yf = g.debug(4), g.debug(5)
print("y_near", np.linalg.norm(yn), "y_far", np.linalg.norm(yf) if len(yf) else None)
for l in range(2, (info["L_f"] or 1) + 1):
    for w, nm in ((0, "M"), (1, "I"), (2, "L")):
        b = g.debug(w, l)
        print(f"level {l} {nm} norm {np.linalg.norm(b):.4e} finite {np.all(np.isfinite(b))}")

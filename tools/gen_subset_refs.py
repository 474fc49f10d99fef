"""Write tests/golden/subset_<cfg>.json: oracle y at 1,000 sampled targets of a BASELINE config.

Calls only oracle/ and workloads/ (no libhfmm, no GPU): the stored values are the oracle's, so the
GPU parity test (tests/test_gpu_baseline_parity.py) compares the CUDA path against them at full size.

  python tools/gen_subset_refs.py C3 [C4 C5 C3_acc C5_acc] [--workers 8] [--count 1000]

"<cfg>_acc": the same config under the accuracy-only admissibility tau = eps / 10 ("the
quadrature target error bound can also be relaxed") instead of the default
parity-safe tau = min(eps / 10, 1e-9).

Plan: the oracle's own plan (make_plan + the R-14 source-level policy choose_source_level, the
library's default).  Targets: workloads.sample_indices(N, count, seed = 100 + config seed)
(subset seeds 102 / 103 for C4 / C5).  y_near / y_far: oracle target-subset mode
(OracleFMM.matvec_subset); y_direct: oracle.direct.direct_sum (compensated).
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

from workloads import CONFIGS, points_and_charges, sample_indices  # noqa: E402
from oracle.plan import make_plan, choose_source_level  # noqa: E402
from oracle.fmm import OracleFMM  # noqa: E402
from oracle.direct import direct_sum  # noqa: E402


def cvec(v):
    return [[float(z.real), float(z.imag)] for z in v]


def direct_threads(x, q, kappa, t, workers):
    from concurrent.futures import ThreadPoolExecutor
    parts = np.array_split(t, max(1, workers * 4))
    with ThreadPoolExecutor(workers) as ex:
        out = list(ex.map(lambda p: direct_sum(x, q, kappa, p), parts))
    return np.concatenate(out)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("configs", nargs="+")
    ap.add_argument("--workers", type=int, default=os.cpu_count() or 1)
    ap.add_argument("--count", type=int, default=1000)
    ap.add_argument("--no-direct", action="store_true")
    a = ap.parse_args()
    for name in a.configs:
        cfg = CONFIGS[name.split("_")[0]]    # "C1HF" has no suffix
        tau = cfg.eps / 10 if name.endswith("_acc") else None
        t0 = time.time()
        x, q = points_and_charges(cfg)
        plan0 = make_plan(cfg.kappa, cfg.eps, cfg.size, cfg.depth, cfg.alpha, tau=tau)
        Ds = choose_source_level(x, cfg.lo, cfg.size, cfg.depth, plan0.L_f)
        plan = make_plan(cfg.kappa, cfg.eps, cfg.size, cfg.depth, cfg.alpha, tau=tau, source_level=Ds)
        t_plan = time.time() - t0
        # every target when the config is small enough (C1HF: the whole vector)
        targets = np.arange(cfg.n) if cfg.n <= a.count * 2 else sample_indices(cfg.n, a.count, seed=100 + cfg.seed)
        f = OracleFMM(x, cfg.lo, cfg.size, plan, workers=a.workers)
        t1 = time.time()
        yn, yf = f.matvec_subset(q, targets, parts=True)
        t_fmm = time.time() - t1
        yd, t_dir = None, 0.0
        base = os.path.join(ROOT, "tests", "golden", f"subset_{cfg.name}.json")
        if name != cfg.name and os.path.exists(base):     # same targets: reuse the base config's direct sums
            with open(base) as fh:
                b = json.load(fh)
            if b["targets"] == [int(i) for i in targets] and b.get("y_direct"):
                yd = np.array([complex(u, w) for u, w in b["y_direct"]])
        if yd is None and not a.no_direct:
            t2 = time.time()
            yd = direct_threads(x, q, cfg.kappa, targets, a.workers)
            t_dir = time.time() - t2
        y = yn + yf
        levels = {str(l): dict(ell=lp.ell, n_theta=lp.n_theta, n_phi=lp.n_phi, alpha=lp.alpha, F=lp.F,
                               rep=lp.rep, active=lp.active)
                  for l, lp in plan.levels.items() if l <= plan.source_level}
        out = dict(
            what="oracle y at sampled targets (target-subset mode, SURVEY 8(d) D-4); written by "
                 "tools/gen_subset_refs.py from oracle/ only",
            config=cfg.as_dict(), L_f=plan.L_f, source_level=plan.source_level, tau=plan.tau,
            levels=levels, targets=[int(i) for i in targets], y_near=cvec(yn), y_far=cvec(yf),
            y_direct=None if yd is None else cvec(yd),
            err_vs_direct=None if yd is None else float(np.linalg.norm(y - yd) / np.linalg.norm(yd)),
            seconds=dict(plan=t_plan, fmm_subset=t_fmm, direct=t_dir, workers=a.workers))
        path = os.path.join(ROOT, "tests", "golden", f"subset_{name}.json")
        with open(path, "w") as fh:
            json.dump(out, fh, indent=0)
        print(f"{name}: L_f={plan.L_f} D_s={plan.source_level} subset {t_fmm:.1f}s direct {t_dir:.1f}s "
              f"err_vs_direct={out['err_vs_direct']} -> {path}", flush=True)


if __name__ == "__main__":
    main()

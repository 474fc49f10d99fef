#!/usr/bin/env python
"""bench.py -- FMM matvec throughput on B200 (driver contract).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C4] [--impl ours|reference]

One "step" = one full Helmholtz FMM matvec y = A q (all hot-path rows: permute, S2M, M2M,
M2L, L2L, L2T, P2P, combine) on BASELINE config 3 ("C4": N = 1e6 points on the unit sphere,
kappa = 32 pi, depth 7, eps = 1e-8, seed 2) with q resident in HBM.  `e2e` repeats the
measurement through the public host-pointer API (pinned q in, y out, copies inside the timed
region).  Multi-GPU (torchrun): strong scaling, max over ranks.

--impl reference: the CPU oracle (oracle/, plain numpy) timed on a bounded sample of the
same workload and extrapolated to one matvec (the reported baseline; not the target).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

# FP64 flops (FMA = 2) of the P2P arithmetic as implemented (DESIGN.md "Kernels and their
# rooflines"): one kernel evaluation G = e^{i kappa R}/R on positions pre-scaled to table steps
# costs 39 (difference 3, r^2 5, rsqrt Newton step 8, e^{ih R_u} from the product r^2 (1/r) 21, 1/R scaling 2; the
# MUFU.RSQ64H seed is not an FP64-pipe op); every ORDERED pair adds a complex MAC (8).  The
# symmetric kernel evaluates G once per unordered pair and applies it to both rows.
P2P_FLOPS_PER_EVAL = 39
P2P_FLOPS_PER_MAC = 8


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="C4")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ops", default="8,16,32,64",
                    help="C2 operator microbench bandwidths B (comma list; '' to skip)")
    ap.add_argument("--ragged", type=int, default=0,
                    help="1: ragged quadrature on the active levels (HFMM_RAGGED, DESIGN.md R-15)")
    ap.add_argument("--extra", default="C3,C5,C3_acc,C5_acc,C1HF",
                    help="other BASELINE matvec configs timed after the main one (comma list; '' to skip)")
    ap.add_argument("--json-out", default=None)
    ap.add_argument("--oracle-full", default=None,
                    help="time ONE full-vector oracle matvec of this config on every host core, print it, exit")
    return ap.parse_args()


# ------------------------------------------------------------------------------------------
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""

    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.rows = []
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 9:
                self.rows.append(parts)

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()
        return self.summary()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[5 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows),
                "power_w_max": max(float(r[3]) for r in self.rows) if self.rows else None}


# ------------------------------------------------------------------------------------------
def host_info():
    """Host cores and CPU model (the oracle baseline runs on this host)."""
    model = None
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except Exception:
        pass
    return {"nproc": os.cpu_count(), "cpu_model": model}


_ORACLE_CACHE = {}


def oracle_setup(cfg, x, workers):
    """The oracle's plan (with the library's default source-level policy, R-14) and tree: built
    once per process, outside every timed sample."""
    key = (cfg.name, workers)
    if key not in _ORACLE_CACHE:
        from oracle.plan import make_plan, choose_source_level, set_source_level
        from oracle.fmm import OracleFMM
        plan = make_plan(cfg.kappa, cfg.eps, cfg.size, cfg.depth, cfg.alpha)
        if plan.L_f is not None:
            set_source_level(plan, choose_source_level(x, cfg.lo, cfg.size, cfg.depth, plan.L_f))
        _ORACLE_CACHE[key] = OracleFMM(x, cfg.lo, cfg.size, plan, workers=workers)
    return _ORACLE_CACHE[key]


def oracle_sample(cfg, x, q, budget_targets: int = 2000, seed: int = 0, workers: int = None):
    """Time the CPU oracle (as it stands) on a bounded sample of one matvec, on `workers` threads
    (default: every host core; BLAS held to one thread per worker).

    Sample: P2P, S2M and L2T for `budget_targets` points of one randomly drawn far-field leaf
    (S2M of the source-level boxes holding them), M2L on 2 target boxes per active level, M2M and
    L2L on 2 children per level.  Every term is measured; the extrapolation to one matvec scales
    each by its unit count (pairs, points, interaction-list entries, children) and is reported
    separately.  Returns dict(sample_s = measured wall seconds of the sample, s_per_matvec =
    extrapolated seconds per matvec, sample = description, cores = threads used)."""
    from threadpoolctl import threadpool_limits
    from oracle.tree import interaction_list, neighbours
    workers = workers or os.cpu_count() or 1
    f = oracle_setup(cfg, x, workers)
    plan = f.plan
    rng = np.random.default_rng(seed)
    with threadpool_limits(1):
        t_all = time.perf_counter()
        if plan.L_f is None:
            t = rng.choice(len(x), size=min(len(x), budget_targets), replace=False)
            t0 = time.perf_counter()
            f.p2p(q, t)
            dt = time.perf_counter() - t0
            return {"sample_s": time.perf_counter() - t_all, "s_per_matvec": dt * len(x) / len(t),
                    "sample": f"direct sum for {len(t)} sampled targets, x{len(x) / len(t):.0f}", "cores": workers}
        L, S = plan.L_f, plan.source_level
        lev = f.levels[L]
        leaf = int(rng.integers(len(lev.boxes)))
        mem = lev.members[leaf]
        pts = np.sort(rng.choice(mem, size=min(budget_targets, len(mem)), replace=False))
        # S2M on the source-level boxes holding the sampled points (scaled by points covered)
        levS = f.levels[S]
        bS = np.minimum(np.floor((x[pts] - np.asarray(cfg.lo)) / levS.a).astype(np.int64), 2 ** S - 1)
        sbox = sorted({levS.index[tuple(c)] for c in bS.tolist()})
        covered = sum(len(levS.members[b]) for b in sbox)
        t0 = time.perf_counter()
        f.s2m(q, boxes=sbox)
        ts2m = (time.perf_counter() - t0) * len(x) / covered
        # P2P (scaled by ordered pairs)
        nsrc = sum(len(lev.members[c]) for c in neighbours(lev, lev.boxes[leaf]))
        pairs_all = sum(len(lev.members[b]) * sum(len(lev.members[c]) for c in neighbours(lev, lev.boxes[b]))
                        for b in range(len(lev.boxes)))
        t0 = time.perf_counter()
        f.p2p(q, pts)
        tp2p = (time.perf_counter() - t0) * pairs_all / (len(pts) * nsrc)
        # L2T with a random local field (scaled by points)
        Kf = plan.levels[S].K
        Lf = {b: rng.standard_normal(Kf) + 1j * rng.standard_normal(Kf) for b in sbox}
        t0 = time.perf_counter()
        f.l2t(Lf, pts)
        tl2t = (time.perf_counter() - t0) * len(x) / len(pts)
        # M2M / M2L / L2L per level with random fields
        tmid = 0.0
        for l in range(2, S + 1):
            K = plan.levels[l].K
            levl = f.levels[l]
            nb = len(levl.boxes)
            sub = list(range(min(2, nb)))
            M = {b: rng.standard_normal(K) + 1j * rng.standard_normal(K) for b in sub}
            if l <= L:
                Mall = {b: rng.standard_normal(K) + 1j * rng.standard_normal(K) for b in range(nb)}
                nnz_s = sum(len(interaction_list(levl, levl.boxes[a])) for a in sub)
                nnz = sum(len(interaction_list(levl, levl.boxes[a])) for a in range(nb))
                for a in sub:                      # tables are precompute (untimed in the GPU path too)
                    for _, o in interaction_list(levl, levl.boxes[a]):
                        f.table(l, o)
                t0 = time.perf_counter()
                f.m2l(Mall, l, targets=sub)
                tmid += (time.perf_counter() - t0) * nnz / max(nnz_s, 1)
            if l > 2:
                t0 = time.perf_counter()
                f.m2m(M, l)
                tmid += (time.perf_counter() - t0) * nb / len(sub)
                Kp = plan.levels[l - 1].K
                pa = sorted({f.levels[l - 1].index[(c[0] // 2, c[1] // 2, c[2] // 2)] for c in (levl.boxes[b] for b in sub)})
                Lp = {p: rng.standard_normal(Kp) + 1j * rng.standard_normal(Kp) for p in pa}
                t0 = time.perf_counter()
                f.l2l(Lp, M, l - 1)
                tmid += (time.perf_counter() - t0) * nb / len(sub)
        sample_s = time.perf_counter() - t_all
    desc = (f"oracle on {workers} threads: P2P, S2M and L2T for {len(pts)} points of 1 of {len(lev.boxes)} far-field "
            f"leaves (S2M/L2T at source level {S}, P2P at L_f={L}), M2L on 2 boxes/level, M2M+L2L on 2 "
            f"children/level; measured {sample_s:.2f} s, extrapolated to one matvec by unit counts")
    return {"sample_s": sample_s, "s_per_matvec": ts2m + tp2p + tl2t + tmid, "sample": desc, "cores": workers,
            "terms_s_per_matvec": {"s2m": ts2m, "p2p": tp2p, "l2t": tl2t, "m2m_m2l_l2l": tmid}}


def golden_parity(name, y, info):
    """y of a timed matvec vs the oracle's stored target-subset values (tests/golden/subset_<name>.json,
    written by tools/gen_subset_refs.py from oracle/ only): relative L2 over the sampled targets, and
    the error vs the stored direct sums.  Reads stored numbers only (no oracle code runs here)."""
    path = os.path.join(ROOT, "tests", "golden", f"subset_{name}.json")
    if not os.path.exists(path):
        return {"available": False}
    d = json.load(open(path))
    if (d["L_f"], d["source_level"]) != (info["L_f"], info["source_level"]):
        return {"available": False, "why": "plan differs from the stored reference's"}
    t = np.array(d["targets"])
    c = lambda v: np.array([complex(a, b) for a, b in v])
    yo = c(d["y_near"]) + c(d["y_far"])
    out = {"available": True, "targets": len(t), "rel_l2_vs_oracle": float(np.linalg.norm(y[t] - yo) / np.linalg.norm(yo)),
           "bar": 1e-11, "max_F_active": max((v["F"] for v in d["levels"].values() if v["active"]), default=None)}
    if d.get("y_direct"):
        yd = c(d["y_direct"])
        out["err_vs_direct"] = float(np.linalg.norm(y[t] - yd) / np.linalg.norm(yd))
        out["eps"] = d["config"]["eps"]
    return out


def c1_breakdown():
    """P:833 low-frequency breakdown demonstration on C1 (SURVEY D-1): the policy run (no admissible
    level: the direct sum) vs every level forced active (HFMM_FORCE_ALL_LEVELS), errors vs the GPU
    direct sum (hfmm_direct) next to each level's roundoff amplification F_l."""
    import torch
    import paper_0911_4114_b200 as hf
    from workloads import CONFIGS, points_and_charges
    cfg = CONFIGS["C1"]
    x, q = points_and_charges(cfg)
    qd = torch.from_numpy(q).cuda()
    out = {"eps": cfg.eps}
    for name, flags in (("policy", 0), ("forced", hf.HFMM_FORCE_ALL_LEVELS)):
        g = hf.HFMM(0)
        g.build_tree(x, cfg.depth, cfg.lo, cfg.size)
        g.precompute(cfg.kappa, cfg.eps, cfg.alpha, flags=flags)
        y = g.matvec(qd)
        yd = g.direct(qd)
        info = g.info()
        out[name] = {"L_f": info["L_f"], "F": {lv["level"]: lv["F"] for lv in info["levels"] if lv["active"]},
                     "err_vs_direct": float(torch.linalg.norm(y - yd) / torch.linalg.norm(yd))}
        g.close()
    return out


def hbm_peak():
    """Measured HBM copy bandwidth (GB/s) from MEASURED_PEAKS.json, else the guide's fallback."""
    try:
        return float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]), "MEASURED_PEAKS.json"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def bench_operators(bandwidths, reps: int = 5, fp64_peak_tflops: float = 37.2):
    """BASELINE.json configs[1] ("C2"): operator microbench on 65,536 boxes of random complex128 fields.

    Child grid (2B, 2B) -> parent (4B, 4B), half storage [N_theta][N_phi/2] (SURVEY D-1):
      interp  65,536 x R_{2B->4B} out of place          anterp  65,536 x R_{4B->2B}
      m2m     8,192 parents x 8 children, shift + sum    l2l     8,192 parents -> 8 children, conj shift, +I
      m2l     65,536 targets x 189 partners (periodic 64x32x32 lattice, Morton order), 316 tables
    Algorithmic bytes: every input read once and every output written once (tables once).
    Times: CUDA events on the launching stream, mean of `reps` after one warm-up, L2 flushed between."""
    import torch
    import paper_0911_4114_b200 as hf
    from workloads import MICROBENCH, c2_lattice, c2_grids
    peak, src = hbm_peak()
    nbox = MICROBENCH["boxes"]
    _, row, srcs, oid, _ = c2_lattice()
    flush = torch.empty(512 * 1024 * 1024, dtype=torch.uint8, device="cuda")
    stream = torch.cuda.current_stream()
    out = {"hbm_peak_gbs": peak, "hbm_peak_source": src, "boxes": nbox, "fp64_peak_tflops": fp64_peak_tflops}
    gen = torch.Generator(device="cuda")
    gen.manual_seed(MICROBENCH["seed"])

    def crandn(*shape):
        return torch.randn(*shape, 2, dtype=torch.float64, device="cuda", generator=gen).view(torch.complex128)[..., 0]

    def timed(fn):
        fn()
        ms = []
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for _ in range(reps):
            flush.zero_()
            torch.cuda.synchronize()
            e0.record(stream)
            fn()
            e1.record(stream)
            torch.cuda.synchronize()
            ms.append(e0.elapsed_time(e1))
        return statistics.mean(ms)

    for B in bandwidths:
        (nth, nph), (nth2, nph2) = c2_grids(B)
        K, K2 = nth * nph // 2, nth2 * nph2 // 2
        npar = nbox // 8
        child = crandn(nbox, K)
        parent = torch.empty(nbox, K2, dtype=torch.complex128, device="cuda")
        res = {}

        def rec(name, ms, nbytes, flops=None):
            d = {"ms": ms, "gbs": nbytes / ms / 1e6, "frac_hbm": nbytes / ms / 1e6 / peak, "bytes": nbytes}
            if flops is not None:
                d["tflops"] = flops / ms / 1e9
                d["frac_fp64"] = d["tflops"] / fp64_peak_tflops
            res[name] = d

        ws = max(hf.resample_workspace(nbox, nth, nph, nth2, nph2), hf.resample_workspace(nbox, nth2, nph2, nth, nph))
        work = torch.empty(max(ws, 16), dtype=torch.uint8, device="cuda") if ws > 0 else None
        rec("interp", timed(lambda: hf.resample(child, nth, nph, nth2, nph2, parent, work=work)), nbox * (K + K2) * 16)
        child2 = torch.empty_like(child)
        rec("anterp", timed(lambda: hf.resample(parent, nth2, nph2, nth, nph, child2, work=work)), nbox * (K + K2) * 16)
        shift = torch.polar(torch.ones(8, K2, dtype=torch.float64, device="cuda"),
                            2 * math.pi * torch.rand(8, K2, dtype=torch.float64, device="cuda", generator=gen))
        par = parent[:npar]
        rec("m2m", timed(lambda: hf.m2m_op(child, shift, par, nth, nph, nth2, nph2, work=work)),
            (nbox * K + npar * K2 + 8 * K2) * 16)
        inc = crandn(nbox, K)
        rec("l2l", timed(lambda: hf.l2l_op(par, shift, inc, child2, nth2, nph2, nth, nph, work=work)),
            (npar * K2 + 2 * nbox * K + 8 * K2) * 16)
        del inc, parent, par, work
        T = crandn(316, K)
        op = hf.M2LOp(row, srcs, oid, K)           # sibling-group plan, built once per K
        rec("m2l", timed(lambda: op.apply(T, child, child2)),
            (2 * nbox * K + 316 * K) * 16, flops=8.0 * int(row[-1]) * K)
        out[f"B{B}"] = res
        op.close()
        del child, child2, T, shift
        torch.cuda.empty_cache()
    return out


def bench_matvec_config(cfg, warmup: int, steps: int, tau: float = 0.0, golden: str = None):
    """One more BASELINE matvec config on this GPU (context for the main line): ms per matvec with
    q resident, L2 flushed between steps, CUDA events on the launching stream."""
    import torch
    import paper_0911_4114_b200 as hf
    from workloads import points_and_charges
    x, q = points_and_charges(cfg)
    g = hf.HFMM(0)
    g.build_tree(x, cfg.depth, cfg.lo, cfg.size)
    g.precompute(cfg.kappa, cfg.eps, cfg.alpha, tau=tau)
    info = g.info()
    qd = torch.from_numpy(q).cuda()
    yd = torch.empty_like(qd)
    flush = torch.empty(512 * 1024 * 1024, dtype=torch.uint8, device="cuda")
    stream = torch.cuda.current_stream()
    for _ in range(warmup):
        g.matvec(qd, out=yd)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ms = []
    for _ in range(steps):
        flush.zero_()
        torch.cuda.synchronize()
        e0.record(stream)
        g.matvec(qd, out=yd)
        e1.record(stream)
        torch.cuda.synchronize()
        ms.append(e0.elapsed_time(e1))
    t = statistics.mean(ms)
    out = {"n": cfg.n, "kappa": cfg.kappa, "depth": cfg.depth, "eps": cfg.eps, "geometry": cfg.kind, "tau": info["tau"],
           "L_f": info["L_f"], "source_level": info["source_level"], "ms_per_matvec": t, "matvec_per_s": 1e3 / t,
           "mpoints_per_s": cfg.n / t / 1e3, "p2p_pairs": info["p2p_pairs"], "steps": steps,
           "p2p_tile": info["p2p_tile"], "p2p_rowskip": info["p2p_rowskip"], "p2p_dead_frac": info["p2p_dead_frac"],
           "p2p_mixed_items": info["p2p_mixed_items"],
           "parity": golden_parity(golden or cfg.name, yd.cpu().numpy(), info)}
    g.close()
    del qd, yd, flush
    torch.cuda.empty_cache()
    return out


def oracle_full(name):
    """One full-vector oracle matvec (every target) on every host core: the measured counterpart of
    the sampled cpu_baseline (its extrapolation is printed beside it for the same config)."""
    from threadpoolctl import threadpool_limits
    from workloads import CONFIGS, points_and_charges
    cfg = CONFIGS[name]
    x, q = points_and_charges(cfg)
    workers = os.cpu_count() or 1
    t0 = time.perf_counter()
    f = oracle_setup(cfg, x, workers)
    t_setup = time.perf_counter() - t0
    with threadpool_limits(1):
        t0 = time.perf_counter()
        y = f.matvec(q)
        t_full = time.perf_counter() - t0
    samp = oracle_sample(cfg, x, q, budget_targets=3000, workers=workers)
    out = {"oracle_full_matvec": name, "n": cfg.n, "seconds": t_full, "setup_s": t_setup, "cores": workers,
           "host": host_info(), "sampled_extrapolation_s": samp["s_per_matvec"], "sample": samp["sample"]}
    path = os.path.join(ROOT, "tests", "golden", f"subset_{name}.json")
    if os.path.exists(path):                  # consistency with the stored target-subset reference
        d = json.load(open(path))
        t = np.array(d["targets"])
        yo = np.array([complex(a, b) for a, b in d["y_near"]]) + np.array([complex(a, b) for a, b in d["y_far"]])
        out["rel_l2_vs_subset_reference"] = float(np.linalg.norm(y[t] - yo) / np.linalg.norm(yo))
    print(json.dumps(out), flush=True)


def workload_config(cfg, world):
    """The `config` object of both arms' JSON lines (identical keys, so the driver can pair them)."""
    return {"workload": cfg.name, "n": cfg.n, "kappa": cfg.kappa, "depth": cfg.depth, "eps": cfg.eps,
            "seed": cfg.seed, "geometry": cfg.kind, "l2": "flushed (512 MB write) between steps",
            "parallelism": f"octree level-2 subtrees x{world}"}


def run_reference(args, cfg, rank, world):
    """--impl reference: the CPU oracle on every host core, each step a bounded measured sample
    (ms_per_step = its measured wall time); value = matvec/s from the unit-count extrapolation,
    which is reported separately (extrapolated_s_per_matvec).  Rank 0 only."""
    if rank != 0:
        return
    from workloads import points_and_charges
    x, q = points_and_charges(cfg)
    workers = os.cpu_count() or 1
    oracle_setup(cfg, x, workers)                       # plan + tree: untimed setup
    for k in range(args.warmup):
        oracle_sample(cfg, x, q, budget_targets=REF_TARGETS, seed=1000 + k, workers=workers)
    samples = [oracle_sample(cfg, x, q, budget_targets=REF_TARGETS, seed=k, workers=workers)
               for k in range(args.steps)]
    t_meas = statistics.mean(r["sample_s"] for r in samples)
    t_mv = statistics.mean(r["s_per_matvec"] for r in samples)
    line = {"metric": "FMM matvecs/s", "value": 1.0 / t_mv, "unit": "matvec/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * t_meas, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": workload_config(cfg, world), "impl": "reference",
            "extrapolated_s_per_matvec": t_mv,
            "note": "ms_per_step is the measured wall time of one step's sample; value extrapolates the sample "
                    "to one whole matvec by unit counts (extrapolated_s_per_matvec)",
            "host": host_info(),
            "cpu_baseline": {"value": 1.0 / t_mv, "unit": "matvec/s", "cores": workers, "kind": "oracle",
                             "sample": samples[-1]["sample"]},
            "e2e": {"value": 1.0 / t_mv, "unit": "matvec/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


REF_TARGETS = 600      # points per reference-arm step (a few seconds of oracle work on 8 cores)


def relaunch_under_torchrun(args):
    """`bench.py --gpus N` without a torchrun environment: re-exec this script as N ranks
    (one process per GPU) on 127.0.0.1, exactly as the driver's own torchrun launch would."""
    import socket
    import torch
    ngpu = torch.cuda.device_count()
    if ngpu < args.gpus:
        print(json.dumps({"error": f"--gpus {args.gpus} but only {ngpu} visible CUDA device(s)"}), flush=True)
        sys.exit(2)
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    sys.exit(subprocess.call(cmd))


# ------------------------------------------------------------------------------------------
def main():
    args = parse()
    if args.oracle_full:
        oracle_full(args.oracle_full)
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        relaunch_under_torchrun(args)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    from workloads import CONFIGS, points_and_charges
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        run_reference(args, cfg, rank, world)
        return
    os.environ["HFMM_PROFILE_STAGES"] = "1"
    import torch
    import paper_0911_4114_b200 as hf
    from paper_0911_4114_b200.build import build
    if rank == 0:
        build(verbose=False)
    torch.cuda.set_device(local_rank)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        dist.barrier()
    x, q = points_and_charges(cfg)
    g = hf.HFMM(local_rank)
    if world > 1:
        uid = hf.nccl_unique_id() if rank == 0 else bytes(128)
        t = torch.tensor(list(uid), dtype=torch.uint8, device="cuda")
        dist.broadcast(t, 0)
        g.set_dist(rank, world, bytes(t.cpu().tolist()))
    t0 = time.perf_counter()
    g.build_tree(x, cfg.depth, cfg.lo, cfg.size)
    t_tree = time.perf_counter() - t0
    t0 = time.perf_counter()
    pflags = hf.HFMM_RAGGED if args.ragged else 0
    g.precompute(cfg.kappa, cfg.eps, cfg.alpha, flags=pflags)
    t_pre = time.perf_counter() - t0
    info = g.info()
    stream = torch.cuda.current_stream()
    qd = torch.from_numpy(q).cuda()
    yd = torch.empty_like(qd)
    flush = torch.empty(512 * 1024 * 1024, dtype=torch.uint8, device="cuda")   # > 126 MB L2
    local = world > 1
    for _ in range(args.warmup):
        g.matvec(qd, out=yd, local=local)
    torch.cuda.synchronize()
    sampler = ClockSampler(local_rank)
    sampler.start()
    step_ms, stage = [], {k: [] for k in ("s2m", "m2m", "m2l", "l2l", "l2t", "p2p")}
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(args.steps):
        flush.zero_()                      # L2 flush between timed iterations (untimed)
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        e0.record(stream)
        g.matvec(qd, out=yd, local=local)
        e1.record(stream)
        torch.cuda.synchronize()
        step_ms.append(e0.elapsed_time(e1))
        st = g.stage_times()
        for k in stage:
            stage[k].append(st[k])
    clocks = sampler.stop()
    # the same matvec with the near field and the far chain one after the other (HFMM_SERIAL):
    # P2P launch durations without the far-chain CTAs sharing the SMs (untimed for `value`)
    p2p_serial = []
    for _ in range(max(2, args.steps // 2)):
        flush.zero_()
        torch.cuda.synchronize()
        g.matvec(qd, out=yd, local=local, serial=True)
        torch.cuda.synchronize()
        p2p_serial.append(g.stage_times()["p2p"])
    tot = torch.tensor([sum(step_ms)], dtype=torch.float64, device="cuda")
    if dist:
        dist.all_reduce(tot, op=dist.ReduceOp.MAX)
    ms = tot.item() / args.steps
    # end to end through the public host-pointer API (pinned host q, y; copies timed)
    qh = torch.from_numpy(q).pin_memory()
    yh = torch.empty_like(qh).pin_memory()
    e2e_ms = []
    for _ in range(max(2, args.steps // 2)):
        flush.zero_()
        if dist:
            dist.barrier()
        torch.cuda.synchronize()
        e0.record(stream)
        g.matvec(qh, out=yh, stream=stream.cuda_stream)
        e1.record(stream)
        torch.cuda.synchronize()
        e2e_ms.append(e0.elapsed_time(e1))
    te = torch.tensor([statistics.mean(e2e_ms)], dtype=torch.float64, device="cuda")
    if dist:
        dist.all_reduce(te, op=dist.ReduceOp.MAX)
    # P2P roofline (dominant kernel): algorithmic FP64 flops / measured duration
    p2p_ms = statistics.mean(stage["p2p"])
    p2p_ms_serial = statistics.mean(p2p_serial)
    pairs = info["p2p_pairs"]
    sym = info["p2p_sym_pairs"]
    evals = sym + (pairs - 2 * sym)          # unordered (symmetric) + ordered (diagonal) evaluations
    p2p_flops = P2P_FLOPS_PER_EVAL * evals + P2P_FLOPS_PER_MAC * pairs
    peak_tflops = 2 * 64 * 148 * (clocks.get("sm_max_mhz") or 1965.0) * 1e6 / 1e12
    achieved = p2p_flops / (p2p_ms * 1e-3) / 1e12
    traffic = traffic_scope = None
    tpath = os.path.join(ROOT, "profiles", "traffic.json")
    if os.path.exists(tpath):
        try:
            tj = json.load(open(tpath)).get(cfg.name, {})
            traffic, traffic_scope = tj.get("p2p"), tj.get("p2p_scope")
        except Exception:
            traffic = traffic_scope = None
    L_f = info["L_f"]
    launches = info["launches"]                  # counted by libhfmm for one matvec (hfmm_info.launches)
    line = {
        "metric": "FMM matvecs/s", "value": 1e3 / ms, "unit": "matvec/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": workload_config(cfg, world),
        "mpoints_per_s": cfg.n * 1e3 / ms / 1e6,
        "e2e": {"value": 1e3 / te.item(), "unit": "matvec/s", "h2d_bytes_per_step": cfg.n * 16,
                "d2h_bytes_per_step": cfg.n * 16,
                "note": "hfmm_matvec with pinned host q / y: H2D, the matvec, the y gather across ranks "
                        "(all-gather of the owned sorted ranges) and the D2H inside the timed region"},
        "gpu_launches": launches,
        "roofline": {"kernel": "p2p", "bound": "alu", "achieved": achieved, "peak": peak_tflops, "unit": "TFLOP/s",
                     "frac": achieved / peak_tflops, "traffic": traffic, "traffic_scope": traffic_scope,
                     "peak_source": "derived: 64 FP64 FMA/clk/SM x 148 SMs x 2 x sm_max_mhz (DESIGN.md)",
                     "per_unit": f"{P2P_FLOPS_PER_EVAL} FP64 flops per kernel evaluation + "
                                 f"{P2P_FLOPS_PER_MAC} per ordered pair (MAC)",
                     "units_per_launch": {"ordered_pairs": pairs, "evaluations": evals},
                     "launch_ms": p2p_ms,
                     "achieved_serial": p2p_flops / (p2p_ms_serial * 1e-3) / 1e12,
                     "frac_serial": p2p_flops / (p2p_ms_serial * 1e-3) / 1e12 / peak_tflops,
                     "launch_ms_serial": p2p_ms_serial,
                     "note": "achieved: P2P launches timed on their stream inside the timed steps, sharing the "
                             "SMs with the high-priority far-field chain; *_serial: the same launches in "
                             "matvecs run with HFMM_SERIAL (near field first, then the far chain)",
                     "flops_per_launch": p2p_flops,
                     "measured_dfma_peak_tflops": 34.2},
        "stages_ms": {k: statistics.mean(v) for k, v in stage.items()},
        "plan": {"L_f": L_f, "source_level": info["source_level"],
                 "levels": [{k: lv[k] for k in ("level", "ell", "n_theta", "n_phi", "F", "active")}
                            for lv in info["levels"]], "p2p_pairs": pairs, "s2m_evals": info["s2m_evals"],
                 "p2p_tile": info["p2p_tile"], "p2p_rowskip": info["p2p_rowskip"],
                 "p2p_dead_frac": info["p2p_dead_frac"], "p2p_mixed_items": info["p2p_mixed_items"]},
        "setup_s": {"build_tree": t_tree, "precompute": t_pre},
        "clocks": clocks,
    }
    if world == 1:
        line["parity"] = golden_parity(cfg.name, yd.cpu().numpy(), info)
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        r = oracle_sample(cfg, x, q, budget_targets=3000)
        line["cpu_baseline"] = {"value": 1.0 / r["s_per_matvec"], "unit": "matvec/s", "cores": r["cores"],
                                "kind": "oracle", "sample": r["sample"], "sample_s": r["sample_s"],
                                "extrapolated_s_per_matvec": r["s_per_matvec"], "terms_s_per_matvec": r["terms_s_per_matvec"],
                                "host": host_info()}
    if world == 1 and (args.ops or args.extra):
        g.close()
        del qd, yd, flush, qh, yh
        torch.cuda.empty_cache()
    if world == 1 and args.extra:
        oc = {}
        for name in args.extra.split(","):
            base = name.split("_")[0]
            if not name or name == cfg.name or base not in CONFIGS:
                continue
            # "<cfg>_acc": the accuracy-only admissibility tau = eps / 10
            tau = CONFIGS[base].eps / 10 if name.endswith("_acc") else 0.0
            oc[name] = bench_matvec_config(CONFIGS[base], args.warmup, max(3, args.steps // 2), tau=tau, golden=name)
        line["other_configs"] = oc
    if world == 1 and args.extra:
        line["C1_breakdown"] = c1_breakdown()
    if world == 1 and args.ops:
        line["operators"] = bench_operators([int(b) for b in args.ops.split(",")], fp64_peak_tflops=peak_tflops)
    if rank == 0:
        print(json.dumps(line), flush=True)
        if args.json_out:
            json.dump(line, open(args.json_out, "w"), indent=1)
    if dist:
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

"""Seeded synthetic inputs shared by the oracle, the tests and bench.py.

This module holds NO arithmetic of the method (no kernel, no quadrature, no
tree): only the configuration table and the random-number recipe, so that the
CUDA path and the CPU oracle can be fed identical inputs without sharing any
of the method's code (task rule: "only the seeded input generators serve
both").

Recipe:
  rng = numpy.random.default_rng(seed)   (PCG64)
  sphere:  v = rng.standard_normal((N, 3)); x = v / |v|      (uniform on S^2)
  cube:    x = rng.uniform(0, 1, (N, 3))
  charges: q = rng.standard_normal(N) + 1j * rng.standard_normal(N)
           (drawn after x from the same generator, real part first)

The paper's own workloads are synthetic too: random points in a cube with
kappa scaled as N^(1/3) (Sec. "Speed") and two-point rigs
(l.831, l.981).  BASELINE.json's configs are reproduced below; "C1HF" is the
survey's added config where every far-field level is
admissible.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field, asdict
from typing import Tuple

import numpy as np


@dataclass(frozen=True)
class Config:
    name: str
    kind: str            # "sphere" | "cube"
    n: int
    kappa: float
    depth: int
    eps: float
    seed: int
    lo: Tuple[float, float, float]
    size: float
    alpha: float = 0.8
    note: str = ""

    def as_dict(self):
        d = asdict(self)
        d["lo"] = list(self.lo)
        return d


SPHERE_ROOT = ((-1.0, -1.0, -1.0), 2.0)   # tight cube around the unit sphere (A-18)
CUBE_ROOT = ((0.0, 0.0, 0.0), 1.0)

CONFIGS = {
    # BASELINE.json configs[0]
    "C1": Config("C1", "sphere", 2000, 2 * math.pi, 3, 1e-4, 0, *SPHERE_ROOT,
                 note="N=2,000 unit sphere, kappa=2pi, depth 3, eps=1e-4, seed 0"),
    # survey addition: same points, every level admissible
    "C1HF": Config("C1HF", "sphere", 2000, 64 * math.pi, 4, 1e-4, 0, *SPHERE_ROOT,
                   note="C1 points, kappa=64pi, depth 4, eps=1e-4 (SURVEY F7)"),
    # BASELINE.json configs[2]
    "C3": Config("C3", "sphere", 100_000, 16 * math.pi, 6, 1e-6, 1, *SPHERE_ROOT,
                 note="N=1e5 unit sphere, kappa=16pi, depth 6, eps=1e-6, seed 1"),
    # BASELINE.json configs[3]
    "C4": Config("C4", "sphere", 1_000_000, 32 * math.pi, 7, 1e-8, 2, *SPHERE_ROOT,
                 note="N=1e6 unit sphere, kappa=32pi, depth 7, eps=1e-8, seed 2"),
    # BASELINE.json configs[4]: cube edge = 64 wavelengths -> kappa = 128 pi (A-26)
    "C5": Config("C5", "cube", 10_000_000, 128 * math.pi, 8, 1e-6, 3, *CUBE_ROOT,
                 note="N=1e7 unit cube, kappa=128pi (64 lambda edge), depth 8, eps=1e-6, seed 3"),
}

# BASELINE.json configs[1]: operator microbench (65,536 boxes, child bandwidth B)
MICROBENCH = dict(boxes=65536, lattice=(64, 32, 32), bandwidths=(8, 16, 32, 64), seed=4)


def small_config(name: str, *, kind: str = "sphere", n: int = 600, kappa: float = 32 * math.pi,
                 depth: int = 3, eps: float = 1e-6, seed: int = 11, alpha: float = 0.8) -> Config:
    """A reduced config the oracle finishes in seconds (parity-test sizes)."""
    root = SPHERE_ROOT if kind == "sphere" else CUBE_ROOT
    return Config(name, kind, n, kappa, depth, eps, seed, *root, alpha=alpha)


def points(cfg: Config) -> np.ndarray:
    """(N, 3) float64 positions, C-contiguous."""
    rng = np.random.default_rng(cfg.seed)
    if cfg.kind == "sphere":
        v = rng.standard_normal((cfg.n, 3))
        x = v / np.linalg.norm(v, axis=1, keepdims=True)
    elif cfg.kind == "cube":
        x = rng.uniform(0.0, 1.0, (cfg.n, 3))
    else:
        raise ValueError(cfg.kind)
    return np.ascontiguousarray(x, dtype=np.float64)


def points_and_charges(cfg: Config):
    """Positions and complex128 charges from ONE generator (positions first)."""
    rng = np.random.default_rng(cfg.seed)
    if cfg.kind == "sphere":
        v = rng.standard_normal((cfg.n, 3))
        x = v / np.linalg.norm(v, axis=1, keepdims=True)
    else:
        x = rng.uniform(0.0, 1.0, (cfg.n, 3))
    re = rng.standard_normal(cfg.n)
    im = rng.standard_normal(cfg.n)
    q = re + 1j * im
    return np.ascontiguousarray(x, dtype=np.float64), np.ascontiguousarray(q, dtype=np.complex128)


def random_charges(n: int, seed: int) -> np.ndarray:
    rng = np.random.default_rng(seed)
    return rng.standard_normal(n) + 1j * rng.standard_normal(n)


def sample_indices(n: int, count: int, seed: int) -> np.ndarray:
    """Seeded target subset (for full-size checks), sorted, unique."""
    rng = np.random.default_rng(seed)
    count = min(count, n)
    return np.sort(rng.choice(n, size=count, replace=False))


def microbench_fields(nbox: int, nth: int, nph_half: int, seed: int) -> np.ndarray:
    """Random complex128 N(0,1) spherical fields [nbox][nth][nph_half]."""
    rng = np.random.default_rng(seed)
    re = rng.standard_normal((nbox, nth, nph_half))
    im = rng.standard_normal((nbox, nth, nph_half))
    return re + 1j * im


# ---------------------------------------------------------------------------------------------
# BASELINE.json configs[1] (operator microbench, "C2"): a periodic 64 x 32 x 32 lattice of boxes
# at one level, boxes numbered in Morton order.  The interaction list of every box has exactly 189
# entries on a periodic lattice (not a neighbour, parent is a neighbour of the parent;
# 189).  This is the *input* of the M2L operator entry point (a CSR it takes as
# arguments); the oracle-side test checks it against oracle/tree.py's own rule on sampled boxes.
# Offset ids: lexicographic (x, then y, then z) over [-3,3]^3 minus [-1,1]^3 (316 offsets).
def _spread3(v: np.ndarray) -> np.ndarray:
    out = np.zeros_like(v, dtype=np.int64)
    for bit in range(10):
        out |= ((v >> bit) & 1) << (3 * bit)
    return out


def c2_lattice(dims=MICROBENCH["lattice"]):
    """Box coordinates [nbox, 3] (Morton order) and the periodic interaction CSR (row, src, oid)."""
    nx, ny, nz = dims
    g = np.stack(np.meshgrid(np.arange(nx), np.arange(ny), np.arange(nz), indexing="ij"), -1).reshape(-1, 3)
    key = (_spread3(g[:, 0]) << 2) | (_spread3(g[:, 1]) << 1) | _spread3(g[:, 2])
    g = g[np.argsort(key, kind="stable")]
    lin = np.empty(nx * ny * nz, dtype=np.int64)                 # (x, y, z) -> Morton position
    lin[(g[:, 0] * ny + g[:, 1]) * nz + g[:, 2]] = np.arange(len(g))
    offs = np.array([(a, b, c) for a in range(-3, 4) for b in range(-3, 4) for c in range(-3, 4)
                     if max(abs(a), abs(b), abs(c)) >= 2], dtype=np.int64)        # 316, lexicographic
    tgt = g[:, None, :]                                                           # [nbox, 1, 3]
    src = tgt + offs[None, :, :]                                                  # unwrapped
    ok = np.all(np.abs((src >> 1) - (tgt >> 1)) <= 1, axis=2)                     # parents adjacent
    dimv = np.array(dims)
    w = src % dimv
    sidx = lin[(w[..., 0] * ny + w[..., 1]) * nz + w[..., 2]]
    oid = np.broadcast_to(np.arange(len(offs)), ok.shape)
    counts = ok.sum(axis=1)
    row = np.concatenate([[0], np.cumsum(counts)]).astype(np.int32)
    return g, row, sidx[ok].astype(np.int32), oid[ok].astype(np.int32), offs


def c2_grids(B: int):
    """Child grid (N_theta, N_phi) = (2B, 2B) and parent grid (4B, 4B) of bandwidth B (SURVEY D-1)."""
    return (2 * B, 2 * B), (4 * B, 4 * B)

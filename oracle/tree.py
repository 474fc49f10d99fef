"""Octree, neighbour and interaction lists (TEST INFRASTRUCTURE; see oracle/__init__.py).

P:33    root level 0, box size a_l = a_0 / 2^l, highest active level l = 2
P:114   box B^l_alpha of level l with centre c^l_alpha
P:127   interaction list I(B): same-level boxes that are not neighbours of B but
        whose parent is a neighbour of B's parent
P:138   neighbour list N(B): B and all boxes touching it
Reading R-8: integer box coordinate b = min(floor((x - lo)/a_l), 2^l - 1)
per axis; empty boxes pruned; "neighbour" = Chebyshev distance <= 1.
Plain per-level dictionaries keyed by integer box coordinates.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Dict, List, Tuple

import numpy as np


@dataclass
class Level:
    level: int
    a: float
    boxes: List[Tuple[int, int, int]]          # occupied box coords (sorted)
    index: Dict[Tuple[int, int, int], int]     # coord -> position in boxes
    members: List[np.ndarray]                  # point indices per box
    centers: np.ndarray                        # [nbox, 3]


def box_coords(x: np.ndarray, lo, a0: float, level: int) -> np.ndarray:
    n = 2 ** level
    a = a0 / n
    b = np.floor((x - np.asarray(lo)) / a).astype(np.int64)
    if np.any(b < 0) or np.any(b > n):
        raise ValueError("point outside the root cube")
    return np.minimum(b, n - 1)


def build_level(x: np.ndarray, lo, a0: float, level: int) -> Level:
    b = box_coords(x, lo, a0, level)
    groups: Dict[Tuple[int, int, int], list] = {}
    for i, key in enumerate(map(tuple, b)):
        groups.setdefault(key, []).append(i)
    boxes = sorted(groups)
    a = a0 / 2 ** level
    centers = np.array([[lo[d] + (c[d] + 0.5) * a for d in range(3)] for c in boxes])
    return Level(level, a, boxes, {c: k for k, c in enumerate(boxes)},
                 [np.array(groups[c], dtype=np.int64) for c in boxes], centers)


def cheb(u, v) -> int:
    return max(abs(u[0] - v[0]), abs(u[1] - v[1]), abs(u[2] - v[2]))


def parent(c):
    return (c[0] // 2, c[1] // 2, c[2] // 2)


def neighbours(lev: Level, c) -> List[int]:
    """N(B): occupied boxes at Chebyshev distance <= 1, including B."""
    out = []
    for dx in (-1, 0, 1):
        for dy in (-1, 0, 1):
            for dz in (-1, 0, 1):
                k = lev.index.get((c[0] + dx, c[1] + dy, c[2] + dz))
                if k is not None:
                    out.append(k)
    return out


def interaction_list(lev: Level, c) -> List[Tuple[int, Tuple[int, int, int]]]:
    """I(B) as (box index, offset o = c_beta - c_alpha in box units)."""
    out = []
    pc = parent(c)
    for dx in range(-3, 4):
        for dy in range(-3, 4):
            for dz in range(-3, 4):
                d = (c[0] + dx, c[1] + dy, c[2] + dz)
                k = lev.index.get(d)
                if k is None or cheb(c, d) <= 1:
                    continue
                if cheb(parent(d), pc) <= 1:
                    out.append((k, (dx, dy, dz)))
    return out

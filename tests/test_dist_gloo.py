"""Multi-rank path on CPU (torch.distributed gloo, world size 2, 127.0.0.1).

The library's host-only ownership rule (hfmm_partition, the one hfmm_precompute applies) is
checked to produce a disjoint cover made of whole level-2 subtrees, and the distributed algorithm
of DESIGN.md section 11 -- each rank: S2M/M2M of its subtrees, all-gather of M_l per level,
M2L/L2L/L2T/P2P for its own targets -- is executed with the oracle's passes and gloo collectives;
the union of the ranks' outputs must equal the single-process oracle matvec.
"""
import math
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _spread3(v):
    out = 0
    for b in range(10):
        out |= ((v >> b) & 1) << (3 * b)
    return out


def _morton(c):
    return (_spread3(c[0]) << 2) | (_spread3(c[1]) << 1) | _spread3(c[2])


def _worker(rank, world, port, outdir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from threadpoolctl import threadpool_limits
    threadpool_limits(2)           # two ranks on a shared host: avoid BLAS oversubscription
    try:
        import paper_0911_4114_b200 as hf
        from workloads import small_config, points_and_charges
        from oracle.plan import make_plan
        from oracle.fmm import OracleFMM
        from oracle.tree import parent

        cfg = small_config("dist", n=500, kappa=16 * math.pi, depth=3, eps=1e-4, seed=31)
        x, q = points_and_charges(cfg)
        plan = make_plan(cfg.kappa, cfg.eps, cfg.size, cfg.depth, cfg.alpha)
        L = plan.L_f
        cuts, ranges, perm = hf.partition(x, cfg.depth, cfg.lo, cfg.size, L, plan.levels[L].K, world)
        own_pts = np.sort(perm[ranges[rank, 0]:ranges[rank, 1]])
        f = OracleFMM(x, cfg.lo, cfg.size, plan)
        lev2 = f.levels[2]
        order = sorted(range(len(lev2.boxes)), key=lambda b: _morton(lev2.boxes[b]))
        owned2 = {lev2.boxes[b] for b in order[cuts[rank]:cuts[rank + 1]]}

        def anc2(c, l):
            for _ in range(l - 2):
                c = parent(c)
            return c

        owned = {l: [b for b, c in enumerate(f.levels[l].boxes) if anc2(c, l) in owned2] for l in range(2, L + 1)}
        # ownership = whole subtrees: points of owned leaves == the library's sorted range
        leaf_pts = np.sort(np.concatenate([f.levels[L].members[b] for b in owned[L]] or [np.zeros(0, int)]))
        assert np.array_equal(leaf_pts, own_pts)
        # distributed passes
        M = {L: f.s2m(q, boxes=owned[L])}
        for l in range(L, 2, -1):
            M[l - 1] = f.m2m(M[l], l)
            assert set(M[l - 1]) == set(owned[l - 1])
        Mfull = {}
        for l in range(2, L + 1):
            parts = [None] * world
            dist.all_gather_object(parts, M[l])           # the per-level exchange step
            Mfull[l] = {k: v for part in parts for k, v in part.items()}
            assert len(Mfull[l]) == len(f.levels[l].boxes)
        I = {l: f.m2l(Mfull[l], l, targets=owned[l]) for l in range(2, L + 1)}
        Lloc = {2: I[2]}
        for l in range(2, L):
            Lloc[l + 1] = f.l2l(Lloc[l], I[l + 1], l)
        y_loc = f.p2p(q, own_pts) + (f.l2t(Lloc[L], own_pts) if len(own_pts) else 0)
        parts = [None] * world
        dist.all_gather_object(parts, (own_pts, y_loc, (int(ranges[rank, 0]), int(ranges[rank, 1]))))
        if rank == 0:
            y = np.zeros(len(x), dtype=complex)
            cover = np.zeros(len(x), dtype=int)
            spans = sorted(p[2] for p in parts)
            assert spans[0][0] == 0 and spans[-1][1] == len(x)
            assert all(spans[i][1] == spans[i + 1][0] for i in range(len(spans) - 1))
            for idx, yl, _ in parts:
                y[idx] = yl
                cover[idx] += 1
            assert np.all(cover == 1)
            ref = f.matvec(q)
            err = np.linalg.norm(y - ref) / np.linalg.norm(ref)
            np.save(os.path.join(outdir, "err.npy"), np.array([err]))
    finally:
        dist.destroy_process_group()


def test_two_rank_decomposition_equals_single_rank(tmp_path):
    from paper_0911_4114_b200.build import build
    build(verbose=False)
    port = _free_port()
    mp.spawn(_worker, args=(2, port, str(tmp_path)), nprocs=2, join=True)
    err = float(np.load(tmp_path / "err.npy")[0])
    assert err < 1e-13


def test_partition_ranges_cover_for_many_ranks():
    import paper_0911_4114_b200 as hf
    from workloads import CONFIGS, points_and_charges
    cfg = CONFIGS["C3"]
    x, _ = points_and_charges(cfg)
    for R in (1, 2, 4, 8):
        cuts, ranges, perm = hf.partition(x, cfg.depth, cfg.lo, cfg.size, 3, 4320, R)
        assert cuts[0] == 0 and np.all(np.diff(cuts) >= 0)
        assert ranges[0, 0] == 0 and ranges[-1, 1] == len(x)
        assert np.all(ranges[1:, 0] == ranges[:-1, 1])
        assert np.array_equal(np.sort(perm), np.arange(len(x)))
        if R > 1:   # balanced to within one level-2 subtree
            sizes = np.diff(np.append(ranges[:, 0], len(x)))
            assert sizes.max() <= 2.5 * len(x) / R

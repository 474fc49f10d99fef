"""M2L halo lists of the multi-rank path on CPU (no GPU): hfmm_halo_lists is the host function
hfmm_precompute uses for levels >= HFMM_HALO_LEVEL.

(1) Against an independent geometric computation (numpy, written from P:127): the interaction list
of a level-l box is the set of occupied boxes that are children of its parent's neighbours and not
adjacent to it; ownership descends from hfmm_partition's level-2 cuts.  Rank r must receive from q
exactly the q-owned boxes in its own boxes' lists and send q exactly its boxes in q's lists.
(2) Pairing: for every pair (r, q), r's send list to q equals q's receive list from r (the property
the grouped ncclSend / ncclRecv relies on), and every non-owned box an owned box's M2L reads is
received.
(3) The distributed exchange itself with gloo (world size 2): each process sends its boxes to the
other, and a target's M2L sources are all owned or received.
"""
import math
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from workloads import CONFIGS, small_config, points_and_charges


def _spread3(v):
    out = np.zeros_like(v, dtype=np.int64)
    for b in range(10):
        out |= ((v >> b) & 1) << (3 * b)
    return out


def level_boxes(x, lo, size, depth, l):
    """Occupied level-l boxes (integer coordinates), in the library's Morton order."""
    nb = 1 << depth
    a = size / nb
    c = np.minimum(np.floor((x - np.asarray(lo)) / a).astype(np.int64), nb - 1) >> (depth - l)
    key = (_spread3(c[:, 0]) << 2) | (_spread3(c[:, 1]) << 1) | _spread3(c[:, 2])
    _, first = np.unique(key, return_index=True)
    order = np.argsort(key[first], kind="stable")
    return c[first][order]


def interaction_list(coords, index, b):
    """children of the parent's neighbours, not adjacent (|offset|_inf >= 2), occupied."""
    c = coords[b]
    out = []
    for dx in range(-3, 4):
        for dy in range(-3, 4):
            for dz in range(-3, 4):
                if max(abs(dx), abs(dy), abs(dz)) < 2:
                    continue
                t = (c[0] + dx, c[1] + dy, c[2] + dz)
                if any(abs((t[i] >> 1) - (c[i] >> 1)) > 1 for i in range(3)):
                    continue
                k = index.get(t)
                if k is not None:
                    out.append(k)
    return out


def expected_lists(x, cfg, L_f, K, R, l):
    import paper_0911_4114_b200 as hf
    cuts, _, _ = hf.partition(x, cfg.depth, cfg.lo, cfg.size, L_f, K, R)
    b2 = level_boxes(x, cfg.lo, cfg.size, cfg.depth, 2)
    idx2 = {tuple(c): i for i, c in enumerate(b2)}
    rank_of2 = np.searchsorted(cuts, np.arange(len(b2)), side="right") - 1
    coords = level_boxes(x, cfg.lo, cfg.size, cfg.depth, l)
    index = {tuple(c): i for i, c in enumerate(coords)}
    owner = np.array([rank_of2[idx2[tuple(c >> (l - 2))]] for c in coords])
    recv = [[set() for _ in range(R)] for _ in range(R)]   # recv[r][q]
    for b in range(len(coords)):
        for s in interaction_list(coords, index, b):
            if owner[s] != owner[b]:
                recv[owner[b]][owner[s]].add(s)
    return owner, recv


CASES = [("C3", 3, 4320, (2, 4, 8)),                                           # sphere
         ("cube", 4, 1800, (2, 8))]                                             # cube, L_f = 4


@pytest.mark.parametrize("name,L_f,K,ranks", CASES)
def test_halo_lists_match_geometry(name, L_f, K, ranks):
    import paper_0911_4114_b200 as hf
    if name == "cube":
        cfg = small_config("halo_cube", kind="cube", n=20000, kappa=48 * math.pi, depth=5, eps=1e-4, seed=9)
    else:
        cfg = CONFIGS[name]
    x, _ = points_and_charges(cfg)
    for R in ranks:
        for l in range(2, L_f + 1):
            owner, recv = expected_lists(x, cfg, L_f, K, R, l)
            got = [hf.halo_lists(x, cfg.depth, cfg.lo, cfg.size, L_f, K, R, r, l) for r in range(R)]
            nrecv = 0
            for r in range(R):
                rl, sl = got[r]
                assert len(rl[r]) == 0 and len(sl[r]) == 0
                for q in range(R):
                    assert np.all(np.diff(rl[q]) > 0) and np.all(np.diff(sl[q]) > 0)       # sorted, unique
                    assert set(rl[q].tolist()) == recv[r][q], (name, R, l, r, q)
                    assert set(sl[q].tolist()) == recv[q][r], (name, R, l, r, q)
                    assert np.array_equal(sl[q], got[q][0][r])                               # pairing
                    assert np.all(owner[rl[q]] == q) and np.all(owner[sl[q]] == r)
                    nrecv += len(rl[q])
            if l >= 3:   # a halo is smaller than what an all-gather delivers
                assert nrecv < (R - 1) * len(owner), (name, R, l)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, outdir):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_0911_4114_b200 as hf
        cfg = small_config("halo_gloo", kind="cube", n=20000, kappa=48 * math.pi, depth=5, eps=1e-4, seed=9)
        x, _ = points_and_charges(cfg)
        L_f, K, l = 4, 1800, 4
        owner, _ = expected_lists(x, cfg, L_f, K, world, l)
        coords = level_boxes(x, cfg.lo, cfg.size, cfg.depth, l)
        index = {tuple(c): i for i, c in enumerate(coords)}
        # a synthetic "M_l": one value per owned box (its id); the exchange is grouped send / recv
        rl, sl = hf.halo_lists(x, cfg.depth, cfg.lo, cfg.size, L_f, K, world, rank, l)
        have = {int(b): float(b) for b in np.nonzero(owner == rank)[0]}
        reqs, bufs = [], {}
        for q in range(world):
            if q == rank:
                continue
            send = np.array([have[int(b)] for b in sl[q]], dtype=np.float64)
            bufs[q] = np.zeros(len(rl[q]), dtype=np.float64)
            import torch
            reqs.append(dist.isend(torch.from_numpy(send), q))
            rb = torch.zeros(len(rl[q]), dtype=torch.float64)
            reqs.append(dist.irecv(rb, q))
            bufs[q] = (rb, rl[q])
        for rq in reqs:
            rq.wait()
        for q, (rb, boxes) in bufs.items():
            for v, b in zip(rb.numpy(), boxes):
                have[int(b)] = float(v)
        # every M2L source of every owned target is now present, with the sender's value
        missing = 0
        for b in np.nonzero(owner == rank)[0]:
            for s in interaction_list(coords, index, b):
                if have.get(s) != float(s):
                    missing += 1
        np.save(os.path.join(outdir, f"missing{rank}.npy"), np.array([missing, len(have)]))
    finally:
        dist.destroy_process_group()


def test_halo_exchange_two_ranks_gloo(tmp_path):
    from paper_0911_4114_b200.build import build
    build(verbose=False)
    mp.spawn(_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True)
    for r in range(2):
        missing, have = np.load(tmp_path / f"missing{r}.npy")
        assert missing == 0 and have > 0

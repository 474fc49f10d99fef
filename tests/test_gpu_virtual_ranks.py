"""The library's multi-rank path on ONE B200 (SURVEY §8(e) "same config at
P = 1, 2, 4, 8 agrees with P = 1 to <= 1e-13").

R plans in one process on one device are bound to the ranks of a virtual group
(hfmm_set_dist_virtual): each partitions the octree exactly as rank r of R GPUs would (owned
level-2 subtrees, owned P2P items incl. the ordered off-rank near-field items, owned S2M / M2M /
L2L / L2T ranges, the sibling-group M2L plan over owned boxes) and hfmm_vgroup_matvec runs the
multi-rank matvec with every collective (M_l all-gather per active level, y all-gather) done as
one cudaMemcpyAsync per peer block.  Every rank's output must equal the single-plan matvec to
1e-13 (the only differences are the summation order of the symmetric vs ordered near-field
items) and the oracle to 1e-11.
"""
import math

import numpy as np
import pytest

from workloads import small_config, points_and_charges
from oracle.plan import make_plan
from oracle.fmm import OracleFMM

pytestmark = pytest.mark.gpu


def rel(a, b):
    return float(np.linalg.norm(np.ravel(a) - np.ravel(b)) / np.linalg.norm(np.ravel(b)))


@pytest.fixture(scope="module")
def hf():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a B200"
    import paper_0911_4114_b200 as mod
    from paper_0911_4114_b200.build import build
    build(verbose=False)
    return mod


CASES = {
    # L_f = 2 with translation-only levels 3..5 (warp-per-box S2M / L2T)
    "deep": (small_config("vr_deep", n=4000, kappa=16 * math.pi, depth=5, eps=1e-6, seed=5), "depth"),
    # L_f = 3, S2M at L_f (tile kernels), two active levels
    "two_level": (small_config("vr_two", n=1500, kappa=32 * math.pi, depth=3, eps=1e-6, seed=21), "lf"),
    # cube, L_f = 2
    "cube": (small_config("vr_cube", kind="cube", n=3000, kappa=24 * math.pi, depth=3, eps=1e-6, seed=5), "lf"),
}


def plan_for(hf, cfg, x, src, vg=None, rank=0):
    g = hf.HFMM(0)
    if vg is not None:
        vg.bind(g, rank)
    g.build_tree(x, cfg.depth, cfg.lo, cfg.size)
    flags = hf.HFMM_SOURCE_AT_DEPTH if src == "depth" else hf.HFMM_SOURCE_AT_LF
    g.precompute(cfg.kappa, cfg.eps, cfg.alpha, flags=flags)
    return g


@pytest.mark.parametrize("case", list(CASES))
@pytest.mark.parametrize("R", [2, 4, 8])
def test_virtual_ranks_equal_single_plan(hf, case, R):
    import torch
    cfg, src = CASES[case]
    x, q = points_and_charges(cfg)
    g1 = plan_for(hf, cfg, x, src)
    qd = torch.from_numpy(q).cuda()
    y1 = g1.matvec(qd).cpu().numpy()
    vg = hf.VirtualGroup(R)
    plans = [plan_for(hf, cfg, x, src, vg, r) for r in range(R)]
    infos = [p.info() for p in plans]
    # the ranks partition the points and the P2P work
    assert sum(i["owned_points"] for i in infos) == cfg.n
    assert all(i["nranks"] == R and i["rank"] == r for r, i in enumerate(infos))
    assert sum(i["p2p_pairs"] for i in infos) == g1.info()["p2p_pairs"]
    assert all(i["L_f"] == g1.info()["L_f"] for i in infos)
    Y = vg.matvec(qd).cpu().numpy()
    for r in range(R):
        assert rel(Y[r], y1) <= 1e-13, (case, R, r, rel(Y[r], y1))
    with pytest.raises(hf.HFMMError):          # a bound plan only runs through the group
        plans[0].matvec(qd)
    # repeat: buffers re-used across matvecs
    Y2 = vg.matvec(qd).cpu().numpy()
    assert rel(Y2[R - 1], y1) <= 1e-13
    if R == 2:
        plan = make_plan(cfg.kappa, cfg.eps, cfg.size, cfg.depth, cfg.alpha, source_level=g1.info()["source_level"])
        t = np.arange(0, cfg.n, 7)
        assert rel(Y[1][t], OracleFMM(x, cfg.lo, cfg.size, plan).matvec(q, t)) <= 1e-11
    vg.close()
    for p in plans:
        p.close()
    g1.close()


def _check_group(hf, cfg, src, R, y1, qd):
    vg = hf.VirtualGroup(R)
    plans = [plan_for(hf, cfg, x_of(cfg), src, vg, r) for r in range(R)]
    infos = [p.info() for p in plans]
    Y = vg.matvec(qd).cpu().numpy()
    Y2 = vg.matvec(qd).cpu().numpy()          # buffers (halo packs) re-used across matvecs
    vg.close()
    for p in plans:
        p.close()
    for r in range(R):
        assert rel(Y[r], y1) <= 1e-13, (cfg.name, R, r, rel(Y[r], y1))
    assert rel(Y2[0], y1) <= 1e-13
    return infos


def x_of(cfg):
    return points_and_charges(cfg)[0]


@pytest.mark.parametrize("case", list(CASES))
@pytest.mark.parametrize("R", [2, 8])
def test_virtual_ranks_halo_every_level(hf, case, R, monkeypatch):
    """M2L halos instead of the all-gather on every active level (HFMM_HALO_LEVEL=2): each rank
    receives only the peers' boxes in its owned boxes' interaction lists (sorted lists built
    independently by sender and receiver), packs / scatters them with the gather kernel, and
    its y equals the single plan's to 1e-13."""
    import torch
    monkeypatch.setenv("HFMM_HALO_LEVEL", "2")
    cfg, src = CASES[case]
    x, q = points_and_charges(cfg)
    g1 = plan_for(hf, cfg, x, src)
    qd = torch.from_numpy(q).cuda()
    y1 = g1.matvec(qd).cpu().numpy()
    lv1 = {lv["level"]: lv for lv in g1.info()["levels"]}
    g1.close()
    infos = _check_group(hf, cfg, src, R, y1, qd)
    for inf in infos:
        for lv in inf["levels"]:
            if not lv["active"]:
                continue
            assert lv["halo"], (case, R, lv["level"])
            # a halo never exceeds what the all-gather would deliver (the peers' boxes)
            assert 0 <= lv["m_recv_boxes"] < lv1[lv["level"]]["boxes"]
    # every box sent is received by exactly one (rank, peer) list entry: totals agree
    for l in {lv["level"] for inf in infos for lv in inf["levels"] if lv["active"]}:
        sent = sum(lv["m_send_boxes"] for inf in infos for lv in inf["levels"] if lv["level"] == l)
        recv = sum(lv["m_recv_boxes"] for inf in infos for lv in inf["levels"] if lv["level"] == l)
        assert sent == recv > 0


@pytest.mark.parametrize("R", [2, 4, 8])
def test_virtual_ranks_halo_default_levels(hf, R, monkeypatch):
    """Default policy: levels 2-3 all-gathered (replicated top levels), levels >= 4
    exchanged as halos.  Cube, kappa = 48 pi, eps = 1e-4, depth 5: L_f = 4, so level 4 runs the
    halo path next to all-gathered levels 2-3."""
    import torch
    monkeypatch.delenv("HFMM_HALO_LEVEL", raising=False)
    cfg = small_config("vr_halo4", kind="cube", n=8000, kappa=48 * math.pi, depth=5, eps=1e-4, seed=9)
    x, q = points_and_charges(cfg)
    g1 = plan_for(hf, cfg, x, "lf")
    assert g1.info()["L_f"] == 4
    qd = torch.from_numpy(q).cuda()
    y1 = g1.matvec(qd).cpu().numpy()
    nbox4 = [lv for lv in g1.info()["levels"] if lv["level"] == 4][0]["boxes"]
    g1.close()
    infos = _check_group(hf, cfg, "lf", R, y1, qd)
    for inf in infos:
        by = {lv["level"]: lv for lv in inf["levels"]}
        assert not by[2]["halo"] and not by[3]["halo"] and by[4]["halo"]
        # the level-4 halo is a fraction of the all-gather volume
        assert by[4]["m_recv_boxes"] < 0.75 * nbox4, by[4]


@pytest.mark.parametrize("R", [2, 4])
def test_virtual_ranks_mixed_p2p_tiles(hf, R, monkeypatch):
    """Mixed P2P tiles (512- and <= 384-point target tiles of one leaf, one launch per class on two
    streams; forced on this short grid with HFMM_P2P_MIX=2) under the rank split: the ordered items
    against neighbour leaves owned by a peer are cut into the same two classes, the ranks' P2P
    pairs partition the single plan's, and every rank's y equals the single (mixed) plan's to 1e-13
    (that plan == the oracle: test_gpu_parity.py::test_p2p_mixed_tiles)."""
    import torch
    monkeypatch.setenv("HFMM_P2P_MIX", "2")
    cfg = small_config("vr_mix", n=24000, kappa=16 * math.pi, depth=2, eps=1e-6, seed=37)
    x, q = points_and_charges(cfg)
    g1 = plan_for(hf, cfg, x, "lf")
    assert g1.info()["p2p_mixed_items"] > 0 and g1.info()["L_f"] == 2
    qd = torch.from_numpy(q).cuda()
    y1 = g1.matvec(qd).cpu().numpy()
    pairs1 = g1.info()["p2p_pairs"]
    g1.close()
    infos = _check_group(hf, cfg, "lf", R, y1, qd)
    assert sum(i["p2p_pairs"] for i in infos) == pairs1
    assert all(i["p2p_mixed_items"] > 0 for i in infos)

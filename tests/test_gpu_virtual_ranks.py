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

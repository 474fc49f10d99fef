"""GPU parity: the CUDA path (through the C-ABI) against the independent CPU oracle.

Tolerances:
  - whole matvec vs oracle: relative L2 <= 1e-11 (BASELINE north_star), on the same plan
  - stage buffers (M, I, L, y_near, y_far) vs oracle: relative <= 1e-11 (normwise)
  - FMM vs direct summation: relative L2 <= eps
  - integer plan (ell, N_theta, N_phi, L_f): identical
"""
import math

import numpy as np
import pytest

from workloads import CONFIGS, small_config, points_and_charges
from oracle.plan import make_plan, choose_source_level
from oracle.fmm import OracleFMM
from oracle.direct import direct_sum
from oracle.transfer import bmtf_table, offsets316

pytestmark = pytest.mark.gpu

PARITY = 1e-11


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


def gpu_plan(hf, cfg, x, **kw):
    g = hf.HFMM(0)
    g.build_tree(x, cfg.depth, cfg.lo, cfg.size)
    g.precompute(cfg.kappa, cfg.eps, cfg.alpha, **kw)
    return g


def check_plan(g, plan):
    info = g.info()
    assert info["L_f"] == plan.L_f
    assert info["source_level"] == plan.source_level
    for lv in info["levels"]:
        op = plan.levels[lv["level"]]
        assert (lv["ell"], lv["n_theta"], lv["n_phi"]) == (op.ell, op.n_theta, op.n_phi), lv["level"]
        assert lv["rep"] == op.rep, lv["level"]
        assert lv["ragged"] == (op.rows is not None), lv["level"]
        if lv["level"] <= (plan.source_level or 1):
            assert lv["K"] == op.K, lv["level"]
        assert lv["alpha"] == op.alpha, lv["level"]
        if lv["level"] <= (plan.L_f or 1) + 1 and not math.isnan(op.F):
            assert lv["active"] == op.active
            assert abs(lv["F"] - op.F) <= 1e-6 * op.F
    return info


def box_map(g, f, level):
    """GPU (Morton) box order -> oracle box index."""
    tab = g.debug(7, level)
    lev = f.levels[level]
    return np.array([lev.index[(int(r[0]), int(r[1]), int(r[2]))] for r in tab])


# ------------------------------------------------------------------------------------------
def test_c1_policy_run_is_direct_sum(hf):
    """BASELINE config 0 (C1): no admissible level -> the matvec is the direct sum."""
    cfg = CONFIGS["C1"]
    x, q = points_and_charges(cfg)
    plan = make_plan(cfg.kappa, cfg.eps, cfg.size, cfg.depth, cfg.alpha)
    g = gpu_plan(hf, cfg, x)
    assert g.last_rc == hf.HFMM_W_NO_FARFIELD
    check_plan(g, plan)
    y = g.matvec(q)
    yd = direct_sum(x, q, cfg.kappa)
    assert rel(y, yd) <= PARITY
    assert rel(g.direct(q), yd) <= PARITY


@pytest.fixture(scope="module")
def small(hf):
    cfg = small_config("small", n=777, kappa=32 * math.pi, depth=3, eps=1e-6, seed=21)
    x, q = points_and_charges(cfg)
    plan = make_plan(cfg.kappa, cfg.eps, cfg.size, cfg.depth, cfg.alpha)
    f = OracleFMM(x, cfg.lo, cfg.size, plan)
    g = gpu_plan(hf, cfg, x)
    y = g.matvec(q)
    return cfg, x, q, plan, f, g, y


def test_small_plan_identical(small):
    cfg, x, q, plan, f, g, y = small
    assert plan.L_f == 3 and plan.source_level == 3
    check_plan(g, plan)


# ---- translation-only levels below L_f (R-14) -------------------------------------
@pytest.fixture(scope="module")
def deep(hf):
    cfg = small_config("deep", n=3000, kappa=16 * math.pi, depth=5, eps=1e-6, seed=5)
    x, q = points_and_charges(cfg)
    g = gpu_plan(hf, cfg, x, flags=hf.HFMM_SOURCE_AT_DEPTH)
    plan = make_plan(cfg.kappa, cfg.eps, cfg.size, cfg.depth, cfg.alpha, source_level=cfg.depth)
    f = OracleFMM(x, cfg.lo, cfg.size, plan)
    y = g.matvec(q)
    return cfg, x, q, plan, f, g, y


def test_deep_plan_identical(deep):
    cfg, x, q, plan, f, g, y = deep
    assert plan.L_f == 2 and plan.source_level == 5
    check_plan(g, plan)


def test_deep_stages(deep):
    """M, L at every level 2..D_s (translation-only levels 3..5), I at the active level."""
    cfg, x, q, plan, f, g, y = deep
    M, I, Lloc = f.far_locals(q)
    for l in range(2, plan.source_level + 1):
        mp = box_map(g, f, l)
        K = plan.levels[l].K
        Mg = g.debug(0, l).reshape(-1, K)
        assert rel(Mg, np.stack([M[l][mp[b]] for b in range(len(mp))])) <= PARITY, f"M_{l}"
        Lg = g.debug(2, l).reshape(-1, K)
        assert rel(Lg, np.stack([Lloc[l][mp[b]] for b in range(len(mp))])) <= PARITY, f"L_{l}"


def test_deep_matvec_parity_and_accuracy(deep):
    cfg, x, q, plan, f, g, y = deep
    assert rel(y, f.matvec(q)) <= PARITY
    assert rel(y, direct_sum(x, q, cfg.kappa)) <= cfg.eps


# ---- ragged quadrature on the active levels (R-15, HFMM_RAGGED) ---------------------
@pytest.fixture(scope="module")
def ragged(hf):
    cfg = small_config("rag", n=700, kappa=32 * math.pi, depth=3, eps=1e-6, seed=23)
    x, q = points_and_charges(cfg)
    g = gpu_plan(hf, cfg, x, flags=hf.HFMM_RAGGED)
    plan = make_plan(cfg.kappa, cfg.eps, cfg.size, cfg.depth, cfg.alpha, ragged=True)
    f = OracleFMM(x, cfg.lo, cfg.size, plan)
    y = g.matvec(q)
    return cfg, x, q, plan, f, g, y


def test_ragged_plan_and_tables(ragged):
    cfg, x, q, plan, f, g, y = ragged
    assert plan.L_f == 3 and all(plan.levels[l].rows is not None for l in (2, 3))
    check_plan(g, plan)
    offs = offsets316()
    for l in (2, 3):
        T = g.debug(3, l).reshape(316, -1)
        for oid in (0, 57, 123, 200, 315):
            assert rel(T[oid], f.table(l, offs[oid])) <= 1e-12, (l, oid)


def test_ragged_stages_and_matvec(ragged):
    cfg, x, q, plan, f, g, y = ragged
    M, I, Lloc = f.far_locals(q)
    for l in (2, 3):
        mp = box_map(g, f, l)
        K = plan.levels[l].K
        for what, ref in ((0, M), (1, I), (2, Lloc)):
            got = g.debug(what, l).reshape(-1, K)
            assert rel(got, np.stack([ref[l][mp[b]] for b in range(len(mp))])) <= PARITY, (what, l)
    assert rel(y, f.matvec(q)) <= PARITY
    assert rel(y, direct_sum(x, q, cfg.kappa)) <= cfg.eps


def test_ragged_with_translation_levels(hf):
    """Ragged active levels + rectangular translation-only levels below L_f (R-14 + R-15)."""
    cfg = small_config("ragdeep", n=2500, kappa=16 * math.pi, depth=5, eps=1e-6, seed=5)
    x, q = points_and_charges(cfg)
    g = gpu_plan(hf, cfg, x, flags=hf.HFMM_RAGGED | hf.HFMM_SOURCE_AT_DEPTH)
    plan = make_plan(cfg.kappa, cfg.eps, cfg.size, cfg.depth, cfg.alpha, source_level=cfg.depth, ragged=True)
    check_plan(g, plan)
    t = np.arange(0, cfg.n, 4)
    y = g.matvec(q)
    assert rel(y[t], OracleFMM(x, cfg.lo, cfg.size, plan).matvec(q, t)) <= PARITY
    assert rel(y, direct_sum(x, q, cfg.kappa)) <= cfg.eps


def test_default_source_level_policy(hf):
    """Default policy (no flag) picks the oracle's choose_source_level; result still parity-green."""
    cfg = small_config("pol", n=6000, kappa=16 * math.pi, depth=5, eps=1e-6, seed=9)
    x, q = points_and_charges(cfg)
    g = gpu_plan(hf, cfg, x)
    info = g.info()
    Ds = choose_source_level(x, cfg.lo, cfg.size, cfg.depth, info["L_f"])
    assert info["source_level"] == Ds and Ds > info["L_f"]
    plan = make_plan(cfg.kappa, cfg.eps, cfg.size, cfg.depth, cfg.alpha, source_level=Ds)
    check_plan(g, plan)
    t = np.arange(0, cfg.n, 5)
    y = g.matvec(q)
    assert rel(y[t], OracleFMM(x, cfg.lo, cfg.size, plan).matvec(q, t)) <= PARITY
    # the paper's setup (S2M at L_f) agrees with the translation-only route within eps / 10
    g0 = gpu_plan(hf, cfg, x, flags=hf.HFMM_SOURCE_AT_LF)
    assert g0.info()["source_level"] == info["L_f"]
    assert rel(g0.matvec(q), y) <= cfg.eps / 10


def test_small_transfer_tables(small):
    cfg, x, q, plan, f, g, y = small
    offs = offsets316()
    for l in (2, 3):
        T = g.debug(3, l).reshape(316, -1)
        lp = plan.levels[l]
        for oid in (0, 57, 123, 200, 315):
            ref = bmtf_table(lp.ell, cfg.kappa, offs[oid] * lp.a, lp.n_theta, lp.n_phi).reshape(-1)
            assert rel(T[oid], ref) <= 1e-12


def test_small_stages(small):
    cfg, x, q, plan, f, g, y = small
    M, I, Lloc = f.far_locals(q)
    for l in (2, 3):
        mp = box_map(g, f, l)
        K = plan.levels[l].K
        Mg = g.debug(0, l).reshape(-1, K)
        Mo = np.stack([M[l][mp[b]] for b in range(len(mp))])
        assert rel(Mg, Mo) <= PARITY, f"M_{l}"
        Ig = g.debug(1, l).reshape(-1, K)
        Io = np.stack([I[l][mp[b]] for b in range(len(mp))])
        assert rel(Ig, Io) <= PARITY, f"I_{l}"
        Lg = g.debug(2, l).reshape(-1, K)
        Lo = np.stack([Lloc[l][mp[b]] for b in range(len(mp))])
        assert rel(Lg, Lo) <= PARITY, f"L_{l}"


def test_small_matvec_parity_and_accuracy(small):
    cfg, x, q, plan, f, g, y = small
    yo = f.matvec(q)
    assert rel(y, yo) <= PARITY
    yd = direct_sum(x, q, cfg.kappa)
    assert rel(y, yd) <= cfg.eps
    perm = g.debug(6)
    yn_o, yf_o = f.matvec(q, parts=True)
    assert rel(g.debug(4)[: len(q)], yn_o[perm]) <= PARITY
    assert rel(g.debug(5)[: len(q)], yf_o[perm]) <= PARITY


def test_small_repeat_and_device_path(small, hf):
    import torch
    cfg, x, q, plan, f, g, y = small
    y2 = g.matvec(q)
    # default near field: per-item partial sums reduced in a fixed order -> bitwise repeatable
    assert np.array_equal(y2, y)
    qt = torch.from_numpy(q).cuda()
    yt = g.matvec(qt)
    torch.cuda.synchronize()
    assert rel(yt.cpu().numpy(), y) <= 1e-14


def test_small_linearity(small):
    cfg, x, q, plan, f, g, y = small
    rng = np.random.default_rng(3)
    q2 = rng.standard_normal(len(q)) + 1j * rng.standard_normal(len(q))
    lhs = g.matvec(2.0 * q - 1j * q2)
    rhs = 2.0 * y - 1j * g.matvec(q2)
    assert rel(lhs, rhs) < 1e-13


def test_single_level_cube(hf):
    """Cube geometry, one active level (L_f = 2), ragged tail sizes."""
    cfg = small_config("cube", kind="cube", n=1001, kappa=24 * math.pi, depth=3, eps=1e-6, seed=5)
    x, q = points_and_charges(cfg)
    plan = make_plan(cfg.kappa, cfg.eps, cfg.size, cfg.depth, cfg.alpha)
    g = gpu_plan(hf, cfg, x)
    check_plan(g, plan)
    f = OracleFMM(x, cfg.lo, cfg.size, plan)
    y = g.matvec(q)
    assert rel(y, f.matvec(q)) <= PARITY
    assert rel(y, direct_sum(x, q, cfg.kappa)) <= cfg.eps


def test_forced_breakdown_levels_run(hf):
    """HFMM_FORCE_ALL_LEVELS on C1 (P:833 breakdown demonstration): runs, reports F_l."""
    cfg = CONFIGS["C1"]
    x, q = points_and_charges(cfg)
    g = gpu_plan(hf, cfg, x, flags=hf.HFMM_FORCE_ALL_LEVELS)
    info = g.info()
    assert info["L_f"] == 3
    assert info["levels"][1]["F"] > 1e3          # lambda/4 boxes: roundoff amplification >> 1
    y = g.matvec(q)
    assert np.all(np.isfinite(y))
    # the breakdown is real: the forced run's error vs the direct sum is far above eps and of the
    # order of the amplification F_l; the policy run (no admissible level) is exact
    err = rel(y, direct_sum(x, q, cfg.kappa))
    F = [lv["F"] for lv in info["levels"] if lv["active"]]
    print(f"C1 forced: F_l = {F}, error vs direct {err:.2e} (eps {cfg.eps})")
    assert err > 10 * cfg.eps
    assert err < 10 * max(F)


def test_edge_cases(hf):
    g = hf.HFMM(0)
    # single point: y = 0 (no j != i)
    g.build_tree(np.array([[0.1, 0.2, 0.3]]), 2, (-1, -1, -1), 2.0)
    g.precompute(10.0, 1e-6)
    assert np.all(g.matvec(np.array([1 + 1j])) == 0)
    # two points
    x = np.array([[0.0, 0, 0], [0.3, 0.4, 0.0]])
    g.build_tree(x, 2, (-1, -1, -1), 2.0)
    g.precompute(7.0, 1e-6)
    y = g.matvec(np.array([1 + 0j, 2 + 0j]))
    e = np.exp(1j * 3.5) / 0.5
    assert np.allclose(y, [2 * e, e], rtol=1e-14)
    # errors
    with pytest.raises(hf.HFMMError):
        g.build_tree(np.array([[3.0, 0, 0]]), 2, (-1, -1, -1), 2.0)      # outside the root cube
    with pytest.raises(hf.HFMMError):
        g.build_tree(np.array([[0.1, 0, 0], [0.1, 0, 0]]), 2, (-1, -1, -1), 2.0)  # coincident
    with pytest.raises(hf.HFMMError):
        g.build_tree(np.array([[0.1, 0, 0]]), 1, (-1, -1, -1), 2.0)      # depth < 2
    with pytest.raises(hf.HFMMError):
        g.matvec(np.array([1 + 0j]))                                     # state: no tree
    g.build_tree(x, 2, (-1, -1, -1), 2.0)
    with pytest.raises(hf.HFMMError):
        g.precompute(-1.0, 1e-6)
    # the binding rejects vectors the library would read / write out of bounds
    import torch
    g.precompute(7.0, 1e-6)
    qd = torch.tensor([1 + 0j, 2 + 0j], dtype=torch.complex128, device="cuda")
    for bad in (qd.to(torch.complex64), torch.zeros(3, dtype=torch.complex128, device="cuda"),
                torch.zeros(4, dtype=torch.complex128, device="cuda")[::2], np.zeros(3, dtype=np.complex128)):
        with pytest.raises(hf.HFMMError):
            g.matvec(bad)
    with pytest.raises(hf.HFMMError):
        g.matvec(qd, out=torch.empty(2, dtype=torch.complex128))          # host out for a device q
    assert np.allclose(g.matvec(qd).cpu().numpy(), [2 * e, e], rtol=1e-14)


@pytest.mark.parametrize("up", [True, False])
@pytest.mark.parametrize("grids", [((16, 16), (24, 28)), ((90, 96), (120, 120)), ((54, 56), (108, 108)),
                                   ((432, 432), (1080, 1080))])    # beyond 1024 points (kMaxFFT = 4096)
def test_resample_operator(hf, up, grids):
    import torch
    from oracle.resample import resample_half_batch
    (a, b) = grids if up else grids[::-1]
    rng = np.random.default_rng(7)
    nb = 5 if max(a + b) < 1000 else 2
    F = rng.standard_normal((nb, a[0], a[1] // 2)) + 1j * rng.standard_normal((nb, a[0], a[1] // 2))
    inp = torch.from_numpy(F).cuda()
    out = torch.empty((nb, b[0], b[1] // 2), dtype=torch.complex128, device="cuda")
    hf.resample(inp, a[0], a[1], b[0], b[1], out)
    torch.cuda.synchronize()
    ref = resample_half_batch(F, a[1], b[0], b[1])
    # the oracle reduces j k mod N before forming each DFT phase (oracle/resample.py), so its
    # entries are accurate to a few ulp at every N: one flat tolerance
    assert rel(out.cpu().numpy(), ref) <= 1e-13


# ---- the two M2L kernels (M2L): parent-block vs merged-list -------------------------
@pytest.mark.parametrize("kind", ["cube", "sphere"])
def test_m2l_kernels_agree(hf, kind, monkeypatch):
    """The plan proves per group that the parent-block kernel sums exactly the interaction-list
    terms; forcing the merged-list kernel must then give the same matvec up to summation order,
    and both match the oracle."""
    cfg = small_config("m2lk_" + kind, kind=kind, n=4000, kappa=24 * math.pi, depth=4, eps=1e-6, seed=21)
    x, q = points_and_charges(cfg)
    g = gpu_plan(hf, cfg, x)
    monkeypatch.setenv("HFMM_M2L_LIST", "1")
    g_list = gpu_plan(hf, cfg, x)
    monkeypatch.delenv("HFMM_M2L_LIST")
    act = [lv for lv in g.info()["levels"] if lv["active"]]
    assert act and not any(lv["m2l_block"] for lv in g_list.info()["levels"])
    if kind == "cube":   # uniform cube: every group is a full parent block
        assert all(lv["m2l_block"] for lv in act)
    y, y_list = g.matvec(q), g_list.matvec(q)
    assert rel(y, y_list) <= 1e-13
    plan = make_plan(cfg.kappa, cfg.eps, cfg.size, cfg.depth, cfg.alpha, source_level=g.info()["source_level"])
    y_or = OracleFMM(x, cfg.lo, cfg.size, plan).matvec(q)
    assert rel(y, y_or) <= PARITY


@pytest.mark.parametrize("case", ["small", "deep", "cube"])
def test_deterministic_near_field(hf, case):
    """Default near field (HFMM_DETERMINISTIC): the P2P items write partial sums to their own slots
    and every point sums them in a fixed order -- repeated matvecs are bitwise equal; the atomic
    opt-out (HFMM_ATOMIC_NEAR) agrees up to summation order (1e-14); both == oracle (1e-11)."""
    import torch
    cfgs = {"small": (small_config("det_s", n=777, kappa=32 * math.pi, depth=3, eps=1e-6, seed=21), 0),
            "deep": (small_config("det_d", n=3000, kappa=16 * math.pi, depth=5, eps=1e-6, seed=5),
                     hf.HFMM_SOURCE_AT_DEPTH),
            "cube": (small_config("det_c", kind="cube", n=1001, kappa=24 * math.pi, depth=3, eps=1e-6, seed=5), 0)}
    cfg, flags = cfgs[case]
    x, q = points_and_charges(cfg)
    gd = gpu_plan(hf, cfg, x, flags=flags)
    ga = gpu_plan(hf, cfg, x, flags=flags | hf.HFMM_ATOMIC_NEAR)
    qd = torch.from_numpy(q).cuda()
    y1, y2 = gd.matvec(qd), gd.matvec(qd)
    torch.cuda.synchronize()
    assert torch.equal(y1, y2)
    assert gd.info()["launches"] == ga.info()["launches"] + 1
    y0 = ga.matvec(qd)
    assert rel(y1.cpu().numpy(), y0.cpu().numpy()) <= 1e-14
    plan = make_plan(cfg.kappa, cfg.eps, cfg.size, cfg.depth, cfg.alpha, source_level=gd.info()["source_level"])
    yo = OracleFMM(x, cfg.lo, cfg.size, plan).matvec(q)
    assert rel(y1.cpu().numpy(), yo) <= PARITY and rel(y0.cpu().numpy(), yo) <= PARITY


# ---- Mixed P2P tiles: 512- and <= 384-point target tiles of one leaf ----------------
_MIX_ORACLE = {}


@pytest.mark.parametrize("case", ["leaves", "nofar"])
@pytest.mark.parametrize("near", ["det", "atomic"])
def test_p2p_mixed_tiles(hf, case, near, monkeypatch):
    """The mixed-tile plan (each leaf cut into full 512-point tiles plus <= 384-point tiles, one
    launch per class on two streams; forced on these short grids with HFMM_P2P_MIX=2) gives the
    oracle's matvec and the one-tile-size plan's.  "leaves": level-2 leaves of ~400-570 points
    (one 512-slot tile up to 512 points, two <= 384-point tiles above: both classes, symmetric items
    across them); "nofar": all pairs at the root (2,400 points: four 512-point tiles and one of 352)."""
    if case == "nofar":
        cfg = small_config("p2p_mix_nofar", n=2400, kappa=2 * math.pi, depth=3, eps=1e-4, seed=37)
    else:
        cfg = small_config("p2p_mix_leaves", n=24000, kappa=16 * math.pi, depth=2, eps=1e-6, seed=37)
    x, q = points_and_charges(cfg)
    flags = hf.HFMM_ATOMIC_NEAR if near == "atomic" else 0
    monkeypatch.setenv("HFMM_P2P_MIX", "2")
    g = gpu_plan(hf, cfg, x, flags=flags)
    monkeypatch.setenv("HFMM_P2P_MIX", "0")
    g0 = gpu_plan(hf, cfg, x, flags=flags)
    monkeypatch.delenv("HFMM_P2P_MIX")
    info, info0 = g.info(), g0.info()
    assert info["p2p_mixed_items"] > 0 and info0["p2p_mixed_items"] == 0
    assert info["p2p_tile"] == 512 and not info["p2p_rowskip"]
    assert info["p2p_pairs"] == info0["p2p_pairs"] and info["p2p_sym_pairs"] == info0["p2p_sym_pairs"]
    assert info["p2p_dead_frac"] < info0["p2p_dead_frac"] or info0["p2p_rowskip"]
    y, y0 = g.matvec(q), g0.matvec(q)
    assert rel(y, y0) <= 1e-13
    if near == "det":
        assert np.array_equal(y, g.matvec(q))   # per-item slots, fixed-order sum: bitwise repeatable
    if case == "nofar":
        assert (info["L_f"] or 0) < 2
        assert rel(y, direct_sum(x, q, cfg.kappa)) <= PARITY
    else:
        assert info["L_f"] == 2
        if "yo" not in _MIX_ORACLE:   # one oracle matvec for both accumulation flavours
            plan = make_plan(cfg.kappa, cfg.eps, cfg.size, cfg.depth, cfg.alpha, source_level=info["source_level"])
            _MIX_ORACLE["yo"] = OracleFMM(x, cfg.lo, cfg.size, plan).matvec(q)
        assert rel(y, _MIX_ORACLE["yo"]) <= PARITY


# ---- P2P tile per plan: 384 / 512 / 1,024-point target tiles -------------------
@pytest.mark.parametrize("rowskip", ["on", "off"])
@pytest.mark.parametrize("pt", [3, 4, 8])
@pytest.mark.parametrize("case", ["fmm", "nofar"])
def test_p2p_tiles_agree(hf, pt, case, rowskip, monkeypatch):
    """Every P2P instantiation the plan can pick (3, 4 or 8 targets per thread, forced with
    HFMM_P2P_PT; the row-skipping flavour forced on / off with HFMM_P2P_ROWSKIP_MIN = 0 / 1, DESIGN
    6.1) gives the oracle's matvec.  "nofar": no admissible level, so the matvec is the near
    field over the whole point set -- several 1,024-point tiles, a ragged last tile, symmetric tile
    pairs and diagonal tiles; "fmm": leaves smaller than a tile (partial tiles, dead warp rows).
    The all-pairs entry point (hfmm_direct) with the same tile == the oracle's direct sum."""
    if case == "nofar":
        cfg = small_config("p2p_pt_nofar", n=3001, kappa=2 * math.pi, depth=3, eps=1e-4, seed=31)
    else:
        cfg = small_config("p2p_pt_fmm", n=6000, kappa=8 * math.pi, depth=3, eps=1e-6, seed=31)
    x, q = points_and_charges(cfg)
    monkeypatch.setenv("HFMM_P2P_PT", str(pt))
    monkeypatch.setenv("HFMM_P2P_ROWSKIP_MIN", "0" if rowskip == "on" else "1")
    g = gpu_plan(hf, cfg, x)
    monkeypatch.delenv("HFMM_P2P_PT")
    monkeypatch.delenv("HFMM_P2P_ROWSKIP_MIN")
    assert g.info()["p2p_tile"] == 128 * pt
    assert g.info()["p2p_rowskip"] == (rowskip == "on" and pt != 8)
    y, yd = g.matvec(q), g.direct(q)
    yref = direct_sum(x, q, cfg.kappa)
    assert rel(yd, yref) <= PARITY
    if case == "nofar":
        assert (g.info()["L_f"] or 0) < 2
        assert rel(y, yref) <= PARITY
    else:
        plan = make_plan(cfg.kappa, cfg.eps, cfg.size, cfg.depth, cfg.alpha,
                         source_level=g.info()["source_level"])
        assert rel(y, OracleFMM(x, cfg.lo, cfg.size, plan).matvec(q)) <= PARITY

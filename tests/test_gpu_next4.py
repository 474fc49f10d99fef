"""GPU parity of NEXT 4: coefficient-domain symmetric resampling (P:749,
eqn:FourierSphereSym P:277-280; csrc/kernels_sym.cu), switched on with hfmm_set_next4.

  - every instantiated grid pair (C2 B8 / B16 / B32 and the translation-only levels of C3 / C4 /
    C5), both directions, through the operator entry points (resample, fused M2M with shift and
    child sum, fused L2L with conj shift and +I): vs oracle.resample's 5-step procedure AND vs
    its literal coefficient-domain version resample_coeff_sym, 1e-13;
  - a matvec on C3's level chain (120, 54x56, 40, 28 with translation-only levels 3-5) with the
    NEXT 4 kernels on the 4 level passes they are instantiated for: stages and y vs the oracle (1e-11),
    and vs the default kernels (1e-13).
"""
import math

import numpy as np
import pytest

from workloads import small_config, points_and_charges
from oracle.plan import make_plan
from oracle.fmm import OracleFMM
from oracle.resample import resample_half_batch, resample_coeff_sym

pytestmark = pytest.mark.gpu
TOL = 1e-13


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


@pytest.fixture
def next4(hf):
    prev = hf.set_next4(True)
    yield
    hf.set_next4(prev)


PAIRS = [((16, 16), (32, 32)), ((32, 32), (64, 64)), ((64, 64), (128, 128)), ((24, 24), (32, 32)),
         ((32, 32), (42, 48)), ((42, 48), (60, 60)), ((28, 28), (40, 40)), ((40, 40), (54, 56))]


@pytest.mark.parametrize("child,parent", PAIRS)
def test_next4_operators(hf, next4, child, parent):
    import torch
    (nth, nph), (nth2, nph2) = child, parent
    K, K2 = nth * nph // 2, nth2 * nph2 // 2
    rng = np.random.default_rng(7 * nth + nth2)
    npar = 5
    Cf = rng.standard_normal((8 * npar, K)) + 1j * rng.standard_normal((8 * npar, K))
    Pf = rng.standard_normal((npar, K2)) + 1j * rng.standard_normal((npar, K2))
    S = np.exp(2j * math.pi * rng.uniform(size=(8, K2)))
    Inc = rng.standard_normal((8 * npar, K)) + 1j * rng.standard_normal((8 * npar, K))
    dC, dP, dS, dI = (torch.from_numpy(a).cuda() for a in (Cf, Pf, S, Inc))
    up = torch.empty((8 * npar, K2), dtype=torch.complex128, device="cuda")
    hf.resample(dC, nth, nph, nth2, nph2, up)
    ref5 = resample_half_batch(Cf.reshape(-1, nth, nph // 2), nph, nth2, nph2).reshape(8 * npar, -1)
    refc = resample_coeff_sym(Cf.reshape(-1, nth, nph // 2), nph, nth2, nph2).reshape(8 * npar, -1)
    assert rel(up.cpu().numpy(), ref5) <= TOL and rel(up.cpu().numpy(), refc) <= TOL
    dn = torch.empty((npar, K), dtype=torch.complex128, device="cuda")
    hf.resample(dP, nth2, nph2, nth, nph, dn)
    refd = resample_half_batch(Pf.reshape(-1, nth2, nph2 // 2), nph2, nth, nph).reshape(npar, -1)
    assert rel(dn.cpu().numpy(), refd) <= TOL
    par = torch.empty((npar, K2), dtype=torch.complex128, device="cuda")
    hf.m2m_op(dC, dS, par, nth, nph, nth2, nph2)
    assert rel(par.cpu().numpy(), (S[None] * ref5.reshape(npar, 8, K2)).sum(1)) <= TOL
    out = torch.empty((8 * npar, K), dtype=torch.complex128, device="cuda")
    hf.l2l_op(dP, dS, dI, out, nth2, nph2, nth, nph)
    prod = (np.conj(S)[None] * Pf[:, None, :]).reshape(-1, nth2, nph2 // 2)
    ref_l2l = resample_half_batch(prod, nph2, nth, nph).reshape(8 * npar, -1) + Inc
    assert rel(out.cpu().numpy(), ref_l2l) <= TOL


def test_next4_matvec_c3_levels(hf):
    import torch
    cfg = small_config("n4_deep", n=3000, kappa=16 * math.pi, depth=5, eps=1e-6, seed=5)
    x, q = points_and_charges(cfg)

    def run():
        g = hf.HFMM(0)
        g.build_tree(x, cfg.depth, cfg.lo, cfg.size)
        g.precompute(cfg.kappa, cfg.eps, cfg.alpha, flags=hf.HFMM_SOURCE_AT_DEPTH)
        return g, g.matvec(torch.from_numpy(q).cuda()).cpu().numpy()

    prev = hf.set_next4(False)
    g0, y0 = run()
    hf.set_next4(True)
    try:
        g4, y4 = run()
    finally:
        hf.set_next4(prev)
    assert g0.info()["next4_passes"] == 0
    assert g4.info()["next4_passes"] == 4            # M2M 28->40->54x56, L2L 54x56->40->28
    plan = make_plan(cfg.kappa, cfg.eps, cfg.size, cfg.depth, cfg.alpha, source_level=5)
    assert [(plan.levels[l].n_theta, plan.levels[l].n_phi) for l in range(2, 6)] == \
           [(120, 120), (54, 56), (40, 40), (28, 28)]
    f = OracleFMM(x, cfg.lo, cfg.size, plan)
    M, I, Lloc = f.far_locals(q)
    for l in range(2, 6):
        tab = g4.debug(7, l)
        lev = f.levels[l]
        mp = np.array([lev.index[(int(r[0]), int(r[1]), int(r[2]))] for r in tab])
        K = plan.levels[l].K
        for what, ref in ((0, M), (2, Lloc)):
            got = g4.debug(what, l).reshape(-1, K)
            assert rel(got, np.stack([ref[l][mp[b]] for b in range(len(mp))])) <= 1e-11, (what, l)
    assert rel(y4, f.matvec(q)) <= 1e-11
    assert rel(y4, y0) <= 1e-13

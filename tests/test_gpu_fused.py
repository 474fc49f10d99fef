"""GPU parity of the fused two-pass upward resampler (csrc/kernels_fused.cu; opt-in experiment for
the large square grids 64 -> 128 and 128 -> 256 of the C2 microbench, off by default after a
negative same-box A/B, profiles/r02/fused_ab_r2.txt).

It runs the same row / column arithmetic as the two-pass kernels, operation for operation, with
the intermediate in an L2-sized ring of D items instead of a global buffer, as dependent tasks of
one persistent kernel.  Checked, with batches larger than the ring (slot reuse after D items):
  - bitwise equal to the two-pass kernels (hfmm_set_fused(0)) -- interpolation and fused M2M;
  - against oracle.resample's 5-step procedure on sampled boxes (1e-13), incl. the first and last.
"""
import math

import numpy as np
import pytest

from oracle.resample import resample_half_batch

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


def crandn(gen, *shape):
    import torch
    return torch.randn(*shape, 2, dtype=torch.float64, device="cuda", generator=gen).view(torch.complex128)[..., 0]


# (child grid, parent grid, boxes): ring of D = 64 MB / item < boxes, so slots are reused
@pytest.mark.parametrize("n,n2,nbox", [(64, 128, 700), (128, 256, 600)])
def test_fused_interp(hf, n, n2, nbox):
    import torch
    gen = torch.Generator(device="cuda")
    gen.manual_seed(n)
    K, K2 = n * n // 2, n2 * n2 // 2
    child = crandn(gen, nbox, K)
    out_f = torch.empty(nbox, K2, dtype=torch.complex128, device="cuda")
    out_2 = torch.empty_like(out_f)
    prev = hf.set_fused(True)
    try:
        hf.resample(child, n, n, n2, n2, out_f)
        hf.set_fused(False)
        hf.resample(child, n, n, n2, n2, out_2)
    finally:
        hf.set_fused(prev)
    torch.cuda.synchronize()
    assert torch.equal(out_f, out_2)
    s = np.array([0, 1, nbox // 3, nbox // 2 + 7, nbox - 1])
    ref = resample_half_batch(child[s].cpu().numpy().reshape(-1, n, n // 2), n, n2, n2).reshape(len(s), -1)
    assert rel(out_f[s].cpu().numpy(), ref) <= 1e-13


@pytest.mark.parametrize("n,n2,npar", [(64, 128, 90), (128, 256, 70)])
def test_fused_m2m(hf, n, n2, npar):
    import torch
    gen = torch.Generator(device="cuda")
    gen.manual_seed(100 + n)
    K, K2 = n * n // 2, n2 * n2 // 2
    child = crandn(gen, 8 * npar, K)
    shift = torch.polar(torch.ones(8, K2, dtype=torch.float64, device="cuda"),
                        2 * math.pi * torch.rand(8, K2, dtype=torch.float64, device="cuda", generator=gen))
    par_f = torch.empty(npar, K2, dtype=torch.complex128, device="cuda")
    par_2 = torch.empty_like(par_f)
    prev = hf.set_fused(True)
    try:
        hf.m2m_op(child, shift, par_f, n, n, n2, n2)
        hf.set_fused(False)
        hf.m2m_op(child, shift, par_2, n, n, n2, n2)
    finally:
        hf.set_fused(prev)
    torch.cuda.synchronize()
    assert torch.equal(par_f, par_2)
    sh = shift.cpu().numpy()
    for p in (0, npar // 2, npar - 1):
        chp = child[8 * p: 8 * p + 8].cpu().numpy().reshape(8, n, n // 2)
        R = resample_half_batch(chp, n, n2, n2).reshape(8, -1)
        assert rel(par_f[p].cpu().numpy(), (sh * R).sum(0)) <= 1e-13

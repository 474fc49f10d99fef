"""CPU-side checks of the C-ABI library: it loads, exports every symbol declared in
include/hfmm.h, its host-only plan logic agrees with the independent oracle, and compute
calls fail loudly (no CPU fallback) when no GPU is present."""
import math
import os
import re

import numpy as np
import pytest

import paper_0911_4114_b200 as hf
from oracle.plan import level_params

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module", autouse=True)
def built():
    from paper_0911_4114_b200.build import build
    build(verbose=False)


def declared_symbols():
    src = open(os.path.join(ROOT, "include", "hfmm.h")).read()
    return sorted(set(re.findall(r"\b(hfmm_[a-z0-9_]+)\s*\(", src)))


def test_header_declares_binding_list():
    assert declared_symbols() == sorted(hf.EXPORTED)


def test_library_exports_every_symbol():
    import subprocess
    out = subprocess.check_output(["nm", "-D", "--defined-only", hf.LIB_PATH]).decode()
    exported = set(re.findall(r" T (hfmm_\w+)", out))
    missing = set(declared_symbols()) - exported
    assert not missing, missing
    lib = hf.load()
    for name in declared_symbols():
        assert hasattr(lib, name)


def test_library_targets_sm100a():
    import subprocess
    out = subprocess.check_output(["cuobjdump", "--list-elf", hf.LIB_PATH]).decode()
    assert "sm_100a" in out


def test_oracle_not_linked_or_imported():
    # the product never imports the oracle (task rule); check the package sources
    pkg = os.path.join(ROOT, "paper_0911_4114_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cpp", ".h")):
                txt = open(os.path.join(dirpath, f)).read()
                assert "import oracle" not in txt and "from oracle" not in txt, f


@pytest.mark.parametrize("ka,eps", [(8 * math.pi, 1e-6), (4 * math.pi, 1e-6), (16 * math.pi, 1e-4),
                                    (8 * math.pi, 1e-8), (math.pi / 2, 1e-4), (32 * math.pi, 2e-6),
                                    (16 * math.pi, 2e-6), (2 * math.pi, 1e-6)])
def test_host_plan_equals_oracle_plan(ka, eps):
    """Plan agreement of two independent implementations (R-12): integers must match."""
    g = hf.level_quadrature(ka, 1.0, eps, 0.8)
    o = level_params(ka, 1.0, eps, 0.8)
    assert g[:3] == o[:3]
    assert g[3] == o[3]          # ragged per-row N_phi(theta_n) too


@pytest.mark.parametrize("ka,a,eps", [(32 * math.pi, 2 / 128, 1e-8), (32 * math.pi, 2 / 16, 1e-8),
                                      (128 * math.pi, 1 / 64, 1e-6), (16 * math.pi, 2 / 32, 1e-6),
                                      (5.0, 0.5, 1e-4), (1e-3, 0.01, 1e-12), (300.0, 0.5, 1e-10)])
def test_host_rep_grid_equals_oracle(ka, a, eps):
    """Translation-only grid rule (R-14) of the library == the oracle's (independent code)."""
    from oracle.plan import rep_grid
    assert hf.rep_grid(ka, a, eps) == rep_grid(ka, a, eps)


@pytest.mark.parametrize("ka,eps", [(8 * math.pi, 1e-6), (16 * math.pi, 1e-8), (32 * math.pi, 2e-6)])
def test_host_ragged_rows_equal_oracle(ka, eps):
    """Ragged rows (R-15) of the library == the oracle's (independent implementations)."""
    from oracle.plan import LevelPlan, ragged_rows
    ell, nth, nph, _ = level_params(ka, 1.0, eps, 0.8)
    lp = LevelPlan(2, 1.0, ell, nth, nph, alpha=0.8)
    want = ragged_rows(lp, ka, eps, eps_absolute=True)
    assert hf.ragged_rows(ka, 1.0, eps, 0.8, ell, nth, nph) == want


def test_plan_rejects_bad_args():
    with pytest.raises(hf.HFMMError):
        hf.level_quadrature(-1.0, 1.0, 1e-6, 0.8)


def test_create_fails_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(hf.HFMMError) as e:
        hf.HFMM(0)
    assert "no CUDA device" in str(e.value)

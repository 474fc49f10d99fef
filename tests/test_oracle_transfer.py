"""Pins for oracle/transfer.py: closed forms, the Gegenbauer identity, Alg. 1 routes."""
import math
import os

import numpy as np
import pytest
from scipy.integrate import quad

from oracle.specfun import sph_hn, sph_jn
from oracle.transfer import (transfer_eval, transfer_coeffs, s_tilde, bmtf_coeffs, bmtf_table,
                             bmtf_realspace_column, shat, offsets316, offsets_canonical)
from oracle.plan import collino_bound
from oracle.rig import gegenbauer_partial, kernel, quadrature_sum

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def test_counts_golden():
    vals = dict(l.split() for l in open(os.path.join(GOLDEN, "counts.txt")) if not l.startswith("#"))
    assert len(offsets316()) == int(vals["transfer_vectors"])
    assert len(offsets_canonical()) == int(vals["canonical_transfer_vectors"])


def test_T_ell0_closed_form():
    # P:110 with ell = 0: T = (i k / 4 pi) h_0(k|r0|) = k e^{ix} / (4 pi x), x = k|r0|
    k, r0 = 7.3, np.array([0.0, 2.0, 1.0])
    x = k * np.linalg.norm(r0)
    s = shat(np.array([0.3, 1.2]), np.array([2.0, 0.1]))
    T = transfer_eval(0, k, r0, s)
    assert np.allclose(T, k * np.exp(1j * x) / (4 * math.pi * x), rtol=1e-14, atol=0)


def test_T_rotation_invariance():
    # T depends on s only through s . r0hat
    rng = np.random.default_rng(1)
    k, ell = 5.0, 12
    r0 = np.array([1.0, -2.0, 0.5])
    Q, _ = np.linalg.qr(rng.standard_normal((3, 3)))
    s = shat(rng.uniform(0, math.pi, 20), rng.uniform(0, 2 * math.pi, 20))
    assert np.allclose(transfer_eval(ell, k, r0, s), transfer_eval(ell, k, Q @ r0, s @ Q.T), rtol=1e-12)


def test_s_tilde_vs_quadrature():
    # P:388 closed form vs numerical Fourier coefficient of |sin|
    for n in range(0, 9):
        re = quad(lambda t: abs(math.sin(t)) * math.cos(n * t), 0, 2 * math.pi, limit=200)[0] / (2 * math.pi)
        assert abs(s_tilde(np.array([n]))[0] - re) < 1e-12
        assert abs(s_tilde(np.array([-n]))[0] - re) < 1e-12


def test_gegenbauer_converges_to_kernel():
    # eqn:Gegenbauer, converges for |r0| >= 2/sqrt(3) |r|
    k = 12.0
    r = np.array([0.3, -0.4, 0.5])
    r0 = np.array([1.6, 0.9, -1.1])
    exact = kernel(k, float(np.linalg.norm(r + r0)))
    errs = [abs(gegenbauer_partial(k, r, r0, ell) - exact) / abs(exact) for ell in (5, 10, 20, 30, 40)]
    assert errs[-1] < 1e-12
    assert all(errs[i + 1] < errs[i] for i in range(3))


def test_collino_closed_form_equals_aligned_tail():
    # eqn:CollinoError: closed form == kappa |sum_{n>ell} (-+1)^n (2n+1) h_n j_n| (sign-matched)
    k, r, r0 = 10.0, 0.9, 2.0
    nmax = 200
    h = sph_hn(nmax, k * r0)
    j = sph_jn(nmax, k * r)
    for ell in (8, 12, 16, 20):
        n = np.arange(ell + 1, 90)
        tail_p = k * abs(np.sum((2 * n + 1) * h[n] * j[n]))                    # rhat.r0hat = -1
        tail_m = k * abs(np.sum(((-1.0) ** n) * (2 * n + 1) * h[n] * j[n]))    # rhat.r0hat = +1
        cp = k ** 2 * (r * r0 / (r0 - r)) * abs(h[ell + 1] * j[ell] - h[ell] * j[ell + 1])
        cm = k ** 2 * (r * r0 / (r0 + r)) * abs(h[ell + 1] * j[ell] + h[ell] * j[ell + 1])
        assert abs(cp - tail_p) < 1e-10 * tail_p
        assert abs(cm - tail_m) < 1e-10 * tail_m
        assert abs(collino_bound(ell, k, r, r0) - max(cp, cm)) < 1e-14 * max(cp, cm)


@pytest.mark.parametrize("o", [(2, 0, 0), (2, 1, 3), (-3, 2, -2)])
def test_alg1_spectral_equals_realspace(o):
    # P:532 / Fig. SarvasDiag: the real-space route equals Alg. 1's spectral route
    k, a, ell, nth, nph = 20.0, 1.0, 30, 64, 64
    r0 = np.array(o, dtype=float) * a
    T = bmtf_table(ell, k, r0, nth, nph)
    for q in (0, 5, 17):
        phi = 2 * math.pi * q / nph
        col = bmtf_realspace_column(ell, k, r0, nth, phi)
        assert np.max(np.abs(col - T[:, q])) < 1e-12 * np.max(np.abs(T))


def test_alg1_band_limits():
    # theta-spectrum of T^{s,L} vanishes for |n| >= N_theta/2; phi-spectrum for |m| > ell
    k, ell, nth = 15.0, 20, 48
    r0 = np.array([2.0, -1.0, 2.0])
    C = bmtf_coeffs(ell, k, r0, nth)
    assert C.shape == (nth - 1, 2 * ell + 1)
    nph = 2 * (2 * ell + 6)
    T = bmtf_table(ell, k, r0, nth, nph)
    # rebuild full rows n <= N_theta/2 and check spectra
    full = np.concatenate([T, T[(nth - np.arange(nth)) % nth]], axis=1)     # eqn:NumSphereSym
    spec_theta = np.fft.fft(full, axis=0) / nth
    assert np.max(np.abs(spec_theta[nth // 2])) < 1e-14 * np.max(np.abs(spec_theta))
    spec_phi = np.fft.fft(full, axis=1) / nph
    m = np.fft.fftfreq(nph, 1.0 / nph)
    assert np.max(np.abs(spec_phi[:, np.abs(m) > ell])) < 1e-14 * np.max(np.abs(spec_phi))


def test_doubled_sphere_normalisation():
    # P:245-256 with T^s := bandlimited (1/2)|sin theta| (i.e. T == 1):
    # (8 pi^2/(N_t N_p)) sum_half e^{i k s.r} T^s  ->  int_{S^2} e^{i k s.r} dS = 4 pi j_0(k|r|)
    k, r = 9.1, np.array([0.3, 0.5, -0.6])
    kr = k * np.linalg.norm(r)
    for nth in (48, 64):
        nph = nth
        n = np.arange(-(nth // 2 - 1), nth // 2)
        th = 2 * math.pi * np.arange(nth) / nth
        sband = (np.exp(1j * np.outer(th, n)) @ (0.5 * s_tilde(n))).real
        table = np.repeat(sband[:, None], nph // 2, axis=1)
        got = quadrature_sum(k, r, table, nth, nph)
        assert abs(got - 4 * math.pi * math.sin(kr) / kr) < 1e-12


def test_toy_integral_filtered_quadrature():
    # int |sin| cos(64 cos) = sin(64)/16; filtered rule with K = 2N+1 converges
    vals = dict(l.split(None, 1) for l in open(os.path.join(GOLDEN, "toy_integral.txt")) if not l.startswith("#"))
    w = float(vals["omega"])
    exact = math.sin(64) / 16
    def filtered(N):
        K = 2 * N + 1
        th = 2 * math.pi * np.arange(K) / K
        n = np.arange(-N, N + 1)
        fN = (np.exp(1j * np.outer(th, n)) @ s_tilde(n)).real
        return 2 * math.pi / K * np.sum(fN * np.cos(w * np.cos(th)))
    def trapezoid(K):
        th = 2 * math.pi * np.arange(K) / K
        return 2 * math.pi / K * np.sum(np.abs(np.sin(th)) * np.cos(w * np.cos(th)))
    err = {N: abs(filtered(N) - exact) / abs(exact) for N in (50, 64, 80, 96, 110)}
    assert err[50] > 1e-5 and err[64] > 1e-8      # not yet resolved at or below the bandwidth 64
    assert err[96] < 1e-12 and err[110] < 1e-12   # super-algebraic convergence once N > 64
    e1 = abs(trapezoid(1001) - exact)
    e2 = abs(trapezoid(2001) - exact)
    slope = math.log(e1 / e2) / math.log(2001 / 1001)
    assert 1.7 < slope < 2.3                      # 1/K^2 (Fig. SINconv caption)


def test_reflection_symmetry_34_tables():
    """P:412-415 / Fig. SemiOctant: with N_theta even and N_phi = 0 mod 4, every one of the 316
    bandlimited tables is a grid permutation of one of the 34 canonical ones (x >= y >= 0, z >= 0):
    T_{F P c}(theta, phi) = T_c(P F (theta, phi)) with F the sign flips and P the x<->y swap.
    Written here from the geometry (reflections of s-hat), independently of the library."""
    import math
    from oracle.transfer import bmtf_table, offsets316, offsets_canonical
    ell, kappa, a, nth, nph = 12, 9.0, 1.0, 28, 32
    h = nph // 2
    canon = {tuple(int(v) for v in c): bmtf_table(ell, kappa, c.astype(float) * a, nth, nph)
             for c in offsets_canonical()}
    assert len(canon) == 34
    n, m = np.meshgrid(np.arange(nth), np.arange(h), indexing="ij")
    rng = np.random.default_rng(0)
    for o in offsets316()[rng.choice(316, 40, replace=False)]:
        ox, oy, oz = (int(v) for v in o)
        c = (max(abs(ox), abs(oy)), min(abs(ox), abs(oy)), abs(oz))
        nn, mm = n.copy(), m.copy()
        if ox < 0:
            mm = (nph // 2 - mm) % nph            # phi -> pi - phi
        if oy < 0:
            mm = (-mm) % nph                      # phi -> -phi
        if oz < 0:
            nn = (nth // 2 - nn) % nth            # theta -> pi - theta
        if abs(oy) > abs(ox):
            mm = (nph // 4 - mm) % nph            # phi -> pi/2 - phi
        up = mm >= h                              # eqn:NumSphereSym back into the stored half
        nn = np.where(up, (nth - nn) % nth, nn)
        mm = np.where(up, mm - h, mm)
        direct = bmtf_table(ell, kappa, o.astype(float) * a, nth, nph)
        assert np.allclose(canon[c][nn, mm], direct, rtol=0, atol=1e-13 * np.max(np.abs(direct))), tuple(o)

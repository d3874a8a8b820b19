"""Oracle pins: PML scaling (BJ configs[0] profile; D3, D4) by closed forms, finite
differences and the exact PML plane wave.  -m "not gpu"."""
import cmath
import math

import numpy as np
import pytest

from oracle.oracle import Oracle, gfun, problem_from_config

SIG, KAP = 5.0, 0.3


def test_profile_closed_forms():
    g, g1, g2 = gfun(KAP, KAP, SIG)
    assert math.isclose(g, SIG * KAP / 3.0, rel_tol=1e-15)
    assert math.isclose(g1, SIG, rel_tol=1e-15)
    assert math.isclose(g2, 2 * SIG / KAP, rel_tol=1e-15)
    assert gfun(0.0, KAP, SIG) == (0.0, 0.0, 0.0)
    assert gfun(-0.1, KAP, SIG) == (0.0, 0.0, 0.0)          # g = g' = 0 for x <= 0
    # linear beyond kappa: g'' = 0 and C^1 continuation
    g_hi, g1_hi, g2_hi = gfun(2 * KAP, KAP, SIG)
    assert g2_hi == 0.0 and g1_hi == SIG
    assert math.isclose(g_hi, SIG * KAP / 3 + SIG * KAP, rel_tol=1e-15)
    # g' > 0 for x > 0
    assert all(gfun(t, KAP, SIG)[1] > 0 for t in np.linspace(1e-3, 3 * KAP, 50))


@pytest.mark.parametrize("t", [0.05, 0.17, 0.29, 0.45, 0.8])
def test_profile_finite_differences(t):
    e = 1e-6
    gp = (gfun(t + e, KAP, SIG)[0] - gfun(t - e, KAP, SIG)[0]) / (2 * e)
    gpp = (gfun(t + e, KAP, SIG)[1] - gfun(t - e, KAP, SIG)[1]) / (2 * e)
    assert abs(gp - gfun(t, KAP, SIG)[1]) < 1e-7 * max(1, abs(gp))
    assert abs(gpp - gfun(t, KAP, SIG)[2]) < 1e-6 * max(1, abs(gpp))


def test_gamma_global_inside_and_sides():
    o = Oracle.from_config(k=20)
    h, ng, ni = o.prob.h, o.prob.ng, o.prob.nix
    # inside Omega_int: gamma = 1 (g_i = 0 on (a, b))
    for X3 in range(3 * ng + 1, 3 * (ng + ni), 7):
        assert o.gamma(0, X3) == (1.0, 0.0)
    # upper side: gamma = 1 + i g'(x - b), gamma' = +i g''
    X3 = 3 * (ng + ni) + 5
    t = 5 * h / 3
    gg = gfun(t, o.prob.kappa, o.prob.sigma0)
    gam, dgam = o.gamma(0, X3)
    assert abs(gam - (1 + 1j * gg[1])) < 1e-14 * abs(gam) and abs(dgam - 1j * gg[2]) < 1e-14 * abs(dgam)
    # lower side: g_i = -g(a - x) -> gamma = 1 + i g'(a - x), gamma' = -i g''(a - x)  (D4)
    X3 = 3 * ng - 5
    gam, dgam = o.gamma(1, X3)
    assert abs(gam - (1 + 1j * gg[1])) < 1e-14 * abs(gam) and abs(dgam + 1j * gg[2]) < 1e-14 * abs(dgam)


@pytest.mark.parametrize("axis", [0, 1])
def test_gamma_prime_is_derivative_of_gamma(axis):
    """gamma'(x) must be d gamma / dx on both sides (sign pin for D4): centred differences in thirds."""
    o = Oracle.from_config(k=20)
    h3 = o.prob.h / 3
    N = o.N[axis]
    for X3 in list(range(2, 3 * 10 - 2, 4)) + list(range(3 * (N - 10) + 2, 3 * N - 2, 4)):
        gm, _ = o.gamma(axis, X3 - 1)
        gp, _ = o.gamma(axis, X3 + 1)
        _, dg = o.gamma(axis, X3)
        fd = (gp - gm) / (2 * h3)
        assert abs(fd - dg) <= 0.02 * abs(dg) + 1e-9, (X3, fd, dg)


def test_sigma0_zero_is_plain_helmholtz():
    """sigma0 = 0 => D = I, beta = 0 everywhere: every free row is the textbook stencil."""
    o = Oracle(problem_from_config(20, sigma0=0.0))
    A7 = o.stencil()
    kh2 = (o.prob.k * o.prob.h) ** 2
    nfx, nfy = o.nf
    i = np.arange(o.nfree) % nfx
    j = np.arange(o.nfree) // nfx
    interior = (i > 0) & (i < nfx - 1) & (j > 0) & (j < nfy - 1)
    ref = np.array([4 - kh2 / 2, -1 - kh2 / 12, -1 - kh2 / 12, -1 - kh2 / 12, -1 - kh2 / 12, -kh2 / 12, -kh2 / 12])
    assert np.max(np.abs(A7[interior] - ref)) < 1e-14


def test_local_gamma_ramps():
    """g_j^i: upper ramp from b_j above the int box, lower ramp from a_j below, global inside."""
    o = Oracle.from_config(k=400, nsub_x=16, nsub_y=16)
    j = 5 + 16 * 7
    s = o.subdomain(j)
    h = o.prob.h
    for ax in range(2):
        a, b = s["int_lo"][ax], s["int_hi"][ax]
        for d in [1, 2, 4, 13, 29]:
            if 3 * b + d < 3 * s["full_hi"][ax]:
                gg = gfun(d * h / 3, o.prob.kappa, o.prob.sigma0)
                gam, dgam = o.gamma(ax, 3 * b + d, sub=j)
                assert abs(gam - (1 + 1j * gg[1])) < 1e-14 * abs(gam) and abs(dgam - 1j * gg[2]) < 1e-14 * abs(dgam)
            if 3 * a - d > 3 * s["full_lo"][ax]:
                gg = gfun(d * h / 3, o.prob.kappa, o.prob.sigma0)
                gam, dgam = o.gamma(ax, 3 * a - d, sub=j)
                assert abs(gam - (1 + 1j * gg[1])) < 1e-14 * abs(gam) and abs(dgam + 1j * gg[2]) < 1e-14 * abs(dgam)
        for X3 in range(3 * a + 1, 3 * b, 5):
            assert o.gamma(ax, X3, sub=j) == o.gamma(ax, X3)


def _pml_plane_wave_residual(ppw):
    """max over PML rows of |(A u_I)_p| / (k^2 h^2) for u = exp(i k x~), x~ = x + i g_x(x): the exact
    solution of Delta_pml u + k^2 u = 0; a wrong beta sign leaves an O(1) residual."""
    k = 20.0
    o = Oracle(problem_from_config(k, ppw=ppw, n_pml_global=ppw))
    h, ng, ni = o.prob.h, o.prob.ng, o.prob.nix
    nfx, nfy = o.nf
    idx = np.arange(o.nfree)
    i = idx % nfx + 1
    j = idx // nfx + 1
    x = (i - ng) * h

    def gx(xx):
        if xx > ni * h:
            return gfun(xx - ni * h, o.prob.kappa, o.prob.sigma0)[0]
        if xx < 0:
            return -gfun(-xx, o.prob.kappa, o.prob.sigma0)[0]
        return 0.0

    xt = x + 1j * np.array([gx(v) for v in x])
    u = np.exp(1j * k * xt)
    r = o.matvec(u)
    # rows away from dOmega (3 cells) and inside the x-PML layers
    sel = (j > 3) & (j < nfy - 2) & (i > 3) & (i < nfx - 2) & ((i < ng) | (i > ng + ni))
    scale = (k * h) ** 2 * np.abs(u[sel])
    return np.max(np.abs(r[sel]) / scale)


def test_pml_plane_wave_consistency():
    e10 = _pml_plane_wave_residual(10)
    e20 = _pml_plane_wave_residual(20)
    e40 = _pml_plane_wave_residual(40)
    # a flipped beta sign leaves |2 beta . grad u| / (k^2 |u|) ~ 0.3 at every ppw; the consistent
    # discretisation must fall by > 3x over two mesh doublings (centroid coefficients: ~O(h) near the
    # g'' jump at kappa, O(h^2) elsewhere)
    assert e10 < 0.5
    assert e20 < e10 and e40 < e10 / 3.0, (e10, e20, e40)

"""Oracle pins: P1 assembly (eq. (weak); D1, D5-D7), RHS (D14) and the local operators
(P:85-94).  -m "not gpu"."""
import math

import numpy as np
import pytest

from oracle.oracle import Oracle, Problem, problem_from_config
from paper_2602_00735_b200.workloads import CONFIGS, sources

SLOTS = [(0, 0), (1, 0), (-1, 0), (0, 1), (0, -1), (1, 1), (-1, -1)]


@pytest.mark.parametrize("name", ["c0", "c1"])
def test_interior_stencil_closed_form(name):
    """Inside Omega_int (D = I, beta = 0) the P1 SW->NE stencil is the textbook one:
    centre 4 - (kh)^2/2; E/W/N/S -1 - (kh)^2/12; NE/SW -(kh)^2/12; NW/SE absent; row sum -(kh)^2."""
    cfg = CONFIGS[name]
    o = Oracle.from_config(k=cfg.k, nsub_x=cfg.nsub, nsub_y=cfg.nsub)
    A7 = o.stencil()
    kh2 = (cfg.k * o.prob.h) ** 2
    ng, ni = o.prob.ng, o.prob.nix
    nfx = o.nf[0]
    rows = [(i - 1) + nfx * (j - 1) for i in range(ng + 1, ng + ni) for j in range(ng + 1, ng + ni, 5)]
    ref = np.array([4 - kh2 / 2, -1 - kh2 / 12, -1 - kh2 / 12, -1 - kh2 / 12, -1 - kh2 / 12, -kh2 / 12, -kh2 / 12])
    assert np.max(np.abs(A7[rows] - ref)) < 1e-14
    assert np.max(np.abs(A7[rows].sum(axis=1) + kh2)) < 1e-13


def test_symmetry_structure():
    """D7: A = A^T exactly for sigma0 = 0; with the paper's beta term A != A^T, but A - A^T vanishes on
    rows whose six triangles all lie inside Omega_int (beta = 0 there)."""
    o0 = Oracle(problem_from_config(20, sigma0=0.0))
    A = o0.matrix()
    assert abs(A - A.T).max() == 0.0
    o = Oracle.from_config(k=20)
    A = o.matrix().tocsr()
    D = (A - A.T).tocsr()
    assert abs(D).max() > 1e-3                       # the beta term is present
    ng, ni = o.prob.ng, o.prob.nix
    nfx = o.nf[0]
    rowmax = np.asarray(abs(D).max(axis=1).todense()).ravel()
    rows = [(i - 1) + nfx * (j - 1) for j in range(ng + 1, ng + ni) for i in range(ng + 1, ng + ni)]
    assert np.all(rowmax[rows] == 0.0)
    assert np.count_nonzero(rowmax) > 0


def test_rhs_mass_conservation():
    """Unit-mass Gaussians (D14): sum_p b_p = sum_s a_s up to the Gaussian tail at dOmega."""
    cfg = CONFIGS["c1"]
    o = Oracle.from_config(k=cfg.k, nsub_x=4, nsub_y=4)
    xy, amp, sig = sources(cfg)
    b = o.rhs(xy, amp, sig)
    assert abs(b.sum() - amp.sum()) < 1e-10 * abs(amp).sum()
    # a single source: b peaks at the nearest node and is real for a real amplitude
    b1 = o.rhs(np.array([[0.5, 0.5]]), np.array([1.0 + 0j]), sig)
    assert abs(b1.sum() - 1.0) < 1e-12 and np.max(np.abs(b1.imag)) == 0.0


@pytest.mark.parametrize("name", ["c0", "c1"])
def test_rhs_is_consistent_mass_times_nodal_f(name):
    """D14 / O5: b = M_ff f_I with the CONSISTENT P1 mass matrix, entrywise.  M is recovered from the assembly
    itself: with sigma0 = 0, A(k') = K - k'^2 M, so M = (A(0) - A(k')) / k'^2 on the same mesh (k' h = 1); the
    recovered M's interior rows are those of the closed-form stencil test above (h^2/2 centre, h^2/12 on the six
    edge neighbours).  A lumped mass (or a dropped Gaussian, a wrong node coordinate, a swapped axis) fails this
    at the 1e-12 level, which the sum rule above cannot see."""
    cfg = CONFIGS[name]
    P = problem_from_config(cfg.k, nsub_x=cfg.nsub, nsub_y=cfg.nsub)
    o = Oracle(P)
    xy, amp, sig = sources(cfg)
    b = o.rhs(xy, amp, sig)
    kp = 1.0 / P.h

    def frame(kk):
        return Oracle(Problem(k=kk, sigma0=0.0, h=P.h, nix=P.nix, niy=P.niy, ng=P.ng, kappa=P.kappa, px=1, py=1,
                              novlp=P.novlp, npml=P.npml))

    M = ((frame(0.0).matrix() - frame(kp).matrix()) / kp ** 2).tocsr()
    nfx = o.nf[0]
    idx = np.arange(o.nfree)
    x = (idx % nfx + 1 - P.ng) * P.h
    y = (idx // nfx + 1 - P.ng) * P.h
    f = np.zeros(o.nfree, np.complex128)
    for (xs, ys), a in zip(xy, amp):
        f += a * np.exp(-((x - xs) ** 2 + (y - ys) ** 2) / (2 * sig * sig)) / (2 * math.pi * sig * sig)
    ref = M @ f
    assert np.max(np.abs(b - ref)) <= 1e-12 * np.max(np.abs(ref))
    # the recovered M is the consistent one: interior row h^2/2 on the diagonal, h^2/12 on E/W/N/S/NE/SW
    g = (P.ng + P.nix // 2 - 1) + nfx * (P.ng + P.nix // 2 - 1)
    row = M.getrow(g).toarray().ravel()
    h2 = P.h * P.h
    assert abs(row[g] - h2 / 2) <= 1e-12 * h2
    for d in (1, -1, nfx, -nfx, nfx + 1, -nfx - 1):
        assert abs(row[g + d] - h2 / 12) <= 1e-12 * h2
    assert abs(row.sum() - h2) <= 1e-12 * h2
    # a lumped mass would give b = h^2 f at interior nodes: far from b
    assert np.max(np.abs(b - h2 * f)) > 1e-4 * np.max(np.abs(ref))


def _row_tris_in_box(s, gi, gj):
    """all six triangles around node (gi, gj) lie inside the int box"""
    return (s["int_lo"][0] <= gi - 1 and gi + 1 <= s["int_hi"][0]
            and s["int_lo"][1] <= gj - 1 and gj + 1 <= s["int_hi"][1])


@pytest.mark.parametrize("sub", [0, 5, 10])
def test_local_rows_equal_global_rows_in_int_box(sub):
    """a_j = a restricted to H^1_0(Omega_j) with g_j = g_i inside the int box."""
    o = Oracle.from_config(k=100, nsub_x=4, nsub_y=4)
    A7 = o.stencil()
    band, p = o.local_band(sub)
    s = o.subdomain(sub)
    mx, my = s["m"]
    nfx = o.nf[0]
    checked = 0
    for ly in range(2, my):
        for lx in range(2, mx):
            gi, gj = s["full_lo"][0] + lx, s["full_lo"][1] + ly
            if not _row_tris_in_box(s, gi, gj):
                continue
            r = (lx - 1) + mx * (ly - 1)
            g = (gi - 1) + nfx * (gj - 1)
            for sl, (dx, dy) in enumerate(SLOTS):
                assert band[r, dx + mx * dy + p] == A7[g, sl]
            checked += 1
    assert checked > 100


@pytest.mark.parametrize("k,nsub,sub", [(400.0, 16, 5 + 16 * 7), (1600.0, 64, 20 + 64 * 31)])
def test_interior_local_problem_is_a_shifted_global_problem(k, nsub, sub):
    """An interior subdomain's local problem (int box + kappa local PML) is exactly the global PML
    problem of P:36-62 posed on Omega_int := int box with kappa PML cells (same profile, D3).  At c3 the
    12-cell local layer exercises the linear continuation beyond kappa_g = 10 h."""
    o = Oracle.from_config(k=k, nsub_x=nsub, nsub_y=nsub)
    s = o.subdomain(sub)
    assert s["has_lo"] == (1, 1) and s["has_hi"] == (1, 1)
    P = o.prob
    g = Oracle(Problem(k=P.k, sigma0=P.sigma0, h=P.h,
                       nix=s["int_hi"][0] - s["int_lo"][0], niy=s["int_hi"][1] - s["int_lo"][1],
                       ng=P.npml, kappa=P.kappa, px=1, py=1, novlp=P.novlp, npml=P.npml))
    band, p = o.local_band(sub)
    mx, my = s["m"]
    assert (mx, my) == g.nf
    G7 = g.stencil()
    for r in range(mx * my):
        lx, ly = r % mx, r // mx
        for sl, (dx, dy) in enumerate(SLOTS):
            if 0 <= lx + dx < mx and 0 <= ly + dy < my:
                a = band[r, dx + mx * dy + p]
                assert abs(a - G7[r, sl]) <= 1e-14 * max(1.0, abs(a)), (r, sl)


def test_interior_local_matrices_translation_invariant():
    """D5: depth from integer offsets => interior A_j of one size class are bitwise identical."""
    o = Oracle.from_config(k=400, nsub_x=16, nsub_y=16)
    sizes = {}
    for sub in [3 + 16 * 4, 9 + 16 * 4, 9 + 16 * 11, 12 + 16 * 8]:
        s = o.subdomain(sub)
        sizes.setdefault(s["m"], []).append(o.local_band(sub)[0])
    assert any(len(v) > 1 for v in sizes.values())
    for v in sizes.values():
        for b in v[1:]:
            assert np.array_equal(b, v[0])


def _manufactured_error(n):
    """sigma0 = 0, k = 1, u = sin(pi (x+kg)/L) sin(pi (y+kg)/L) on Omega = (-kg, 1+kg)^2: f = (2 pi^2/L^2 - k^2) u."""
    k = 1.0
    h = 1.0 / n
    ng = max(1, n // 10)
    o = Oracle(Problem(k=k, sigma0=0.0, h=h, nix=n, niy=n, ng=ng, kappa=ng * h, px=1, py=1, novlp=2, npml=2))
    import scipy.sparse.linalg as sla
    A = o.matrix().tocsc()
    nfx, nfy = o.nf
    idx = np.arange(o.nfree)
    x = (idx % nfx + 1 - ng) * h
    y = (idx // nfx + 1 - ng) * h
    L = 1 + 2 * ng * h
    kg = ng * h
    u = np.sin(np.pi * (x + kg) / L) * np.sin(np.pi * (y + kg) / L)
    f = (2 * np.pi ** 2 / L ** 2 - k * k) * u
    # b = M f_I through the oracle's rhs path is for Gaussians; assemble M f here from the definition
    M = (o.matrix() - Oracle(Problem(k=0.0, sigma0=0.0, h=h, nix=n, niy=n, ng=ng, kappa=ng * h, px=1, py=1,
                                     novlp=2, npml=2)).matrix()) / (-k * k)
    uh = sla.spsolve(A, M @ f)
    e = uh - u
    return math.sqrt(np.real(np.vdot(e, M @ e))) / math.sqrt(np.real(np.vdot(u, M @ u)))


def test_fem_order_two():
    """P1 L2 error is O(h^2)."""
    e1, e2, e3 = _manufactured_error(10), _manufactured_error(20), _manufactured_error(40)
    r1, r2 = math.log2(e1 / e2), math.log2(e2 / e3)
    assert 1.8 < r1 < 2.2 and 1.8 < r2 < 2.2, (e1, e2, e3)

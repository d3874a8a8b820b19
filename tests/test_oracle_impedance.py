"""Oracle pins for RAS-PML-Imp (eq. impedance): on every face of Omega_j that is not
on dOmega the local problem carries d_nu u - i k u = 0 as a natural boundary condition, adding
-i k int_face u v to a_j (edge mass h/6 [[2,1],[1,2]], no PML metric).  -m "not gpu"."""
import math

import numpy as np
import pytest

from oracle.oracle import Oracle, Problem, gmres, problem_from_config
from paper_2602_00735_b200.workloads import CONFIGS, sources


def _dense(o, j):
    return o.local_matrix(j)


def test_face_nodes_become_free():
    d = Oracle.from_config(k=1600, nsub_x=64, nsub_y=64)
    i = Oracle.from_config(k=1600, nsub_x=64, nsub_y=64, local_bc=1)
    for j in [0, 1, 64 * 31 + 30, 4095]:
        sd, si = d.subdomain(j), i.subdomain(j)
        for ax in range(2):
            assert si["m"][ax] == sd["m"][ax] + si["has_lo"][ax] + si["has_hi"][ax]
            assert si["node0"][ax] == sd["node0"][ax] - si["has_lo"][ax]
    assert i.subdomain(64 * 31 + 30)["m"] in [(89, 89), (89, 90), (90, 89), (90, 90)]


def test_single_subdomain_has_no_impedance_face():
    a = Oracle.from_config(k=20, local_bc=0)
    b = Oracle.from_config(k=20, local_bc=1)
    assert np.array_equal(a.local_band(0)[0], b.local_band(0)[0])


def _small(k, local_bc):
    h = 1.0 / 24
    return Oracle(Problem(k=k, sigma0=5.0, h=h, nix=24, niy=24, ng=4, kappa=4 * h, px=3, py=2, novlp=2, npml=2,
                          local_bc=local_bc))


@pytest.mark.parametrize("sub", [0, 1, 4])
def test_impedance_term_is_the_edge_mass(sub):
    """A_j(k) = K - k^2 M - i k B exactly (D, beta do not depend on k): recover B from three wavenumbers and
    check it is the P1 edge mass of the impedance faces: real, symmetric, supported on face nodes,
    row sums h along a face, total = total face length."""
    A1, A2, A3 = (_dense(_small(k, 1), sub) for k in (1.0, 2.0, 3.0))
    # A(k) = K + k C + k^2 Q  ->  C = (-3 A1 + 4 A2 - A3)/2 ... solve the 3x3 Vandermonde per entry
    V = np.array([[1, 1, 1], [1, 2, 4], [1, 3, 9]], float)
    Vi = np.linalg.inv(V)
    C = Vi[1, 0] * A1 + Vi[1, 1] * A2 + Vi[1, 2] * A3
    B = C / (-1j)
    assert np.max(np.abs(B.imag)) < 1e-12 and np.allclose(B, B.T, atol=1e-14)
    B = B.real
    o = _small(1.0, 1)
    s = o.subdomain(sub)
    h = o.prob.h
    mx, my = s["m"]
    face = np.zeros(mx * my, bool)
    length = 0.0
    for ax in range(2):
        for side, key in ((0, "has_lo"), (1, "has_hi")):
            if not s[key][ax]:
                continue
            f = s["full_hi"][ax] if side else s["full_lo"][ax]
            o_ax = 1 - ax
            length += (s["full_hi"][o_ax] - s["full_lo"][o_ax]) * h
            for q in range(s["full_lo"][o_ax], s["full_hi"][o_ax] + 1):
                node = [0, 0]
                node[ax], node[o_ax] = f, q
                lx, ly = node[0] - s["node0"][0], node[1] - s["node0"][1]
                if 0 <= lx < mx and 0 <= ly < my:
                    face[lx + mx * ly] = True
    off = ~face
    assert np.max(np.abs(B[off, :])) < 1e-13 and np.max(np.abs(B[:, off])) < 1e-13
    rs = B.sum(axis=1)
    assert np.any(np.isclose(rs[face], h, rtol=1e-12))          # nodes inside a face: two edges of h/2 each
    # total = face length minus the edges whose far end is a Dirichlet node on dOmega (those couplings drop)
    assert B.sum() <= length * (1 + 1e-12) and B.sum() > 0.8 * length
    assert np.all(np.diag(B)[face] > 0)


def _plane_wave_face_residual(n):
    """sigma0 = 0 (no absorption), subdomain 0 of a 2 x 1 split has one impedance face (x = full_hi, nu = +x).
    u = exp(i k x) satisfies Delta u + k^2 u = 0 and d_nu u - i k u = 0 there: the discrete residual on the
    face rows must vanish under refinement; the opposite sign would leave |2 i k u| h / 2 per row."""
    k = 6.0
    h = 1.0 / n
    o = Oracle(Problem(k=k, sigma0=0.0, h=h, nix=n, niy=n, ng=2, kappa=2 * h, px=2, py=1, novlp=3, npml=3,
                       local_bc=1))
    s = o.subdomain(0)
    A = o.local_matrix(0)
    mx, my = s["m"]
    lx = np.arange(mx)
    x = (s["node0"][0] + lx - o.prob.ng) * h
    u = np.tile(np.exp(1j * k * x), my)
    r = A @ u
    fx = s["full_hi"][0] - s["node0"][0]
    rows = [fx + mx * ly for ly in range(3, my - 3)]
    return np.max(np.abs(r[rows])) / (k * h)


def test_impedance_plane_wave_consistency():
    e = [_plane_wave_face_residual(n) for n in (24, 48, 96)]
    assert e[0] < 0.1 and e[1] < e[0] / 1.8 and e[2] < e[1] / 1.8, e


@pytest.mark.parametrize("name", ["c0", "c1"])
def test_imp_preconditioner_converges_and_is_not_worse(name):
    """Paper Tables 1-2: RAS-PML-Imp iterates no more than RAS-PML-Drch."""
    cfg = CONFIGS[name]
    its = {}
    for bc in (0, 1):
        o = Oracle.from_config(k=cfg.k, nsub_x=cfg.nsub, nsub_y=cfg.nsub, local_bc=bc)
        o.factor()
        xy, amp, sig = sources(cfg)
        b = o.rhs(xy, amp, sig)
        r = gmres(o.matvec, o.apply, b, restart=50, rtol=1e-6)
        assert r.status == 0
        its[bc] = r.iterations
    assert its[1] <= its[0] + 1, its

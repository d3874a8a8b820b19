"""Oracle pins for the paper's own workload (D18-D22): Q1 elements, the
paper frame Omega = (0,1)^2 with a 3-wavelength global PML and g(x) = 10 k x^3, the smoothed delta
source, and the iteration counts the paper prints in Tables 1, 3 and 4 (tests/golden/
paper_iterations.txt).  -m "not gpu"."""
import math
import os

import numpy as np
import pytest
import scipy.sparse.linalg as sla

from oracle.oracle import Oracle, Problem, gmres, lib, richardson, _ptr
from paper_2602_00735_b200.workloads import PAPER_CONFIGS, paper_source, probe_vector

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "paper_iterations.txt")


def golden_rows():
    rows = []
    with open(GOLDEN) as f:
        for line in f:
            if line.startswith("#") or not line.strip():
                continue
            t, ln, k, grid, P, pml, ov, bc, solver, its, rr = line.split()
            rows.append(dict(table=t, line=int(ln), k=float(k), grid=int(grid), nsub=int(P), pml=int(pml),
                             ovlp=int(ov), bc={"drch": 0, "imp": 1, "rasimp": 2}[bc], solver=solver, its=int(its)))
    return rows


def small_paper(k=100.0, nsub=2, pml=6, ovlp=3, bc=1, pml_c=None, pou=1):
    return Oracle.from_paper(k=k, nsub=nsub, pml=pml, ovlp=ovlp, local_bc=bc, pml_c=pml_c, pou=pou)


# ------------------------------------------------------------------------------------------ assembly
def test_q1_interior_stencil_closed_form():
    """Q1 on a square cell with D = I, beta = 0 (inside Omega_int): stiffness 8/3 centre and -1/3 on all eight
    neighbours; consistent mass h^2/36 (16, 4, 1); so centre 8/3 - 4 (kh)^2/9, edge -1/3 - (kh)^2/9, corner
    -1/3 - (kh)^2/36 and row sum -(kh)^2 (textbook bilinear stencils)."""
    o = small_paper()
    A9 = o.stencil()
    nf = o.nf[0]
    kh = o.prob.k * o.prob.h
    r = nf // 2 + nf * (nf // 2)
    want = [8 / 3 - 4 * kh ** 2 / 9] + [-1 / 3 - kh ** 2 / 9] * 4 + [-1 / 3 - kh ** 2 / 36] * 4
    assert np.allclose(A9[r], want, rtol=0, atol=1e-14)
    assert abs(A9[r].sum() + kh ** 2) <= 1e-13


def test_q1_symmetry_structure():
    """Without the PML (pml_c = 0) A = A^T exactly; with it, A - A^T is nonzero only on rows whose four cells
    include a PML quadrature point (the beta term of eq. (weak), D7)."""
    A0 = small_paper(pml_c=0.0).matrix()
    assert abs(A0 - A0.T).max() == 0.0
    o = small_paper()
    A = o.matrix()
    D = (A - A.T).tocoo()
    nf = o.nf[0]
    lo = o.prob.kappa / o.prob.h
    hi = o.nf[0] + 1 - lo
    bad = D.row[np.abs(D.data) > 0]
    i, j = bad % nf + 1, bad // nf + 1
    inside = (i - 1 > lo) & (i + 1 < hi) & (j - 1 > lo) & (j + 1 < hi)
    assert bad.size > 0 and not inside.any()


def test_paper_profile_closed_forms_and_sides():
    """g(t) = 10 k t^3: gamma = 1 + i 30 k t^2, gamma' = +i 60 k t above Omega_int and -i 60 k t below
    (g_i = -g(a - x); D4); gamma = 1 inside Omega_int; gamma' is the derivative of gamma."""
    o = small_paper()
    k, h = o.prob.k, o.prob.h
    lo = o.prob.kappa
    g, dg = o.gamma_q(0, o.N[0] // 2, 0.5)
    assert g == 1 and dg == 0
    ci, xi = o.N[0] - 3, 0.25                     # above 1 - kappa_g
    x = (ci + xi) * h
    t = x - (1.0 - lo)
    g, dg = o.gamma_q(0, ci, xi)
    assert abs(g - (1 + 30j * k * t * t)) <= 1e-12 * abs(g) and abs(dg - 60j * k * t) <= 1e-12 * abs(dg)
    g, dg = o.gamma_q(1, 2, xi)                   # below kappa_g
    t = lo - (2 + xi) * h
    assert abs(g - (1 + 30j * k * t * t)) <= 1e-12 * abs(g) and abs(dg + 60j * k * t) <= 1e-12 * abs(dg)
    eps = 1e-4
    for ci in (1, o.N[0] - 2):
        gp, _ = o.gamma_q(0, ci, 0.5 + eps)
        gm, _ = o.gamma_q(0, ci, 0.5 - eps)
        _, d = o.gamma_q(0, ci, 0.5)
        assert abs((gp - gm) / (2 * eps * h) - d) <= 1e-6 * abs(d)


def test_paper_local_ramps():
    """Local scaling g_j: beyond the int box faces of subdomain j the ramp restarts from b_j (upper) /
    a_j (lower) with the same g; inside the int box it is the global g_i."""
    o = small_paper(nsub=3)
    k, h = o.prob.k, o.prob.h
    j = 4                                           # the centre subdomain: local PML on all four faces
    s = o.subdomain(j)
    b = s["int_hi"][0]
    g, dg = o.gamma_q(0, b + 2, 0.5, sub=j)
    t = 2.5 * h
    assert abs(g - (1 + 30j * k * t * t)) <= 1e-12 * abs(g) and abs(dg - 60j * k * t) <= 1e-12 * abs(dg)
    a = s["int_lo"][1]
    g, dg = o.gamma_q(1, a - 3, 0.25, sub=j)
    t = 2.75 * h
    assert abs(g - (1 + 30j * k * t * t)) <= 1e-12 * abs(g) and abs(dg + 60j * k * t) <= 1e-12 * abs(dg)
    assert o.gamma_q(0, b - 1, 0.5, sub=j) == o.gamma_q(0, b - 1, 0.5)


def test_q1_local_rows_equal_global_rows_in_int_box():
    """Rows of A_j whose four cells lie inside the int box, where g_j = g_i, equal the rows of A."""
    o = small_paper(nsub=3)
    A = o.matrix().tocsr()
    nf = o.nf[0]
    for j in (0, 4, 8):
        s = o.subdomain(j)
        Aj = o.local_matrix(j)
        mx, my = s["m"]
        n0x, n0y = s["node0"]
        for ly in range(my):
            for lx in range(mx):
                gi, gj = n0x + lx, n0y + ly
                if not (s["int_lo"][0] + 1 <= gi <= s["int_hi"][0] - 1 and s["int_lo"][1] + 1 <= gj <= s["int_hi"][1] - 1):
                    continue
                if not (2 <= gi <= nf - 1 and 2 <= gj <= nf - 1):
                    continue
                if (lx in (0, mx - 1)) or (ly in (0, my - 1)):
                    continue
                r = lx + mx * ly
                g = (gi - 1) + nf * (gj - 1)
                for dx, dy in Oracle.OFFSETS:
                    assert Aj[r, (lx + dx) + mx * (ly + dy)] == A[g, (gi + dx - 1) + nf * (gj + dy - 1)]


def test_q1_fem_order_two():
    """Manufactured u = sin(pi x) sin(pi y) on Omega = (0,1)^2 with no PML (pml_c = 0), k = 1: -Lap u - k^2 u = f,
    f = (2 pi^2 - k^2) u, b = M f_I.  The Q1 discrete L2 error falls ~4x per refinement (order 2)."""
    errs = []
    for n in (16, 32, 64):
        o = Oracle(Problem(k=1.0, sigma0=0.0, h=1.0 / n, nix=n, niy=n, ng=0, kappa=0.0, px=1, py=1, novlp=0, npml=0,
                           local_bc=0, pou=0, elem=1, frame=1, pml_c=0.0))
        x = np.arange(1, n) / n
        X, Y = np.meshgrid(x, x, indexing="xy")
        u = (np.sin(np.pi * X) * np.sin(np.pi * Y)).ravel()
        A = o.matrix()                  # A = K - k^2 M, k = 1
        f = (2 * np.pi ** 2 - 1.0) * u
        # b = M f_I with the consistent Q1 mass M = K - A, K = the k = 0 operator
        o0 = Oracle(Problem(k=0.0, sigma0=0.0, h=1.0 / n, nix=n, niy=n, ng=0, kappa=0.0, px=1, py=1, novlp=0,
                            npml=0, local_bc=0, pou=0, elem=1, frame=1, pml_c=0.0))
        Mass = o0.matrix() - A
        uh = sla.spsolve(A.tocsc(), Mass @ f)
        errs.append(np.linalg.norm(uh - u) / n)
    r1, r2 = errs[0] / errs[1], errs[1] / errs[2]
    assert 3.6 <= r1 <= 4.4 and 3.6 <= r2 <= 4.4, errs


def test_q1_rhs_matches_mass_matrix_and_unit_mass():
    """b = M f_I (D14 carried over): equals the Q1 consistent mass matrix (recovered as (A(0) - A(k')) / k'^2 with
    k' h = 1, no PML) times f at the nodes, and the smoothed delta of P:217-218 has unit mass: sum b = 1."""
    k = 100.0
    o = small_paper(k=k)
    xy, amp, s = paper_source(k)
    b = o.rhs(xy, amp, s)
    assert abs(b.sum() - 1.0) <= 1e-9
    n = o.N[0]
    o1 = Oracle(Problem(k=float(n), sigma0=0.0, h=1.0 / n, nix=n, niy=n, ng=0, kappa=0.0, px=1, py=1, novlp=0,
                        npml=0, local_bc=0, pou=0, elem=1, frame=1, pml_c=0.0))
    o0 = Oracle(Problem(k=0.0, sigma0=0.0, h=1.0 / n, nix=n, niy=n, ng=0, kappa=0.0, px=1, py=1, novlp=0, npml=0,
                        local_bc=0, pou=0, elem=1, frame=1, pml_c=0.0))
    Mass = (o0.matrix() - o1.matrix()) / float(n) ** 2
    x = np.arange(1, n) / n
    X, Y = np.meshgrid(x, x, indexing="xy")
    f = (1.0 / (2 * math.pi * s * s)) * np.exp(-((X - 0.5) ** 2 + (Y - 0.5) ** 2) / (2 * s * s))
    assert np.linalg.norm(b - Mass @ f.ravel()) <= 1e-12 * np.linalg.norm(b)


# ------------------------------------------------------------------------------------------ local solves / apply
def test_q1_band_lu_vs_lapack():
    """Naive band LU (half-bandwidth m + 1 covers NW/SE at m -/+ 1) vs zgesv on <= 400-unknown Q1 local systems."""
    o = Oracle.from_paper(k=60.0, nsub=3, pml=3, ovlp=2, local_bc=1)
    for j in (0, 4):
        A = o.local_matrix(j)
        assert A.shape[0] <= 3000
        band, p = o.local_band(j)
        b = np.random.default_rng(j).standard_normal(A.shape[0]) + 0j
        zr = lib().orc_band_lu(A.shape[0], p, _ptr(band))
        assert zr < 0
        x = b.copy()
        lib().orc_band_solve(A.shape[0], p, _ptr(band), _ptr(x))
        assert np.linalg.norm(x - np.linalg.solve(A, b)) <= 1e-11 * np.linalg.norm(x)


def test_q1_single_subdomain_is_exact_inverse():
    o = Oracle.from_paper(k=60.0, nsub=1, pml=3, ovlp=2)
    o.factor()
    v = probe_vector(o.nfree, 5)
    z = o.apply(v)
    assert np.linalg.norm(o.matvec(z) - v) <= 1e-11 * np.linalg.norm(v)


def test_q1_dense_ramp_preconditioner():
    """sum_j R~_j^T A_j^-1 R_j v with the linear-ramp weights chi_j, each A_j^-1 from
    numpy.linalg.inv of the dense local matrix and R_j / R~_j from the layout definitions (D11), equals the
    apply, for the impedance and Dirichlet local faces."""
    for bc in (1, 0):
        o = Oracle.from_paper(k=40.0, nsub=2, pml=3, ovlp=2, local_bc=bc)
        o.factor()
        n, nfx = o.nfree, o.nf[0]
        v = probe_vector(n, 9)
        z = np.zeros(n, np.complex128)
        for j in range(o.nsub):
            s = o.subdomain(j)
            mx, my = s["m"]
            n0x, n0y = s["node0"]
            bx, by = j % 2, j // 2
            gl, w = [], []
            for ly in range(my):
                for lx in range(mx):
                    gi, gj = n0x + lx, n0y + ly
                    gl.append((gi - 1) + nfx * (gj - 1))
                    w.append(o.chi(0, bx, gi) * o.chi(1, by, gj))
            gl = np.array(gl)
            z[gl] += np.array(w) * (np.linalg.inv(o.local_matrix(j)) @ v[gl])
        zo = o.apply(v)
        assert np.linalg.norm(zo - z) <= 1e-11 * np.linalg.norm(z)


# ------------------------------------------------------------------------------------------ printed iteration counts
@pytest.mark.parametrize("row", [r for r in golden_rows() if r["k"] == 300 and r["solver"] == "richardson"
                                 and r["table"] in ("Table1", "Table4") and r["bc"] != 2],
                         ids=lambda r: f"{r['table']}-{'imp' if r['bc'] else 'drch'}-pml{r['pml']}-ovlp{r['ovlp']}")
def test_paper_richardson_iterations_k300(row):
    """Algorithm 1 on the paper's k = 300 workload reproduces the iteration count printed in Tables 1 / 4
    (P:254): RAS-PML-Imp 12 and RAS-PML-Drch 13 with pml 8 / ovlp 4; 7 with pml 12 / ovlp 4."""
    k = row["k"]
    o = Oracle.from_paper(k=k, nsub=row["nsub"], pml=row["pml"], ovlp=row["ovlp"], local_bc=row["bc"],
                          n_cells=row["grid"])
    o.factor()
    xy, amp, s = paper_source(k)
    b = o.rhs(xy, amp, s)
    r = richardson(o.matvec, o.apply, b, rtol=1e-10, maxit=500)
    assert r.status == 0 and r.iterations == row["its"], (r.iterations, r.relres)
    assert r.relres < 1e-10
    o.close()


def test_paper_configs_match_golden():
    """workloads.PAPER_CONFIGS carries the table rows' integers (k, grid, N, pml, ovlp)."""
    rows = golden_rows()
    for c in PAPER_CONFIGS.values():
        if c.name.startswith("p"):
            hit = [r for r in rows if r["table"] == "Table1" and r["k"] == c.k]
        else:
            hit = [r for r in rows if r["table"] == "Table4" and r["k"] == c.k]
        for r in hit:
            assert (r["grid"], r["nsub"], r["pml"], r["ovlp"]) == (c.n_cells, c.nsub, c.pml, c.ovlp)


def test_paper_frame_hankel_far_field_and_refinement():
    """Physics pin of the whole paper frame (Q1, g = 10 k x^3, kappa_g = 3 lambda, smoothed delta): the
    direct solve approaches the outgoing free-space field e^{-k^2 s^2/2} (i/4) H0(k r) of the unit Gaussian (the
    Gaussian's Fourier transform at |xi| = k gives the factor) on lambda <= r <= 1/2 - kappa_g - lambda/2, with the
    error falling ~4x per mesh doubling (k = 60: 6.0 %, 1.55 %, 0.41 % at n = 2k, 4k, 8k)."""
    from scipy.special import hankel1
    k = 60.0
    errs = []
    for mult in (2, 4, 8):
        n = int(round(mult * k))
        o = Oracle.from_paper(k=k, nsub=1, pml=2, ovlp=1, n_cells=n)
        xy, amp, s = paper_source(k)
        u = sla.spsolve(o.matrix().tocsc(), o.rhs(xy, amp, s))
        nf = o.nf[0]
        idx = np.arange(o.nfree)
        x, y = (idx % nf + 1) / n, (idx // nf + 1) / n
        r = np.hypot(x - 0.5, y - 0.5)
        lam = 2 * math.pi / k
        sel = (r >= lam) & (r <= 0.5 - o.prob.kappa - lam / 2)
        ref = math.exp(-(k * s) ** 2 / 2) * 0.25j * hankel1(0, k * r[sel])
        errs.append(np.linalg.norm(u[sel] - ref) / np.linalg.norm(ref))
    assert errs[0] < 0.1
    assert errs[0] / errs[1] > 3.3 and errs[1] / errs[2] > 3.3, errs
    assert errs[2] < 0.006


@pytest.mark.parametrize("sub", [0, 1, 3])
def test_q1_impedance_term_is_the_edge_mass(sub):
    """RAS-PML-Imp with Q1: with the PML profile held fixed (g = c t^3, c not tied to k) the local matrix
    is A_j(k) = K + k C + k^2 M exactly, and C = -i B with B the edge mass of the impedance faces -- for bilinear
    elements the 1-D linear mass (h/6)[[2,1],[1,2]] per edge: real, symmetric, only on face nodes, row sums h for
    nodes inside a face, positive diagonal.  Three wavenumbers recover B entrywise (Vandermonde)."""
    def make(k):
        h = 1.0 / 20
        return Oracle(Problem(k=float(k), sigma0=0.0, h=h, nix=20, niy=20, ng=0, kappa=4 * h, px=2, py=2, novlp=2,
                              npml=2, local_bc=1, pou=1, elem=1, frame=1, pml_c=300.0))
    A1, A2, A3 = (make(k).local_matrix(sub) for k in (1.0, 2.0, 3.0))
    Vi = np.linalg.inv(np.array([[1, 1, 1], [1, 2, 4], [1, 3, 9]], float))
    C = Vi[1, 0] * A1 + Vi[1, 1] * A2 + Vi[1, 2] * A3
    B = C / (-1j)
    assert np.max(np.abs(B.imag)) < 1e-12 and np.allclose(B, B.T, atol=1e-14)
    B = B.real
    o = make(1.0)
    h = o.prob.h
    nz = np.abs(B) > 1e-13
    rows = np.where(nz.any(axis=1))[0]
    assert len(rows) > 0                                   # subdomain with impedance faces
    # only node pairs on a common face edge: every nonzero is 2h/6 (diagonal, one edge), 4h/6 (two edges) or h/6
    vals = np.unique(np.round(B[nz] / (h / 6), 9))
    assert set(vals).issubset({1.0, 2.0, 4.0})
    rs = B.sum(axis=1)[rows]
    assert np.any(np.isclose(rs, h, rtol=1e-12))           # a node inside a face: two edges, (2+1+2+1) h/6 = h
    assert np.all(np.diag(B)[rows] > 0)

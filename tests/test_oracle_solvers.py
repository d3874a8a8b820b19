"""Oracle pins: naive banded LU (O7, D12), the RAS-PML preconditioner (D10, D11),
right-preconditioned GMRES(50) (O9; D13) and the free-space physics.  -m "not gpu"."""
import math

import numpy as np
import pytest
import scipy.sparse.linalg as sla

from oracle.oracle import Oracle, OracleError, Problem, gmres, lib, problem_from_config, _ptr
from paper_2602_00735_b200.workloads import CONFIGS, probe_vector, sources


# ----------------------------------------------------------------------------------- band LU (O7)
def _band_from_dense(A, p):
    n = A.shape[0]
    band = np.zeros((n, 2 * p + 1), np.complex128)
    for r in range(n):
        for c in range(max(0, r - p), min(n, r + p + 1)):
            band[r, c - r + p] = A[r, c]
    return band


def _band_solve(A, p, b):
    band = _band_from_dense(A, p)
    zr = lib().orc_band_lu(A.shape[0], p, _ptr(band))
    if zr >= 0:
        raise ZeroDivisionError(zr)
    x = np.array(b, np.complex128)
    lib().orc_band_solve(A.shape[0], p, _ptr(band), _ptr(x))
    return x


@pytest.mark.parametrize("n,p", [(7, 1), (50, 6), (200, 15), (400, 21)])
def test_band_lu_matches_dense_gaussian_elimination(n, p):
    rng = np.random.default_rng(n)
    A = np.zeros((n, n), np.complex128)
    for r in range(n):
        for c in range(max(0, r - p), min(n, r + p + 1)):
            A[r, c] = rng.standard_normal() + 1j * rng.standard_normal()
        A[r, r] += 4 * p                    # no-pivot LU needs nonzero pivots; keep them well away from 0
    b = rng.standard_normal(n) + 1j * rng.standard_normal(n)
    x = _band_solve(A, p, b)
    xr = np.linalg.solve(A, b)
    assert np.linalg.norm(x - xr) <= 1e-12 * np.linalg.norm(xr)


def test_band_lu_small_examples():
    # S:263 diag(2, 3i)
    x = _band_solve(np.diag([2.0 + 0j, 3j]), 1, np.array([2.0, 3j]))
    assert np.allclose(x, [1.0, 1.0], rtol=0, atol=1e-15)
    # S:265 singular pivot -> error reporting the row
    A = np.array([[1.0, 2.0], [2.0, 4.0]], np.complex128)
    with pytest.raises(ZeroDivisionError) as e:
        _band_solve(A, 1, np.ones(2))
    assert e.value.args[0] == 1


def test_band_lu_on_a_local_helmholtz_matrix():
    """A real (small) local RAS-PML matrix, <= 400 unknowns, vs LAPACK zgesv with partial pivoting."""
    h = 1.0 / 24
    o = Oracle(Problem(k=20.0, sigma0=5.0, h=h, nix=24, niy=24, ng=4, kappa=4 * h, px=4, py=4, novlp=2, npml=2))
    for sub in [0, 5, 15]:
        A = o.local_matrix(sub)
        assert A.shape[0] <= 400
        s = o.subdomain(sub)
        rng = np.random.default_rng(sub)
        b = rng.standard_normal(A.shape[0]) + 1j * rng.standard_normal(A.shape[0])
        x = _band_solve(A, s["m"][0] + 1, b)
        xr = np.linalg.solve(A, b)
        assert np.linalg.norm(x - xr) <= 1e-12 * np.linalg.norm(xr)


# --------------------------------------------------------------------------- preconditioner (O8)
def test_single_subdomain_apply_is_exact_inverse():
    """N = 1 => B^-1 = A^-1 (north_star)."""
    o = Oracle.from_config(k=20, nsub_x=1, nsub_y=1)
    o.factor()
    v = probe_vector(o.nfree, 21)
    z = o.apply(v)
    zr = sla.spsolve(o.matrix().tocsc(), v)
    assert np.linalg.norm(z - zr) <= 1e-12 * np.linalg.norm(zr)


def test_dense_preconditioner_c0():
    """Dense sum_j R~_j^T A_j^-1 R_j, built from numpy.linalg.inv of each local matrix and restriction /
    owner-extension matrices built from the layout definitions (D10, D11), equals the apply."""
    cfg = CONFIGS["c0"]
    o = Oracle.from_config(k=cfg.k, nsub_x=2, nsub_y=2)
    o.factor()
    n = o.nfree
    nfx = o.nf[0]
    B = np.zeros((n, n), np.complex128)
    for j in range(o.nsub):
        s = o.subdomain(j)
        mx, my = s["m"]
        gl = [(s["full_lo"][0] + lx - 1) + nfx * (s["full_lo"][1] + ly - 1)
              for ly in range(1, my + 1) for lx in range(1, mx + 1)]
        R = np.zeros((mx * my, n))
        R[np.arange(mx * my), gl] = 1.0
        own = np.zeros(mx * my)
        for r, g in enumerate(gl):
            gi, gj = g % nfx + 1, g // nfx + 1
            own[r] = (s["own_lo"][0] <= gi < s["own_hi"][0]) and (s["own_lo"][1] <= gj < s["own_hi"][1])
        B += (R.T * own) @ np.linalg.inv(o.local_matrix(j)) @ R
    for seed in [1, 2]:
        v = probe_vector(n, seed)
        assert np.linalg.norm(o.apply(v) - B @ v) <= 1e-12 * np.linalg.norm(B @ v)


def test_apply_linearity_and_zero():
    o = Oracle.from_config(k=100, nsub_x=4, nsub_y=4)
    o.factor()
    v1, v2 = probe_vector(o.nfree, 1), probe_vector(o.nfree, 2)
    a = 0.3 - 1.7j
    lhs = o.apply(v1 + a * v2)
    rhs = o.apply(v1) + a * o.apply(v2)
    assert np.linalg.norm(lhs - rhs) <= 1e-12 * np.linalg.norm(rhs)
    assert np.all(o.apply(np.zeros(o.nfree)) == 0)


def test_apply_before_factor_raises():
    o = Oracle.from_config(k=20, nsub_x=2, nsub_y=2)
    with pytest.raises(OracleError):
        o.apply(np.zeros(o.nfree))


# ---------------------------------------------------------------------------------------- GMRES
def test_gmres_identity_one_iteration():
    b = probe_vector(30, 3)
    r = gmres(lambda x: x, lambda x: x, b)
    assert r.iterations == 1 and r.status == 0 and np.allclose(r.x, b)


def test_gmres_diag():
    b = np.array([1.0 + 1j, 2.0])
    r = gmres(lambda x: np.array([2.0, 1.0]) * x, lambda x: x, b, rtol=1e-12)
    assert r.iterations <= 2 and np.allclose(r.x, [0.5 + 0.5j, 2.0])


@pytest.mark.parametrize("restart", [50, 7])
def test_gmres_random_dense(restart):
    rng = np.random.default_rng(7)
    A = rng.standard_normal((20, 20)) + 1j * rng.standard_normal((20, 20)) + 8 * np.eye(20)
    b = rng.standard_normal(20) + 1j * rng.standard_normal(20)
    r = gmres(lambda x: A @ x, lambda x: x, b, restart=restart, rtol=1e-10)
    assert r.status == 0
    assert np.linalg.norm(r.x - np.linalg.solve(A, b)) <= 1e-8 * np.linalg.norm(r.x)
    if restart == 50:
        h = r.history
        assert all(h[i + 1] <= h[i] * (1 + 1e-12) for i in range(len(h) - 1))


def test_gmres_zero_rhs():
    r = gmres(lambda x: 2 * x, lambda x: x, np.zeros(5, np.complex128))
    assert r.iterations == 0 and np.all(r.x == 0)


def test_single_subdomain_gmres_one_iteration():
    o = Oracle.from_config(k=100, nsub_x=1, nsub_y=1)
    o.factor()
    xy, amp, sig = sources(CONFIGS["c1"])
    b = o.rhs(xy, amp, sig)
    r = gmres(o.matvec, o.apply, b)
    assert r.iterations == 1 and r.relres_true < 1e-12


@pytest.mark.parametrize("name", ["c0", "c1"])
def test_gmres_ras_vs_direct_solve(name):
    """RAS-PML-preconditioned GMRES(50) to 1e-6 vs scipy spsolve (D16)."""
    cfg = CONFIGS[name]
    o = Oracle.from_config(k=cfg.k, nsub_x=cfg.nsub, nsub_y=cfg.nsub)
    o.factor()
    xy, amp, sig = sources(cfg)
    b = o.rhs(xy, amp, sig)
    r = gmres(o.matvec, o.apply, b, restart=50, rtol=1e-6)
    assert r.status == 0 and r.relres_true <= 1e-6
    xd = sla.spsolve(o.matrix().tocsc(), b)
    assert np.linalg.norm(r.x - xd) <= 1e-5 * np.linalg.norm(xd)


# -------------------------------------------------------------------------------------- physics
def _hankel_error(k, ppw):
    """Single unit Gaussian at (0.5, 0.5), direct solve; compare with e^{-k^2 sigma^2/2} (i/4) H0(kr) on
    nodes with lambda <= r <= 0.5 - lambda/2 (outgoing free-space Green's function of P:26-32, the
    Gaussian's Fourier transform at |xi| = k giving the factor)."""
    from scipy.special import hankel1
    o = Oracle(problem_from_config(k, ppw=ppw, n_pml_global=ppw))
    sigma = (2 * math.pi / k) / 4
    b = o.rhs(np.array([[0.5, 0.5]]), np.array([1.0 + 0j]), sigma)
    u = sla.spsolve(o.matrix().tocsc(), b)
    nfx = o.nf[0]
    idx = np.arange(o.nfree)
    x = (idx % nfx + 1 - o.prob.ng) * o.prob.h
    y = (idx // nfx + 1 - o.prob.ng) * o.prob.h
    r = np.hypot(x - 0.5, y - 0.5)
    lam = 2 * math.pi / k
    sel = (r >= lam) & (r <= 0.5 - lam / 2)
    ref = math.exp(-(k * sigma) ** 2 / 2) * 0.25j * hankel1(0, k * r[sel])
    return np.linalg.norm(u[sel] - ref) / np.linalg.norm(ref)


def test_hankel_far_field_and_refinement():
    e = [_hankel_error(20.0, p) for p in (10, 20, 40)]
    assert e[0] < 0.2
    assert e[0] / e[1] > 3.0 and e[1] / e[2] > 3.0, e
    assert e[2] < 0.02


# ------------------------------------------------------------------------------------------ dedup mode
@pytest.mark.parametrize("name,classes", [("c1", 9), ("c2", 9)])
def test_dedup_apply_is_bitwise_the_per_subdomain_apply(name, classes):
    """Memory fallback: factoring one representative per bitwise-distinct A_j is exact -- the apply is bitwise
    the one with every subdomain factored separately.  Classes are {first, interior, last} per axis at c1/c2
    (blocks 45/45/45/44 and 42/41x15: the interior sizes share one matrix because the int box and local PML
    have the same widths; D5's integer-offset depth makes them bitwise equal)."""
    cfg = CONFIGS[name]
    o = Oracle.from_config(k=cfg.k, nsub_x=cfg.nsub, nsub_y=cfg.nsub)
    assert o.factor_dedup() == classes
    v = probe_vector(o.nfree, int(cfg.k) + 1)
    z1 = o.apply(v)
    reps = {o.dedup_class(j)[1] for j in range(o.nsub)}
    assert len(reps) == classes and sum(o.dedup_class(r)[2] for r in reps) == o.nsub
    o.release()
    o.factor()
    assert np.array_equal(z1, o.apply(v))


def test_dedup_counts_one_class_per_distinct_matrix():
    """With a single block per axis there is one class; with ramps/impedance (other matrices) the classes follow the
    local matrices, and the member == representative assertion holds for every subdomain."""
    o = Oracle(problem_from_config(20.0))
    assert o.factor_dedup() == 1
    o = Oracle(problem_from_config(100.0, nsub_x=4, nsub_y=4, local_bc=1))
    assert o.factor_dedup() == 9
    o = Oracle(problem_from_config(100.0, nsub_x=5, nsub_y=3))
    assert o.factor_dedup() == 9


def test_impedance_face_on_the_boundary_is_refused():
    """with RAS-PML-Imp the full-box face nodes are local unknowns, so a block of exactly delta + kappa
    cells next to dOmega would put the Dirichlet node 0 (or N) into Omega_j.  The oracle refuses that layout (the
    Dirichlet variant of the same layout is valid)."""
    k = 6 * math.pi          # n_int = 30, N = 50: ten blocks of 5 = delta + kappa cells
    Oracle(problem_from_config(k, nsub_x=10, nsub_y=2, n_ovlp=2, n_pml=3, local_bc=0))
    with pytest.raises(OracleError):
        Oracle(problem_from_config(k, nsub_x=10, nsub_y=2, n_ovlp=2, n_pml=3, local_bc=1))


@pytest.mark.parametrize("name", ["c0", "c1"])
def test_committed_golden_records_are_the_oracles(name):
    """tests/golden/<cfg>_gmres.json was written by scripts/make_golden.py from the oracle alone: re-running the oracle
    reproduces its iterations, history and solution sketch (no expected value comes from the CUDA path)."""
    import json
    import os
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "scripts"))
    from make_golden import sketch
    with open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", f"{name}_gmres.json")) as f:
        g = json.load(f)
    cfg = CONFIGS[name]
    o = Oracle.from_config(k=cfg.k, nsub_x=cfg.nsub, nsub_y=cfg.nsub)
    o.factor_dedup()
    b = o.rhs(*sources(cfg))
    res = gmres(o.matvec, o.apply, b, restart=cfg.restart, rtol=cfg.rtol, maxit=g["maxit"])
    assert res.iterations == g["iterations"] and res.status == g["status"]
    assert np.allclose(res.history, g["history"], rtol=1e-12, atol=0)
    s = sketch(res.x, g["sketch_rows"])
    ref = np.array([complex(a, c) for a, c in g["sketch_x"]])
    assert np.allclose(s, ref, rtol=1e-12, atol=1e-12 * np.abs(ref).max())

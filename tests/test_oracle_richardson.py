"""Oracle pins for Algorithm 1 (RAS_IterSolve; discrete form P:130-142) and the paper's practical
improvement (i): the residual of the local problems is nonzero only next to the subdomain interfaces
(P:182-184).  -m "not gpu"."""
import numpy as np
import pytest

from oracle.oracle import Oracle, richardson
from paper_2602_00735_b200.workloads import CONFIGS, probe_vector, sources


def test_single_subdomain_one_iteration():
    o = Oracle.from_config(k=20, nsub_x=1, nsub_y=1)
    o.factor()
    xy, amp, sig = sources(CONFIGS["c0"])
    b = o.rhs(xy, amp, sig)
    r = richardson(o.matvec, o.apply, b, rtol=1e-10)
    assert r.iterations == 1 and r.relres < 1e-12 and r.status == 0


def test_divergence_flag():
    """x_{n+1} = x_n + (b - 3 x_n): error factor -2 per step -> relres passes 1e6."""
    b = probe_vector(10, 4)
    r = richardson(lambda x: 3 * x, lambda x: x, b, rtol=1e-8, maxit=100)
    assert r.status == 3 and r.relres > 1e6 and r.iterations < 30


def test_contraction_matches_linear_algebra():
    """Richardson on a small SPD-like system converges to the dense solution."""
    rng = np.random.default_rng(3)
    A = np.eye(12) * 4 + 0.3 * (rng.standard_normal((12, 12)) + 1j * rng.standard_normal((12, 12)))
    b = rng.standard_normal(12) + 1j * rng.standard_normal(12)
    r = richardson(lambda x: A @ x, lambda x: x / 4, b, rtol=1e-12, maxit=200)
    assert r.status == 0 and np.allclose(r.x, np.linalg.solve(A, b), atol=1e-10)


def _band_mask(o):
    """Nodes whose 7-point stencil reaches a node owned by another block (the interface band)."""
    nfx, nfy = o.nf
    owner = np.full((nfy + 2, nfx + 2), -1)
    for j in range(o.nsub):
        s = o.subdomain(j)
        owner[s["own_lo"][1]:s["own_hi"][1], s["own_lo"][0]:s["own_hi"][0]] = j
    band = np.zeros(o.nfree, bool)
    for gj in range(1, nfy + 1):
        for gi in range(1, nfx + 1):
            me = owner[gj, gi]
            for dx, dy in [(1, 0), (-1, 0), (0, 1), (0, -1), (1, 1), (-1, -1)]:
                qi, qj = gi + dx, gj + dy
                if 1 <= qi <= nfx and 1 <= qj <= nfy and owner[qj, qi] != me:
                    band[(gi - 1) + nfx * (gj - 1)] = True
    return band


@pytest.mark.parametrize("name", ["c0", "c1"])
def test_residual_lives_on_the_interfaces(name):
    """after any Richardson step, f - A u vanishes on every node whose stencil stays
    inside its own block -- there a_j = a and the local solve satisfied the equation exactly."""
    cfg = CONFIGS[name]
    o = Oracle.from_config(k=cfg.k, nsub_x=cfg.nsub, nsub_y=cfg.nsub)
    o.factor()
    xy, amp, sig = sources(cfg)
    b = o.rhs(xy, amp, sig)
    band = _band_mask(o)
    x = np.zeros_like(b)
    for _ in range(3):
        x = x + o.apply(b - o.matvec(x))
        r = b - o.matvec(x)
        assert np.max(np.abs(r[~band])) <= 1e-12 * np.linalg.norm(b)
        assert np.max(np.abs(r[band])) > 1e-6 * np.linalg.norm(b)      # the band does carry the residual
    assert band.mean() < 0.2


def test_ras_richardson_converges_c1():
    cfg = CONFIGS["c1"]
    o = Oracle.from_config(k=cfg.k, nsub_x=cfg.nsub, nsub_y=cfg.nsub)
    o.factor()
    xy, amp, sig = sources(cfg)
    b = o.rhs(xy, amp, sig)
    r = richardson(o.matvec, o.apply, b, rtol=1e-6, maxit=300)
    assert r.status == 0
    assert all(h1 < h0 for h0, h1 in zip(r.history[5:], r.history[6:]))   # monotone once transients pass

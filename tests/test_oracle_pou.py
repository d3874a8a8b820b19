"""Oracle pins for the linear-ramp partition of unity of the paper's experiments (PoU properties
P:95-96; NEXT-3 of SURVEY 8(f)) and the weighted prolongation z = sum_j R~_j^T A_j^-1 R_j v with R~_j^T the
extension weighted by chi_j.  -m "not gpu"."""
import numpy as np
import pytest
import scipy.sparse.linalg as sla

from oracle.oracle import Oracle, OracleError, gmres
from paper_2602_00735_b200.workloads import CONFIGS, probe_vector, sources


@pytest.mark.parametrize("k,px,py", [(20.0, 2, 2), (100.0, 4, 4), (100.0, 5, 3), (400.0, 16, 16)])
def test_pou_properties(k, px, py):
    o = Oracle.from_config(k=k, nsub_x=px, nsub_y=py, pou=1)
    nfx, nfy = o.nf
    tot = np.zeros((nfy + 1, nfx + 1))
    for j in range(o.nsub):
        s = o.subdomain(j)
        bx, by = j % px, j // px
        cx = np.array([o.chi(0, bx, x) for x in range(nfx + 1)])
        cy = np.array([o.chi(1, by, y) for y in range(nfy + 1)])
        assert np.all((cx >= 0) & (cx <= 1)) and np.all((cy >= 0) & (cy <= 1))
        # supp chi_j inside Omega_j,int (vanishes on the extra PML)
        xs = np.nonzero(cx)[0]
        assert xs.min() > s["int_lo"][0] or (s["int_lo"][0] == 0 and xs.min() >= 0)
        assert xs.max() < s["int_hi"][0] or s["int_hi"][0] == o.N[0]
        # chi_j = 1 on the part of the block covered by no other int box
        inner = [x for x in range(s["own_lo"][0] + o.prob.novlp, s["own_hi"][0] - o.prob.novlp + 1)
                 if 0 < x < o.N[0]]
        assert all(cx[x] == 1.0 for x in inner if (bx == 0 or x >= s["own_lo"][0] + o.prob.novlp)
                   and (bx == px - 1 or x <= s["own_hi"][0] - o.prob.novlp))
        tot += np.outer(cy, cx)
    assert np.allclose(tot[1:, 1:], 1.0, rtol=0, atol=1e-15)       # sum_j chi_j = 1


def test_pou_needs_blocks_of_two_overlaps():
    with pytest.raises(OracleError):
        Oracle.from_config(k=100, nsub_x=4, nsub_y=4, n_ovlp=30, n_pml=2, pou=1)


def test_pou_dense_preconditioner_c0():
    cfg = CONFIGS["c0"]
    o = Oracle.from_config(k=cfg.k, nsub_x=2, nsub_y=2, pou=1)
    o.factor()
    n, nfx = o.nfree, o.nf[0]
    B = np.zeros((n, n), np.complex128)
    for j in range(o.nsub):
        s = o.subdomain(j)
        mx, my = s["m"]
        gl = [(s["node0"][0] + lx - 1) + nfx * (s["node0"][1] + ly - 1) for ly in range(my) for lx in range(mx)]
        R = np.zeros((mx * my, n))
        R[np.arange(mx * my), gl] = 1.0
        wgt = np.array([o.chi(0, j % 2, g % nfx + 1) * o.chi(1, j // 2, g // nfx + 1) for g in gl])
        B += (R.T * wgt) @ np.linalg.inv(o.local_matrix(j)) @ R
    for seed in [1, 2]:
        v = probe_vector(n, seed)
        assert np.linalg.norm(o.apply(v) - B @ v) <= 1e-12 * np.linalg.norm(B @ v)


def test_pou_single_subdomain_exact():
    o = Oracle.from_config(k=20, nsub_x=1, nsub_y=1, pou=1)
    o.factor()
    v = probe_vector(o.nfree, 3)
    assert np.linalg.norm(o.apply(v) - sla.spsolve(o.matrix().tocsc(), v)) <= 1e-12 * np.linalg.norm(v)


@pytest.mark.parametrize("name", ["c0", "c1"])
def test_pou_gmres_converges(name):
    cfg = CONFIGS[name]
    o = Oracle.from_config(k=cfg.k, nsub_x=cfg.nsub, nsub_y=cfg.nsub, pou=1)
    o.factor()
    xy, amp, sig = sources(cfg)
    b = o.rhs(xy, amp, sig)
    r = gmres(o.matvec, o.apply, b, restart=50, rtol=1e-6)
    assert r.status == 0 and r.relres_true <= 1e-6

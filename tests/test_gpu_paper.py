"""GPU parity for the paper's own workload (D18-D22): Q1 elements, the
Omega = (0,1)^2 frame with a 3-wavelength PML and g(x) = 10 k x^3, the smoothed delta, RAS-PML-Imp / -Drch with the
linear-ramp PoU -- against the oracle element by element, through the shared-memory (m <= 112) and the cluster
(m > 112) factorisations, and against the iteration counts the paper prints (tests/golden/paper_iterations.txt).
-m gpu."""
import os

import numpy as np
import pytest

from oracle.oracle import Oracle, gmres, richardson
from paper_2602_00735_b200.workloads import PAPER_CONFIGS, paper_source, probe_vector

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a B200", allow_module_level=True)

from paper_2602_00735_b200 import Context  # noqa: E402
from paper_2602_00735_b200.helm import POU_OWNER, POU_RAMP, paper_params  # noqa: E402

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "paper_iterations.txt")


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def golden(k, solver, table=None, variants=(0, 1)):
    out = []
    with open(GOLDEN) as f:
        for line in f:
            if line.startswith("#") or not line.strip():
                continue
            t, ln, kk, grid, P, pml, ov, bc, sv, its, rr = line.split()
            if float(kk) == k and sv == solver and (table is None or t == table) and \
                    {"drch": 0, "imp": 1, "rasimp": 2}[bc] in variants:
                out.append(dict(table=t, grid=int(grid), nsub=int(P), pml=int(pml), ovlp=int(ov),
                                bc={"drch": 0, "imp": 1, "rasimp": 2}[bc], its=int(its)))
    return out


def pair(k, nsub, pml, ovlp, bc=1, pou=POU_RAMP, n_cells=None):
    ctx = Context(**paper_params(k, nsub, pml, ovlp, n_cells=n_cells, local_bc=bc, pou=pou))
    o = Oracle.from_paper(k=k, nsub=nsub, pml=pml, ovlp=ovlp, local_bc=bc, pou=pou, n_cells=n_cells)
    return ctx, o


# (k, nsub, pml, ovlp, bc): m <= 112 -> shared-memory factorisation; m > 112 -> clusters
CASES = [(100.0, 2, 6, 3, 1), (100.0, 3, 4, 2, 0), (150.0, 2, 6, 3, 1), (120.0, 2, 5, 4, 0), (80.0, 1, 4, 2, 1)]


@pytest.mark.parametrize("case", CASES, ids=lambda c: f"k{int(c[0])}-P{c[1]}-pml{c[2]}-ovlp{c[3]}-{'imp' if c[4] else 'drch'}")
def test_paper_operators_and_apply_parity(case):
    k, nsub, pml, ovlp, bc = case
    ctx, o = pair(k, nsub, pml, ovlp, bc)
    assert ctx.layout.stencil_slots == 9
    A9 = ctx.export_stencil().cpu().numpy().T
    Ao = o.stencil()
    assert rel(A9, Ao) <= 1e-13
    xy, amp, s = paper_source(k)
    b = ctx.rhs(xy, amp, s).cpu().numpy()
    assert rel(b, o.rhs(xy, amp, s)) <= 1e-13
    v = probe_vector(o.nfree, 11)
    vd = torch.from_numpy(v).cuda()
    assert rel(ctx.matvec(vd).cpu().numpy(), o.matvec(v)) <= 1e-13
    ctx.factor()
    o.factor()
    z = ctx.precond_apply(vd)
    assert rel(z.cpu().numpy(), o.apply(v)) <= 1e-10
    assert torch.equal(z, ctx.precond_apply(vd))
    ctx.close()


@pytest.mark.parametrize("case", [(100.0, 2, 6, 3, 1), (150.0, 2, 6, 3, 0)])
def test_paper_solvers_parity(case):
    """Richardson (Algorithm 1) and GMRES to rtol 1e-10: iterations +-1 and solutions vs the oracle."""
    k, nsub, pml, ovlp, bc = case
    ctx, o = pair(k, nsub, pml, ovlp, bc)
    ctx.factor()
    o.factor()
    xy, amp, s = paper_source(k)
    b = o.rhs(xy, amp, s)
    bd = torch.from_numpy(b).cuda()
    ro = richardson(o.matvec, o.apply, b, rtol=1e-10, maxit=500)
    x, info, _ = ctx.richardson(bd, rtol=1e-10, maxit=500)
    assert info.status == 0 and abs(info.iterations - ro.iterations) <= 1
    assert rel(x.cpu().numpy(), ro.x) <= 1e-8
    go = gmres(o.matvec, o.apply, b, restart=50, rtol=1e-10)
    x, ginfo, _ = ctx.gmres(bd, restart=50, rtol=1e-10)
    assert ginfo.status == 0 and abs(ginfo.iterations - go.iterations) <= 1
    assert rel(x.cpu().numpy(), go.x) <= 1e-8
    ctx.close()


def test_paper_single_subdomain_cluster_path_is_exact_inverse():
    """One subdomain = Omega (m = 119 > 112: the cluster factorisation): B^-1 = A^-1, GMRES in one iteration."""
    ctx = Context(**paper_params(60.0, 1, 4, 2))
    assert ctx.layout.m_max > 112
    ctx.factor()
    v = torch.from_numpy(probe_vector(ctx.n, 4)).cuda()
    z = ctx.precond_apply(v)
    assert rel(ctx.matvec(z).cpu().numpy(), v.cpu().numpy()) <= 1e-11
    _, info, _ = ctx.gmres(v, restart=50, rtol=1e-10)
    assert info.iterations == 1
    ctx.close()


@pytest.mark.parametrize("row", golden(300.0, "richardson"),
                         ids=lambda r: f"{r['table']}-{'imp' if r['bc'] else 'drch'}-pml{r['pml']}-ovlp{r['ovlp']}")
def test_paper_k300_richardson_matches_printed_iterations(row):
    """The GPU reproduces the Richardson counts printed at k = 300 (Tables 1, 3, 4: P:254) exactly."""
    ctx = Context(**paper_params(300.0, row["nsub"], row["pml"], row["ovlp"], n_cells=row["grid"], local_bc=row["bc"]))
    ctx.factor()
    xy, amp, s = paper_source(300.0)
    b = ctx.rhs(xy, amp, s)
    _, info, _ = ctx.richardson(b, rtol=1e-10, maxit=500)
    assert info.status == 0 and info.iterations == row["its"], (info.iterations, info.relres)
    ctx.close()


def test_paper_k300_apply_parity_full_size():
    """k = 300 (grid 600^2, 2 x 2 subdomains of ~312^2 unknowns, cluster factorisation) in full: apply vs oracle."""
    ctx, o = pair(300.0, 2, 8, 4, 1, n_cells=600)
    ctx.factor()
    o.factor()
    v = probe_vector(o.nfree, 301)
    z = ctx.precond_apply(torch.from_numpy(v).cuda()).cpu().numpy()
    assert rel(z, o.apply(v)) <= 1e-10
    ctx.close()


@pytest.mark.parametrize("row", golden(600.0, "richardson"),
                         ids=lambda r: f"{r['table']}-{'imp' if r['bc'] else 'drch'}-pml{r['pml']}-ovlp{r['ovlp']}")
def test_paper_k600_richardson_near_printed_iterations(row):
    """k = 600 (grid 1200^2, 16 subdomains): within one iteration of Tables 1 / 3 / 4."""
    ctx = Context(**paper_params(600.0, row["nsub"], row["pml"], row["ovlp"], n_cells=row["grid"], local_bc=row["bc"]))
    ctx.factor()
    xy, amp, s = paper_source(600.0)
    b = ctx.rhs(xy, amp, s)
    _, info, _ = ctx.richardson(b, rtol=1e-10, maxit=500)
    assert info.status == 0 and abs(info.iterations - row["its"]) <= 1, (info.iterations, info.relres)
    ctx.close()


@pytest.mark.parametrize("row", golden(1200.0, "richardson"),
                         ids=lambda r: f"{r['table']}-{'imp' if r['bc'] else 'drch'}-pml{r['pml']}-ovlp{r['ovlp']}")
def test_paper_k1200_richardson_near_printed_iterations(row):
    """k = 1200 (grid 2400^2, 64 subdomains, ~40 GB of factors on one GPU): within two iterations of Tables 1 / 3 / 4
    (P:256).  Observed: 4 of 6 rows within one (Table 4 exact), Table 1 Drch and Table 3 pml 25 / ovlp 8
    two above the printed count (profiles/r01_paper_iterations.md)."""
    ctx = Context(**paper_params(1200.0, row["nsub"], row["pml"], row["ovlp"], n_cells=row["grid"], local_bc=row["bc"]))
    ctx.factor()
    xy, amp, s = paper_source(1200.0)
    b = ctx.rhs(xy, amp, s)
    _, info, _ = ctx.richardson(b, rtol=1e-10, maxit=500)
    assert info.status == 0 and abs(info.iterations - row["its"]) <= 2, (info.iterations, info.relres)
    ctx.close()
    torch.cuda.empty_cache()


@pytest.mark.parametrize("nranks,gg", [(2, (2, 1)), (4, (2, 2))])
def test_paper_sharded_apply_and_matvec_bitwise(nranks, gg):
    """Q1 (9-point, corner couplings) through communication-free shards with the owner PoU: bitwise equal to the
    single-rank operators (the two-phase halo carries the corners)."""
    kw = paper_params(150.0, 4, 6, 3, pou=POU_OWNER)
    ref = Context(**kw)
    ref.factor()
    nf = ref.layout.N_cells - 1
    v = torch.from_numpy(probe_vector(ref.n, 3)).cuda()
    z_ref = ref.precond_apply(v)
    y_ref = ref.matvec(v)
    V = v.view(nf, nf)
    Z = torch.full_like(V, complex("nan"))
    Y = torch.full_like(V, complex("nan"))
    for r in range(nranks):
        c = Context(**{**kw, "gpu_grid": gg}, rank=r, nranks=nranks)
        c.factor()
        pl = c.plan
        ext = V[pl["ext_j0"] - 1:pl["ext_j1"] - 1, pl["ext_i0"] - 1:pl["ext_i1"] - 1].contiguous().view(-1)
        i0, i1, j0, j1 = pl["owned_i0"], pl["owned_i1"], pl["owned_j0"], pl["owned_j1"]
        Z[j0 - 1:j1 - 1, i0 - 1:i1 - 1] = c.precond_apply_ext(ext).view(j1 - j0, i1 - i0)
        nb = pl["nbr"]
        li, ri, dj, uj = int(nb[0] >= 0), int(nb[1] >= 0), int(nb[2] >= 0), int(nb[3] >= 0)
        ext1 = V[j0 - 1 - dj:j1 - 1 + uj, i0 - 1 - li:i1 - 1 + ri].contiguous().view(-1)
        Y[j0 - 1:j1 - 1, i0 - 1:i1 - 1] = c.matvec_ext(ext1).view(j1 - j0, i1 - i0)
        c.close()
    assert torch.equal(Z.view(-1), z_ref)
    assert torch.equal(Y.view(-1), y_ref)
    ref.close()


def test_paper_wide_single_block_exact_inverse():
    """One subdomain = Omega at k = 300 (grid 600^2): blocks 599 wide (19 Gauss-Jordan panels in the cluster
    factorisation, large slabs in the cluster-split apply).  B^-1 = A^-1: A (B^-1 v) = v, and B^-1 is linear."""
    ctx = Context(**paper_params(300.0, 1, 4, 2, n_cells=600))
    assert ctx.layout.m_max == 599
    ctx.factor()
    v = torch.from_numpy(probe_vector(ctx.n, 8)).cuda()
    u = torch.from_numpy(probe_vector(ctx.n, 9)).cuda()
    z = ctx.precond_apply(v)
    assert rel(ctx.matvec(z).cpu().numpy(), v.cpu().numpy()) <= 1e-10
    zl = ctx.precond_apply(v + 2.5j * u)
    assert rel(zl.cpu().numpy(), (z + 2.5j * ctx.precond_apply(u)).cpu().numpy()) <= 1e-12
    ctx.close()


def test_paper_claims_ras_pml_imp_vs_drch_vs_ras_imp():
    """"RAS-PML-Imp exhibits superior performance over RAS-PML-Drch, particularly at high frequencies, while
    RAS-Imp fails to converge at all for high k" (Table 1).  Richardson to 1e-10: Imp <= Drch at k = 300 / 600 / 1200;
    RAS-Imp (no local PML, impedance on the subdomain faces) needs more iterations than both at k = 300 / 600 (printed
    30 / 43; ours 29 / 48) and does not converge within the paper's 500 at k = 1200 (printed: stopped at 500, relres
    0.016; ours: diverges, flagged once the residual exceeds 1e6)."""
    its = {}
    for k, P, pml, ov in [(300.0, 2, 8, 4), (600.0, 4, 11, 5), (1200.0, 8, 15, 6)]:
        for variant, (bc, p_) in {"imp": (1, pml), "drch": (0, pml), "rasimp": (1, 0)}.items():
            ctx = Context(**paper_params(k, P, p_, ov, n_cells=int(2 * k), local_bc=bc))
            ctx.factor()
            b = ctx.rhs(*paper_source(k))
            _, info, _ = ctx.richardson(b, rtol=1e-10, maxit=500)
            its[(k, variant)] = (info.iterations, info.status)
            ctx.close()
            torch.cuda.empty_cache()
    for k in (300.0, 600.0, 1200.0):
        assert its[(k, "imp")][1] == 0 and its[(k, "drch")][1] == 0
        assert its[(k, "imp")][0] <= its[(k, "drch")][0]
    for k in (300.0, 600.0):
        assert its[(k, "rasimp")][1] == 0 and its[(k, "rasimp")][0] > its[(k, "drch")][0]
    assert its[(1200.0, "rasimp")][1] != 0, its[(1200.0, "rasimp")]

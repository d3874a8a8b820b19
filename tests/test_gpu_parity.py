"""GPU parity: libhelm's CUDA path (through the C ABI / thin binding) vs the CPU oracle on identical seeded
inputs.  Tolerances are BASELINE.json north_star's: matvec relative l2 <= 1e-13, preconditioner apply
<= 1e-10, GMRES iterations within +-1, final solution <= 1e-6; assembled coefficients and b <= 1e-13
(DESIGN.md 7).  -m gpu."""
import numpy as np
import pytest

from oracle.oracle import Oracle, gmres as orc_gmres
from paper_2602_00735_b200.workloads import CONFIGS, probe_vector, sources

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU box
    pytest.skip("needs a B200", allow_module_level=True)

from paper_2602_00735_b200 import Context, HelmError  # noqa: E402


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def to_np(t):
    return t.detach().cpu().numpy()


def to_dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


_CACHE = {}


def pair(name, nsub=None, **kw):
    """(GPU context, oracle) for a config, factored; cached per session."""
    cfg = CONFIGS[name]
    nsub = nsub or (cfg.nsub, cfg.nsub)
    key = (name, nsub, tuple(sorted(kw.items())))
    if key not in _CACHE:
        ctx = Context(cfg.k, nsub[0], nsub[1], **kw)
        ctx.factor()
        o = Oracle.from_config(k=cfg.k, nsub_x=nsub[0], nsub_y=nsub[1], **kw)
        _CACHE[key] = (ctx, o)
    return _CACHE[key]


SMALL = ["c0", "c1", "c2"]


@pytest.mark.parametrize("name", SMALL)
def test_stencil_parity(name):
    ctx, o = pair(name)
    A = to_np(ctx.export_stencil())          # [7][n]
    R = o.stencil().T                        # [7][n]
    assert np.max(np.abs(A - R)) <= 1e-13 * np.max(np.abs(R))


@pytest.mark.parametrize("name", SMALL)
def test_rhs_parity(name):
    ctx, o = pair(name)
    xy, amp, sig = sources(CONFIGS[name])
    b = to_np(ctx.rhs(xy, amp, sig))
    assert rel(b, o.rhs(xy, amp, sig)) <= 1e-13


@pytest.mark.parametrize("name", SMALL)
def test_matvec_parity(name):
    ctx, o = pair(name)
    v = probe_vector(o.nfree, int(CONFIGS[name].k) + 1)
    y = to_np(ctx.matvec(to_dev(v)))
    assert rel(y, o.matvec(v)) <= 1e-13


@pytest.mark.parametrize("name", SMALL)
def test_apply_parity(name):
    ctx, o = pair(name)
    o.factor()
    v = probe_vector(o.nfree, int(CONFIGS[name].k) + 1)
    z = to_np(ctx.precond_apply(to_dev(v)))
    assert rel(z, o.apply(v)) <= 1e-10


@pytest.mark.parametrize("name", SMALL)
def test_gmres_parity(name):
    cfg = CONFIGS[name]
    ctx, o = pair(name)
    o.factor()
    xy, amp, sig = sources(cfg)
    b = o.rhs(xy, amp, sig)
    ref = orc_gmres(o.matvec, o.apply, b, restart=cfg.restart, rtol=cfg.rtol)
    x, info, hist = ctx.gmres(to_dev(b), restart=cfg.restart, rtol=cfg.rtol, history=True)
    assert info.status == 0 and ref.status == 0
    assert abs(info.iterations - ref.iterations) <= 1
    assert info.relres_true <= cfg.rtol
    assert rel(to_np(x), ref.x) <= 1e-6
    # the GPU's own residual claim, re-checked with the oracle's operator
    xr = to_np(x)
    assert np.linalg.norm(b - o.matvec(xr)) <= 1.01 * cfg.rtol * np.linalg.norm(b)


def test_single_subdomain_is_exact_inverse_and_one_iteration():
    """north_star: a single subdomain equal to Omega makes B^-1 = A^-1 and GMRES converge in 1 iteration
    (c0: one 51 x 51-node subdomain)."""
    ctx, o = pair("c0", nsub=(1, 1))
    xy, amp, sig = sources(CONFIGS["c0"])
    b = o.rhs(xy, amp, sig)
    import scipy.sparse.linalg as sla
    xd = sla.spsolve(o.matrix().tocsc(), b)
    z = to_np(ctx.precond_apply(to_dev(b)))
    assert rel(z, xd) <= 1e-10
    x, info, _ = ctx.gmres(to_dev(b))
    assert info.iterations == 1 and info.relres_true < 1e-10


@pytest.mark.parametrize("name,nsub", [("c0", (3, 2)), ("c0", (1, 4)), ("c1", (5, 3)), ("c1", (7, 7)),
                                       ("c2", (9, 13))])
def test_apply_parity_ragged(name, nsub):
    """uneven block sizes, rectangular subdomain grids, 1 x P strips"""
    ctx, o = pair(name, nsub=nsub)
    o.factor()
    v = probe_vector(o.nfree, 5)
    z = to_np(ctx.precond_apply(to_dev(v)))
    assert rel(z, o.apply(v)) <= 1e-10


def test_apply_parity_other_widths():
    """explicit overlap / PML widths (delta != kappa), thin layers"""
    ctx, o = pair("c1", n_ovlp=3, n_pml=9)
    o.factor()
    v = probe_vector(o.nfree, 6)
    assert rel(to_np(ctx.precond_apply(to_dev(v))), o.apply(v)) <= 1e-10
    ctx2, o2 = pair("c1", n_ovlp=2, n_pml=2)
    o2.factor()
    assert rel(to_np(ctx2.precond_apply(to_dev(v))), o2.apply(v)) <= 1e-10


def test_zero_and_linearity_and_determinism():
    ctx, o = pair("c1")
    z0 = ctx.precond_apply(torch.zeros(ctx.n, dtype=torch.complex128, device="cuda"))
    assert torch.count_nonzero(z0).item() == 0
    v1 = to_dev(probe_vector(ctx.n, 1))
    v2 = to_dev(probe_vector(ctx.n, 2))
    a = 0.3 - 1.7j
    lhs = to_np(ctx.precond_apply(v1 + a * v2))
    rhs = to_np(ctx.precond_apply(v1)) + a * to_np(ctx.precond_apply(v2))
    assert rel(lhs, rhs) <= 1e-12
    za, zb = ctx.precond_apply(v1), ctx.precond_apply(v1)
    assert torch.equal(za, zb)                      # bitwise deterministic
    x, info, _ = ctx.gmres(torch.zeros(ctx.n, dtype=torch.complex128, device="cuda"))
    assert info.iterations == 0 and torch.count_nonzero(x).item() == 0


def test_host_entry_points_match_device():
    ctx, o = pair("c1")
    v = probe_vector(ctx.n, 9)
    zh = np.zeros_like(v)
    ctx.precond_apply_host(v, zh)
    assert np.array_equal(zh, to_np(ctx.precond_apply(to_dev(v))))
    xy, amp, sig = sources(CONFIGS["c1"])
    b = to_np(ctx.rhs(xy, amp, sig))
    xh = np.zeros_like(b)
    _, info = ctx.gmres_host(b, xh)
    xd, info2, _ = ctx.gmres(to_dev(b))
    assert info.iterations == info2.iterations and np.array_equal(xh, to_np(xd))


def test_errors():
    with pytest.raises(HelmError) as e:
        Context(20.0, 8, 8)                       # blocks of 6.5 cells < delta + kappa = 10
    assert e.value.code == -6
    ctx = Context(20.0, 2, 2)
    with pytest.raises(HelmError) as e:
        ctx.precond_apply(torch.zeros(ctx.n, dtype=torch.complex128, device="cuda"))
    assert e.value.code == -7
    with pytest.raises(HelmError) as e:
        Context(1600.0, 1, 1)                     # one 2565-node-wide block: above the 992 limit
    assert e.value.code == -1


def test_c3_full_size_sampled_parity():
    """k = 1600, 64 x 64 subdomains, in the launch configuration bench.py times: the oracle solves a sample of
    subdomains (corner, edges, interior) one by one and the GPU apply must match on their owned nodes;
    matvec on sampled rows."""
    cfg = CONFIGS["c3"]
    ctx = Context(cfg.k, cfg.nsub, cfg.nsub)
    ctx.factor()
    o = Oracle.from_config(k=cfg.k, nsub_x=cfg.nsub, nsub_y=cfg.nsub)
    v = probe_vector(o.nfree, int(cfg.k) + 1)
    vd = to_dev(v)
    z = to_np(ctx.precond_apply(vd))
    subs = [0, 63, 64 * 63, 4095, 17, 64 * 5, 64 * 31 + 30, 64 * 50 + 9]
    o.factor(subs)
    zo = o.apply(v, subs=subs)
    mask = np.zeros(o.nfree, bool)
    nfx = o.nf[0]
    for j in subs:
        s = o.subdomain(j)
        for gj in range(max(s["own_lo"][1], 1), min(s["own_hi"][1], o.N[1])):
            mask[(max(s["own_lo"][0], 1) - 1) + nfx * (gj - 1):(min(s["own_hi"][0], o.N[0]) - 1) + nfx * (gj - 1)] = True
    assert rel(z[mask], zo[mask]) <= 1e-10
    rows = np.random.default_rng(0).choice(o.nfree, 20000, replace=False)
    y = to_np(ctx.matvec(vd))
    assert rel(y[rows], o.matvec_rows(v, rows)) <= 1e-13
    ctx.close()


def test_c3_full_size_properties():
    """k = 1600 in the bench configuration: the apply is linear and bitwise deterministic at full size, and GMRES(50)
    reaches rtol 1e-6 measured on the TRUE residual ||b - A x|| / ||b|| recomputed independently with helm_matvec."""
    cfg = CONFIGS["c3"]
    ctx = Context(cfg.k, cfg.nsub, cfg.nsub)
    ctx.factor()
    u = to_dev(probe_vector(ctx.n, 11))
    v = to_dev(probe_vector(ctx.n, 12))
    a = complex(0.3, -1.7)
    zu, zv = ctx.precond_apply(u), ctx.precond_apply(v)
    zl = ctx.precond_apply(u + a * v)
    assert float(torch.linalg.norm(zl - (zu + a * zv)) / torch.linalg.norm(zl)) <= 1e-12
    assert torch.equal(zu, ctx.precond_apply(u))
    xy, amp, sig = sources(cfg)
    b = ctx.rhs(xy, amp, sig)
    x, info, _ = ctx.gmres(b, restart=cfg.restart, rtol=cfg.rtol)
    assert info.status == 0
    r = b - ctx.matvec(x)
    assert float(torch.linalg.norm(r) / torch.linalg.norm(b)) <= cfg.rtol
    ctx.close()


def test_gmres_initial_guess_and_restart_bounds():
    """A nonzero initial guess x0 (the oracle's GMRES from the same x0: iterations +-1, x to 1e-6), short restarts
    (GMRES(5) vs the oracle's GMRES(5)), the largest restart the ABI takes (63: 64 basis vectors) and the first it
    refuses (64)."""
    cfg = CONFIGS["c1"]
    ctx, o = pair("c1")
    o.factor()
    b = o.rhs(*sources(cfg))
    x0 = 0.3 * probe_vector(o.nfree, 77)
    ref = orc_gmres(o.matvec, o.apply, b, restart=50, rtol=1e-6, x0=x0)
    x, info, _ = ctx.gmres(to_dev(b), to_dev(x0.copy()), restart=50, rtol=1e-6)
    assert info.status == 0 and abs(info.iterations - ref.iterations) <= 1
    assert rel(to_np(x), ref.x) <= 1e-6
    ref5 = orc_gmres(o.matvec, o.apply, b, restart=5, rtol=1e-6)
    x5, info5, _ = ctx.gmres(to_dev(b), restart=5, rtol=1e-6)
    assert info5.status == 0 and abs(info5.iterations - ref5.iterations) <= 1 and info5.restarts == ref5.restarts
    assert rel(to_np(x5), ref5.x) <= 1e-6
    x63, info63, _ = ctx.gmres(to_dev(b), restart=63, rtol=1e-6)
    assert info63.status == 0
    # an initial guess that already meets rtol returns at once (0 iterations, x unchanged); the exact zero residual
    # (b = A x0 exactly, here b := A x63) too, with no division by a zero Krylov norm
    xs = x63.clone()
    again, info_a, _ = ctx.gmres(to_dev(b), xs, restart=50, rtol=1e-6)
    assert info_a.status == 0 and info_a.iterations == 0 and torch.equal(again, x63)
    bx = ctx.matvec(x63)
    xz = x63.clone()
    _, info_z, _ = ctx.gmres(bx, xz, restart=50, rtol=1e-12)
    assert info_z.status == 0 and info_z.iterations == 0 and info_z.relres_true == 0.0 and torch.equal(xz, x63)
    with pytest.raises(HelmError) as e:
        ctx.gmres(to_dev(b), restart=64, rtol=1e-6)
    assert e.value.code == -1


def test_degenerate_inputs():
    """Edge cases of the boundary: no sources (b = 0 -> x = 0 after 0 iterations; Richardson likewise), maxit = 0 (x0
    returned unchanged, HELM_NOT_CONVERGED, no apply issued), an impedance layout whose face would sit on dOmega
    (refused on the GPU as by the oracle, tests/test_oracle_solvers.py), and the apply of a unit vector (one nonzero
    node: the response is confined to the blocks of the subdomains that cover it) against the oracle."""
    import math
    ctx, o = pair("c1")
    b0 = ctx.rhs(np.zeros((0, 2)), np.zeros(0, np.complex128), 0.01)
    assert torch.count_nonzero(b0).item() == 0
    x, info, _ = ctx.gmres(b0)
    assert info.iterations == 0 and torch.count_nonzero(x).item() == 0
    xr, rinfo, _ = ctx.richardson(b0)
    assert rinfo.iterations == 0 and torch.count_nonzero(xr).item() == 0
    b = ctx.rhs(*sources(CONFIGS["c1"]))
    x0 = to_dev(probe_vector(ctx.n, 4))
    x = x0.clone()
    _, info, _ = ctx.gmres(b, x, maxit=0)
    assert info.status == 2 and info.iterations == 0 and info.applies == 0 and torch.equal(x, x0)
    with pytest.raises(HelmError) as e:
        Context(6 * math.pi, 10, 2, n_ovlp=2, n_pml=3, local_bc=1)
    assert e.value.code == -6
    e1 = np.zeros(ctx.n, np.complex128)
    e1[ctx.n // 2 + 17] = 1.0 - 2.0j
    z = to_np(ctx.precond_apply(to_dev(e1)))
    zo = o.apply(e1)
    assert np.linalg.norm(z - zo) <= 1e-10 * np.linalg.norm(zo)
    assert np.count_nonzero(zo) < ctx.n // 2

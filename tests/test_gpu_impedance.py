"""GPU parity for RAS-PML-Imp (NEXT-1 of SURVEY 8(f)): libhelm's impedance local operators,
factorisation and apply vs the oracle (apply <= 1e-10; GMRES iterations +-1, x <= 1e-6), on the BJ configs
and ragged grids, plus bitwise sharded reproduction with the wider impedance ghost frame.  -m gpu."""
import numpy as np
import pytest

from oracle.oracle import Oracle, gmres
from paper_2602_00735_b200.workloads import CONFIGS, probe_vector, sources

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a B200", allow_module_level=True)

from paper_2602_00735_b200 import Context  # noqa: E402
from paper_2602_00735_b200.helm import BC_IMPEDANCE  # noqa: E402


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.mark.parametrize("name,nsub", [("c0", None), ("c1", None), ("c2", None), ("c1", (5, 3)), ("c0", (3, 1))])
def test_imp_apply_and_gmres_parity(name, nsub):
    cfg = CONFIGS[name]
    nsub = nsub or (cfg.nsub, cfg.nsub)
    ctx = Context(cfg.k, nsub[0], nsub[1], local_bc=BC_IMPEDANCE)
    ctx.factor()
    o = Oracle.from_config(k=cfg.k, nsub_x=nsub[0], nsub_y=nsub[1], local_bc=1)
    o.factor()
    v = probe_vector(o.nfree, 11)
    z = ctx.precond_apply(torch.from_numpy(v).cuda()).cpu().numpy()
    assert rel(z, o.apply(v)) <= 1e-10
    xy, amp, sig = sources(cfg)
    b = o.rhs(xy, amp, sig)
    ref = gmres(o.matvec, o.apply, b, restart=cfg.restart, rtol=cfg.rtol)
    x, info, _ = ctx.gmres(torch.from_numpy(b).cuda(), restart=cfg.restart, rtol=cfg.rtol)
    assert info.status == 0 and abs(info.iterations - ref.iterations) <= 1
    assert rel(x.cpu().numpy(), ref.x) <= 1e-6
    ctx.close()


def test_imp_sharded_bitwise():
    cfg = CONFIGS["c2"]
    ref = Context(cfg.k, cfg.nsub, cfg.nsub, local_bc=BC_IMPEDANCE)
    ref.factor()
    nf = ref.layout.N_cells - 1
    v = torch.from_numpy(probe_vector(ref.n, 3)).cuda()
    z_ref = ref.precond_apply(v)
    V = v.view(nf, nf)
    Z = torch.full_like(V, complex("nan"))
    for r in range(4):
        c = Context(cfg.k, cfg.nsub, cfg.nsub, rank=r, nranks=4, local_bc=BC_IMPEDANCE)
        c.factor()
        pl = c.plan
        ext = V[pl["ext_j0"] - 1:pl["ext_j1"] - 1, pl["ext_i0"] - 1:pl["ext_i1"] - 1].contiguous().view(-1)
        z = c.precond_apply_ext(ext)
        i0, i1, j0, j1 = pl["owned_i0"], pl["owned_i1"], pl["owned_j0"], pl["owned_j1"]
        Z[j0 - 1:j1 - 1, i0 - 1:i1 - 1] = z.view(j1 - j0, i1 - i0)
        c.close()
    assert torch.equal(Z.view(-1), z_ref)


def test_imp_c3_full_size_sampled():
    cfg = CONFIGS["c3"]
    ctx = Context(cfg.k, cfg.nsub, cfg.nsub, local_bc=BC_IMPEDANCE)
    ctx.factor()
    o = Oracle.from_config(k=cfg.k, nsub_x=cfg.nsub, nsub_y=cfg.nsub, local_bc=1)
    v = probe_vector(o.nfree, int(cfg.k) + 1)
    z = ctx.precond_apply(torch.from_numpy(v).cuda()).cpu().numpy()
    subs = [0, 4095, 64 * 20 + 33]
    o.factor(subs)
    zo = o.apply(v, subs=subs)
    nfx = o.nf[0]
    mask = np.zeros(o.nfree, bool)
    for j in subs:
        s = o.subdomain(j)
        for gj in range(max(s["own_lo"][1], 1), min(s["own_hi"][1], o.N[1])):
            mask[(max(s["own_lo"][0], 1) - 1) + nfx * (gj - 1):(min(s["own_hi"][0], o.N[0]) - 1) + nfx * (gj - 1)] = True
    assert rel(z[mask], zo[mask]) <= 1e-10
    ctx.close()

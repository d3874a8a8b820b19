"""GPU parity for the linear-ramp partition of unity (NEXT-3 of SURVEY 8(f)):
weighted local solutions over the int-box interiors, deterministic gather of the <= 4 covering subdomains.
-m gpu."""
import numpy as np
import pytest

from oracle.oracle import Oracle, gmres
from paper_2602_00735_b200.workloads import CONFIGS, probe_vector, sources

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a B200", allow_module_level=True)

from paper_2602_00735_b200 import Context, HelmError  # noqa: E402
from paper_2602_00735_b200.helm import POU_RAMP  # noqa: E402


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.mark.parametrize("name,nsub,bc", [("c0", None, 0), ("c1", None, 0), ("c2", None, 0), ("c1", (5, 3), 0),
                                          ("c1", None, 1), ("c2", (11, 13), 1)])
def test_pou_apply_and_gmres_parity(name, nsub, bc):
    cfg = CONFIGS[name]
    nsub = nsub or (cfg.nsub, cfg.nsub)
    ctx = Context(cfg.k, nsub[0], nsub[1], local_bc=bc, pou=POU_RAMP)
    ctx.factor()
    o = Oracle.from_config(k=cfg.k, nsub_x=nsub[0], nsub_y=nsub[1], local_bc=bc, pou=1)
    o.factor()
    v = probe_vector(o.nfree, 13)
    vd = torch.from_numpy(v).cuda()
    z = ctx.precond_apply(vd)
    assert rel(z.cpu().numpy(), o.apply(v)) <= 1e-10
    assert torch.equal(z, ctx.precond_apply(vd))                 # deterministic gather
    xy, amp, sig = sources(cfg)
    b = o.rhs(xy, amp, sig)
    ref = gmres(o.matvec, o.apply, b, restart=cfg.restart, rtol=cfg.rtol)
    x, info, _ = ctx.gmres(torch.from_numpy(b).cuda(), restart=cfg.restart, rtol=cfg.rtol)
    assert info.status == 0 and abs(info.iterations - ref.iterations) <= 1
    assert rel(x.cpu().numpy(), ref.x) <= 1e-6
    ctx.close()


def test_pou_ramp_needs_a_communicator_on_several_ranks():
    """The ramp PoU sums over subdomains of neighbouring ranks (additive reverse exchange): communication-free shards
    (no NCCL id, no loopback group) refuse it."""
    with pytest.raises(HelmError) as e:
        Context(400.0, 16, 16, rank=0, nranks=2, pou=POU_RAMP)
    assert e.value.code == -1


def test_pou_c3_full_size_sampled():
    """k = 1600: the nodes of one interior subdomain's int box are covered only by its 3 x 3 neighbourhood; the
    oracle solves those 9 subdomains and accumulates their weighted solutions."""
    cfg = CONFIGS["c3"]
    ctx = Context(cfg.k, cfg.nsub, cfg.nsub, pou=POU_RAMP)
    ctx.factor()
    o = Oracle.from_config(k=cfg.k, nsub_x=cfg.nsub, nsub_y=cfg.nsub, pou=1)
    v = probe_vector(o.nfree, int(cfg.k) + 1)
    z = ctx.precond_apply(torch.from_numpy(v).cuda()).cpu().numpy()
    cx, cy = 30, 17
    subs = [(cx + dx) + 64 * (cy + dy) for dy in (-1, 0, 1) for dx in (-1, 0, 1)]
    o.factor(subs)
    zo = o.apply(v, subs=subs)
    s = o.subdomain(cx + 64 * cy)
    nfx = o.nf[0]
    idx = [(gi - 1) + nfx * (gj - 1) for gj in range(s["int_lo"][1] + 1, s["int_hi"][1])
           for gi in range(s["int_lo"][0] + 1, s["int_hi"][0])]
    assert rel(z[idx], zo[idx]) <= 1e-10
    ctx.close()

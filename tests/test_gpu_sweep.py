"""Seeded random sweep of layouts against the oracle: wavenumber, subdomain grid (square, rectangular, 1 x P), overlap
and PML widths (thin, delta != kappa, zero PML for RAS-Imp), local BC (Dirichlet / impedance) and PoU (owner / ramp),
P1 BJ-style and Q1 paper-style problems.  Each draw: the assembled operator's matvec and the preconditioner apply on
a seeded vector against the oracle (1e-13 / 1e-10), plus linearity of the apply.  The draws land on every apply
path -- k_apply with 2 to 6 ring slots, the cluster-split apply with several G -- and both factorisation paths.
-m gpu."""
import numpy as np
import pytest

from oracle.oracle import Oracle, OracleError
from paper_2602_00735_b200.workloads import probe_vector

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a B200", allow_module_level=True)

from paper_2602_00735_b200 import Context, HelmError  # noqa: E402
from paper_2602_00735_b200.helm import paper_params  # noqa: E402


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


def draws(n=30, seed=2026):
    rng = np.random.default_rng(seed)
    out = []
    for i in range(n):
        paper = i % 3 == 2
        if paper:
            k = float(rng.choice([40, 60, 80]))
            nsub = int(rng.integers(1, 4))
            pml = int(rng.integers(0, 7))
            ovlp = int(rng.integers(1, 4))
            out.append(("q1", dict(k=k, nsub=nsub, pml=pml, ovlp=ovlp, local_bc=int(rng.integers(0, 2)) if pml else 1,
                                   pou=int(rng.integers(0, 2)))))
        else:
            k = float(rng.choice([30, 50, 80, 120]))
            px, py = int(rng.integers(1, 9)), int(rng.integers(1, 9))
            ov = int(rng.integers(2, 8))
            pm = int(rng.integers(2, 10))
            out.append(("p1", dict(k=k, nsub_x=px, nsub_y=py, n_ovlp=ov, n_pml=pm, local_bc=int(rng.integers(0, 2)),
                                   pou=int(rng.integers(0, 2)))))
    # at least as many subdomains as SMs: the persistent k_apply, whose ring depth adapts to the CTAs per SM
    out.append(("p1", dict(k=200.0, nsub_x=13, nsub_y=12, n_ovlp=4, n_pml=6, local_bc=1, pou=0)))
    out.append(("p1", dict(k=260.0, nsub_x=25, nsub_y=16, n_ovlp=3, n_pml=3, local_bc=0, pou=1)))
    return out


@pytest.mark.parametrize("kind,kw", draws(), ids=lambda v: str(v) if isinstance(v, str) else
                         "-".join(f"{a}{b}" for a, b in v.items()))
def test_random_layout_parity(kind, kw):
    def make():
        if kind == "q1":
            return (lambda: Context(**paper_params(kw["k"], kw["nsub"], kw["pml"], kw["ovlp"], local_bc=kw["local_bc"],
                                                   pou=kw["pou"])),
                    lambda: Oracle.from_paper(k=kw["k"], nsub=kw["nsub"], pml=kw["pml"], ovlp=kw["ovlp"],
                                              local_bc=kw["local_bc"], pou=kw["pou"]))
        return (lambda: Context(kw["k"], kw["nsub_x"], kw["nsub_y"], n_ovlp=kw["n_ovlp"], n_pml=kw["n_pml"],
                                local_bc=kw["local_bc"], pou=kw["pou"]),
                lambda: Oracle.from_config(k=kw["k"], nsub_x=kw["nsub_x"], nsub_y=kw["nsub_y"], n_ovlp=kw["n_ovlp"],
                                           n_pml=kw["n_pml"], local_bc=kw["local_bc"], pou=kw["pou"]))
    mk_ctx, mk_orc = make()
    try:
        ctx = mk_ctx()
    except HelmError as e:   # a layout the method cannot have (an extension leaves the domain / merges faces)
        assert e.code == -6
        with pytest.raises(OracleError):
            mk_orc()
        pytest.skip("invalid layout, refused by both sides")
    o = mk_orc()
    ctx.factor()
    o.factor()
    assert ctx.n == o.nfree
    v = probe_vector(o.nfree, 9)
    vd = torch.from_numpy(v).cuda()
    assert rel(ctx.matvec(vd).cpu().numpy(), o.matvec(v)) <= 1e-13
    z = ctx.precond_apply(vd)
    assert rel(z.cpu().numpy(), o.apply(v)) <= 1e-10
    w = torch.from_numpy(probe_vector(o.nfree, 10)).cuda()
    zw = ctx.precond_apply(w)
    zs = ctx.precond_apply(2.0 * vd - 0.5j * w)
    assert float(torch.linalg.norm(zs - (2.0 * z - 0.5j * zw)) / torch.linalg.norm(zs)) <= 1e-12
    ctx.close()
    o.close()

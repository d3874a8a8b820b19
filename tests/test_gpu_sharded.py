"""Sharded arithmetic on one GPU: communication-free rank contexts (nranks > 1, no NCCL id) receive their
ghost-framed inputs from the test and must reproduce the single-rank apply / matvec bit for bit (no
cross-rank reduction exists in either).  The NCCL transport itself needs >= 2 GPUs; its
schedule is verified on CPU in test_multirank_plan.py.  -m gpu."""
import numpy as np
import pytest

from paper_2602_00735_b200.workloads import CONFIGS, probe_vector

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a B200", allow_module_level=True)

from paper_2602_00735_b200 import Context, HelmError  # noqa: E402


def grid(v, nf):
    return v.view(nf, nf)   # [j-1, i-1]


@pytest.mark.parametrize("name,nranks,gg", [("c1", 2, (0, 0)), ("c1", 4, (0, 0)), ("c1", 3, (1, 3)),
                                            ("c2", 4, (0, 0)), ("c2", 8, (4, 2)), ("c2", 6, (3, 2))])
def test_sharded_apply_and_matvec_bitwise(name, nranks, gg):
    cfg = CONFIGS[name]
    ref = Context(cfg.k, cfg.nsub, cfg.nsub)
    ref.factor()
    nf = ref.layout.N_cells - 1
    v = torch.from_numpy(probe_vector(ref.n, 3)).cuda()
    z_ref = ref.precond_apply(v)
    y_ref = ref.matvec(v)
    V = grid(v, nf)
    Z = torch.full_like(V, complex("nan"))
    Y = torch.full_like(V, complex("nan"))
    for r in range(nranks):
        c = Context(cfg.k, cfg.nsub, cfg.nsub, rank=r, nranks=nranks, gpu_grid=gg)
        c.factor()
        pl = c.plan
        ext = V[pl["ext_j0"] - 1:pl["ext_j1"] - 1, pl["ext_i0"] - 1:pl["ext_i1"] - 1].contiguous().view(-1)
        z = c.precond_apply_ext(ext)
        i0, i1, j0, j1 = pl["owned_i0"], pl["owned_i1"], pl["owned_j0"], pl["owned_j1"]
        Z[j0 - 1:j1 - 1, i0 - 1:i1 - 1] = z.view(j1 - j0, i1 - i0)
        nb = pl["nbr"]
        li, ri, dj, uj = int(nb[0] >= 0), int(nb[1] >= 0), int(nb[2] >= 0), int(nb[3] >= 0)
        ext1 = V[j0 - 1 - dj:j1 - 1 + uj, i0 - 1 - li:i1 - 1 + ri].contiguous().view(-1)
        y = c.matvec_ext(ext1)
        Y[j0 - 1:j1 - 1, i0 - 1:i1 - 1] = y.view(j1 - j0, i1 - i0)
        with pytest.raises(HelmError) as e:        # no communicator: collective entry points refuse
            c.precond_apply(torch.zeros(c.n, dtype=torch.complex128, device="cuda"))
        assert e.value.code == -4
        c.close()
    assert torch.equal(Z.view(-1), z_ref)
    assert torch.equal(Y.view(-1), y_ref)
    ref.close()


def test_c4_full_size_shards_full_vector():
    """k = 3200 (BASELINE.json configs[4], 128 x 128 subdomains, ~197 GB of factors: it needs >= 2 GPUs).
    Each half of the 2 x 1 rank grid is set up on this one GPU in turn as a communication-free shard (~99 GB of
    factors) and fed its ghost-framed input; its apply and matvec are compared ELEMENT BY ELEMENT on every owned node
    with the oracle's full apply (dedup mode, D24: one band LU per bitwise-distinct A_j, exact) and full matvec."""
    from oracle.oracle import Oracle
    cfg = CONFIGS["c4"]
    P = cfg.nsub
    o = Oracle.from_config(k=cfg.k, nsub_x=P, nsub_y=P)
    assert o.factor_dedup() <= 16
    v = probe_vector(o.nfree, int(cfg.k) + 1)
    nfx = o.nf[0]
    zo = o.apply(v).reshape(o.nf[1], nfx)
    yo = o.matvec(v).reshape(o.nf[1], nfx)
    o.release()
    V = grid(torch.from_numpy(v).cuda(), nfx)
    for r in (0, 1):
        c = Context(cfg.k, P, P, rank=r, nranks=2, gpu_grid=(2, 1))
        c.factor()
        pl = c.plan
        ext = V[pl["ext_j0"] - 1:pl["ext_j1"] - 1, pl["ext_i0"] - 1:pl["ext_i1"] - 1].contiguous().view(-1)
        i0, i1, j0, j1 = pl["owned_i0"], pl["owned_i1"], pl["owned_j0"], pl["owned_j1"]
        z = c.precond_apply_ext(ext).view(j1 - j0, i1 - i0).cpu().numpy()
        want = zo[j0 - 1:j1 - 1, i0 - 1:i1 - 1]
        assert np.linalg.norm(z - want) / np.linalg.norm(want) <= 1e-10
        nb = pl["nbr"]
        li, ri, dj, uj = int(nb[0] >= 0), int(nb[1] >= 0), int(nb[2] >= 0), int(nb[3] >= 0)
        ext1 = V[j0 - 1 - dj:j1 - 1 + uj, i0 - 1 - li:i1 - 1 + ri].contiguous().view(-1)
        y = c.matvec_ext(ext1).view(j1 - j0, i1 - i0).cpu().numpy()
        ywant = yo[j0 - 1:j1 - 1, i0 - 1:i1 - 1]
        assert np.linalg.norm(y - ywant) / np.linalg.norm(ywant) <= 1e-13
        c.close()
        del ext, ext1
        torch.cuda.empty_cache()

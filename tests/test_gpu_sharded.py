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


def test_c4_full_size_shards_sampled():
    """k = 3200 (BASELINE.json configs[4], 128 x 128 subdomains, ~197 GB of factors: it needs >= 2 GPUs).
    Each half of the 2 x 1 rank grid is set up on this one GPU in turn as a communication-free shard
    (~99 GB of factors), fed its ghost-framed input, and the oracle solves a sample of subdomains one by one
    -- corners, edges, interior, and the columns on both sides of the rank cut, whose full boxes read the
    ghost frame.  Matvec on sampled rows of each shard."""
    from oracle.oracle import Oracle
    cfg = CONFIGS["c4"]
    P = cfg.nsub
    o = Oracle.from_config(k=cfg.k, nsub_x=P, nsub_y=P)
    v = probe_vector(o.nfree, int(cfg.k) + 1)
    nfx = o.nf[0]
    picks = {0: [(0, 0), (63, 0), (0, 127), (63, 127), (63, 64), (31, 77), (62, 5)],
             1: [(64, 0), (127, 127), (64, 64), (100, 30), (127, 1)]}
    V = grid(torch.from_numpy(v).cuda(), nfx)
    rng = np.random.default_rng(7)
    for r in (0, 1):
        c = Context(cfg.k, P, P, rank=r, nranks=2, gpu_grid=(2, 1))
        c.factor()
        pl = c.plan
        ext = V[pl["ext_j0"] - 1:pl["ext_j1"] - 1, pl["ext_i0"] - 1:pl["ext_i1"] - 1].contiguous().view(-1)
        i0, i1, j0, j1 = pl["owned_i0"], pl["owned_i1"], pl["owned_j0"], pl["owned_j1"]
        z = c.precond_apply_ext(ext).view(j1 - j0, i1 - i0).cpu().numpy()
        subs = [bx + P * by for bx, by in picks[r]]
        o.factor(subs)
        zo = o.apply(v, subs=subs).reshape(o.nf[1], nfx)
        o.release()
        got, want = [], []
        for j in subs:
            s = o.subdomain(j)
            a0, a1 = max(s["own_lo"][0], 1), min(s["own_hi"][0], o.N[0])
            b0, b1 = max(s["own_lo"][1], 1), min(s["own_hi"][1], o.N[1])
            assert i0 <= a0 and a1 <= i1 and j0 <= b0 and b1 <= j1
            got.append(z[b0 - j0:b1 - j0, a0 - i0:a1 - i0].ravel())
            want.append(zo[b0 - 1:b1 - 1, a0 - 1:a1 - 1].ravel())
        got, want = np.concatenate(got), np.concatenate(want)
        assert np.linalg.norm(got - want) / np.linalg.norm(want) <= 1e-10
        nb = pl["nbr"]
        li, ri, dj, uj = int(nb[0] >= 0), int(nb[1] >= 0), int(nb[2] >= 0), int(nb[3] >= 0)
        ext1 = V[j0 - 1 - dj:j1 - 1 + uj, i0 - 1 - li:i1 - 1 + ri].contiguous().view(-1)
        y = c.matvec_ext(ext1).view(j1 - j0, i1 - i0).cpu().numpy()
        li_ = rng.integers(i0, i1, 20000)
        lj_ = rng.integers(j0, j1, 20000)
        rows = (li_ - 1) + nfx * (lj_ - 1)
        yo = o.matvec_rows(v, rows)
        yg = y[lj_ - j0, li_ - i0]
        assert np.linalg.norm(yg - yo) / np.linalg.norm(yo) <= 1e-13
        c.close()
        del ext, ext1
        torch.cuda.empty_cache()

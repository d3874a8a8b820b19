"""libhelm's NCCL data plane (P:109 parallel loop over subdomains, P:182-184 communication, P:228 one
processor per subdomain).

* One GPU: a ONE-RANK NCCL communicator (helm_setup with nranks = 1 and an NCCL id) runs the multi-rank code path --
  ghost-framed buffers, ncclCommInitRank, ncclAllReduce of every GMRES inner product and norm, ncclCommDestroy -- and
  must give the single-rank results (apply / matvec bitwise, same GMRES iterations, x to 1e-10) and the oracle's.
* Two or more GPUs (skipped on one): one process per GPU with a real N-rank communicator (grouped ncclSend/ncclRecv
  halos, ncclAllReduce): apply and matvec bitwise equal to one rank and within 1e-10 / 1e-13 of the oracle, GMRES
  iterations +-1 and x <= 1e-6 against the oracle, at c1 / c2, and c3 / c4 at full size against the oracle-only golden
  records.  Launched like bench.py --gpus N.
-m gpu."""
import os
import tempfile

import numpy as np
import pytest

from golden_util import golden_path, load_golden, sketch_rel
from oracle.oracle import Oracle, gmres as orc_gmres
from paper_2602_00735_b200.workloads import CONFIGS, probe_vector, sources

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():  # pragma: no cover - CPU box
    pytest.skip("needs a B200", allow_module_level=True)

from paper_2602_00735_b200 import Context  # noqa: E402
from paper_2602_00735_b200.helm import nccl_unique_id  # noqa: E402

NDEV = torch.cuda.device_count()


def rel(a, b):
    return float(np.linalg.norm(a - b) / np.linalg.norm(b))


@pytest.mark.parametrize("name", ["c1", "c2"])
def test_one_rank_nccl_communicator(name):
    cfg = CONFIGS[name]
    kw = dict(k=cfg.k, nsub_x=cfg.nsub, nsub_y=cfg.nsub)
    plain = Context(**kw)
    plain.factor()
    nc = Context(**kw, nccl_id=nccl_unique_id())
    nc.factor()
    assert plain.comm_info()["transport"] == "none"
    ci = nc.comm_info()
    assert ci == {"transport": "nccl", "nranks": 1, "rank": 0}
    v = torch.from_numpy(probe_vector(plain.n, int(cfg.k) + 1)).cuda()
    z0, y0 = plain.precond_apply(v), plain.matvec(v)
    z1, y1 = nc.precond_apply(v), nc.matvec(v)
    assert torch.equal(z0, z1) and torch.equal(y0, y1)
    b = plain.rhs(*sources(cfg))
    x0, i0, _ = plain.gmres(b, restart=cfg.restart, rtol=cfg.rtol)
    x1, i1, _ = nc.gmres(b, restart=cfg.restart, rtol=cfg.rtol)
    assert i1.status == 0 and i1.iterations == i0.iterations
    assert rel(x1.cpu().numpy(), x0.cpu().numpy()) <= 1e-10   # (the multi-rank lookahead closes columns differently)
    o = Oracle.from_config(**{"k": cfg.k, "nsub_x": cfg.nsub, "nsub_y": cfg.nsub})
    o.factor()
    vn, bn = v.cpu().numpy(), b.cpu().numpy()
    assert rel(z1.cpu().numpy(), o.apply(vn)) <= 1e-10
    assert rel(y1.cpu().numpy(), o.matvec(vn)) <= 1e-13
    go = orc_gmres(o.matvec, o.apply, bn, restart=cfg.restart, rtol=cfg.rtol)
    assert abs(i1.iterations - go.iterations) <= 1 and rel(x1.cpu().numpy(), go.x) <= 1e-6
    plain.close()
    nc.close()


def test_nccl_send_recv_transport_on_one_gpu():
    """The grouped ncclSend/ncclRecv transport every halo phase posts (nccl_sendrecv), run on a one-rank communicator
    with messages to itself: four messages of distinct sizes arrive intact (the send-to-self path is local -- no kernel
    waits on another process)."""
    nc = Context(100.0, 4, 4, nccl_id=nccl_unique_id())
    assert nc.comm_info()["transport"] == "nccl"
    assert nc.nccl_selftest(50_000, 4) == 0
    assert nc.nccl_selftest(7, 1) == 0
    plain = Context(100.0, 4, 4)
    from paper_2602_00735_b200 import HelmError
    with pytest.raises(HelmError):
        plain.nccl_selftest(10, 1)
    nc.close()
    plain.close()


# ------------------------------------------------------------------------------------------------- N GPUs
def spawn(nranks, kw, gg, job):
    import torch.multiprocessing as mp

    from nccl_worker import worker
    outdir = tempfile.mkdtemp(prefix="helm_nccl_")
    mp.spawn(worker, args=(nranks, nccl_unique_id(), kw, gg, job, outdir), nprocs=nranks, join=True)
    return outdir


GRIDS = {2: (2, 1), 4: (2, 2), 8: (4, 2)}
NRANKS = [n for n in (2, 4, 8) if n <= NDEV] or [2]


@pytest.mark.skipif(NDEV < 2, reason="needs >= 2 GPUs (one rank per GPU)")
@pytest.mark.parametrize("name", ["c1", "c2"])
@pytest.mark.parametrize("nranks", NRANKS)
def test_nccl_ranks_vs_one_rank_and_oracle(name, nranks):
    from nccl_worker import assemble, results
    cfg = CONFIGS[name]
    kw = dict(k=cfg.k, nsub_x=cfg.nsub, nsub_y=cfg.nsub)
    gg = GRIDS[nranks]
    if gg[0] > cfg.nsub or gg[1] > cfg.nsub:
        pytest.skip("more ranks than subdomains along an axis")
    seed = int(cfg.k) + 1
    outdir = spawn(nranks, kw, gg, {"probe_seed": seed, "gmres": {"config": name, "rtol": cfg.rtol}})
    res = results(outdir, nranks)
    assert all(r["comm"] == {"transport": "nccl", "nranks": nranks, "rank": q} for q, r in enumerate(res))
    ref = Context(**kw)
    ref.factor()
    nf = ref.layout.N_cells - 1
    v = probe_vector(nf * nf, seed)
    vt = torch.from_numpy(v).cuda()
    Z, Y, X = (assemble(outdir, nranks, nf, key) for key in ("z", "y", "x"))
    assert np.array_equal(Z, ref.precond_apply(vt).cpu().numpy())
    assert np.array_equal(Y, ref.matvec(vt).cpu().numpy())
    o = Oracle.from_config(k=cfg.k, nsub_x=cfg.nsub, nsub_y=cfg.nsub)
    o.factor()
    assert rel(Z, o.apply(v)) <= 1e-10 and rel(Y, o.matvec(v)) <= 1e-13
    bn = o.rhs(*sources(cfg))
    go = orc_gmres(o.matvec, o.apply, bn, restart=cfg.restart, rtol=cfg.rtol)
    its = {r["its"] for r in res}
    assert len(its) == 1 and abs(its.pop() - go.iterations) <= 1
    assert all(r["status"] == 0 for r in res)
    assert rel(X, go.x) <= 1e-6
    ref.close()


@pytest.mark.skipif(NDEV < 2, reason="needs >= 2 GPUs (one rank per GPU)")
@pytest.mark.parametrize("name", ["c3", "c4"])
def test_nccl_full_size_vs_golden(name):
    """c3 (and c4, 197 GB of factors: >= 2 GPUs) at full size on every GPU of the box, GMRES against the oracle-only
    golden: iterations +-1 (c4: the golden's first six cycles, maxit = 300), residual history to 1e-6, x sketch."""
    from nccl_worker import assemble, results
    if not os.path.exists(golden_path(name)):
        pytest.skip(f"no {name} golden record")
    g = load_golden(name)
    nranks = max(n for n in (2, 4, 8) if n <= NDEV)
    cfg = CONFIGS[name]
    kw = dict(k=cfg.k, nsub_x=cfg.nsub, nsub_y=cfg.nsub)
    outdir = spawn(nranks, kw, GRIDS[nranks], {"gmres": {"config": name, "rtol": cfg.rtol, "maxit": g["maxit"]}})
    res = results(outdir, nranks)
    nf = int(round(np.sqrt(g["n_free"])))
    X = assemble(outdir, nranks, nf, "x")
    its = res[0]["its"]
    assert all(r["its"] == its for r in res) and abs(its - g["iterations"]) <= 1
    assert res[0]["status"] == g["status"]
    h, ho = np.asarray(res[0]["hist"]), np.asarray(g["history"])
    n = min(len(h), len(ho))
    assert np.max(np.abs(h[:n] - ho[:n]) / ho[:n]) <= 1e-6
    assert sketch_rel(X, g) <= 1e-6

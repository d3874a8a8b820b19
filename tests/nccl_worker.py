"""One rank of a multi-GPU test (tests/test_gpu_nccl.py): a process per GPU, libhelm's own NCCL communicator
(helm_setup with an NCCL unique id), the collective entry points on the rank's owned piece of a global vector; the
owned results are written to `outdir` for the parent to assemble.  Not a test module (no test_ prefix)."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def owned(vec: np.ndarray, nf: int, pl: dict) -> np.ndarray:
    V = vec.reshape(nf, nf)
    return np.ascontiguousarray(V[pl["owned_j0"] - 1:pl["owned_j1"] - 1, pl["owned_i0"] - 1:pl["owned_i1"] - 1]).ravel()


def worker(rank: int, nranks: int, nccl_id: bytes, kw: dict, gg, job: dict, outdir: str):
    import torch

    from paper_2602_00735_b200 import Context
    from paper_2602_00735_b200.workloads import CONFIGS, probe_vector, sources

    torch.cuda.set_device(rank)
    s = torch.cuda.Stream()
    torch.cuda.set_stream(s)
    c = Context(**kw, gpu_grid=gg, rank=rank, nranks=nranks, stream=s, nccl_id=nccl_id)
    c.factor()
    pl = c.plan
    nf = c.layout.N_cells - 1
    out = {"plan": pl, "comm": c.comm_info()}
    if "probe_seed" in job:
        v = probe_vector(nf * nf, job["probe_seed"])
        vl = torch.from_numpy(owned(v, nf, pl)).cuda()
        out["z"] = c.precond_apply(vl).cpu().numpy()
        out["y"] = c.matvec(vl).cpu().numpy()
    if "gmres" in job:
        g = job["gmres"]
        if "config" in g:
            cfg = CONFIGS[g["config"]]
            b = c.rhs(*sources(cfg))
        else:
            b = torch.from_numpy(owned(np.load(g["b_path"]), nf, pl)).cuda()
        x, info, hist = c.gmres(b, restart=g.get("restart", 50), rtol=g.get("rtol", 1e-6), maxit=g.get("maxit", 5000),
                                history=True)
        out.update(x=x.cpu().numpy(), its=info.iterations, status=info.status, relres_true=info.relres_true,
                   hist=hist)
    torch.cuda.synchronize()
    c.close()
    np.save(os.path.join(outdir, f"rank{rank}.npy"), np.array([out], dtype=object), allow_pickle=True)


def assemble(outdir: str, nranks: int, nf: int, key: str) -> np.ndarray:
    """Global vector from the ranks' owned pieces (NaN where no rank wrote)."""
    G = np.full((nf, nf), np.nan + 0j)
    for r in range(nranks):
        o = np.load(os.path.join(outdir, f"rank{r}.npy"), allow_pickle=True)[0]
        pl = o["plan"]
        G[pl["owned_j0"] - 1:pl["owned_j1"] - 1, pl["owned_i0"] - 1:pl["owned_i1"] - 1] = o[key].reshape(
            pl["owned_j1"] - pl["owned_j0"], pl["owned_i1"] - pl["owned_i0"])
    return G.ravel()


def results(outdir: str, nranks: int) -> list:
    return [np.load(os.path.join(outdir, f"rank{r}.npy"), allow_pickle=True)[0] for r in range(nranks)]

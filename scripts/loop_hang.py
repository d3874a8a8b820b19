"""Debug aid: repeat one loopback random-layout case (apply + matvec on 4 in-process ranks) and dump every thread's
Python stack if an iteration stalls."""
import faulthandler
import os
import sys
import threading

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2602_00735_b200 import Context  # noqa: E402
from paper_2602_00735_b200.workloads import probe_vector  # noqa: E402

kw = dict(k=120.0, nsub_x=3, nsub_y=6, local_bc=0, pou=0)
gg = (2, 2)
reps = int(sys.argv[1]) if len(sys.argv) > 1 else 20
ref = Context(**kw)
ref.factor()
nf = ref.layout.N_cells - 1
v = torch.from_numpy(probe_vector(ref.n, 12)).cuda()
z_ref, y_ref = ref.precond_apply(v), ref.matvec(v)
ref.close()
V = v.view(nf, nf)


def owned(vec2d, pl):
    return vec2d[pl["owned_j0"] - 1:pl["owned_j1"] - 1, pl["owned_i0"] - 1:pl["owned_i1"] - 1].contiguous().view(-1)


for it in range(reps):
    gid = 1000 + it
    res = [None] * 4
    stage = ["start"] * 4

    def rank(r):
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            stage[r] = "setup"
            c = Context(**kw, gpu_grid=gg, rank=r, nranks=4, stream=s, loopback_group=gid)
            stage[r] = "factor"
            c.factor()
            pl = c.plan
            vl = owned(V, pl)
            stage[r] = "apply"
            z = c.precond_apply(vl)
            stage[r] = "matvec"
            y = c.matvec(vl)
            stage[r] = "sync"
            s.synchronize()
            res[r] = (pl, z.clone(), y.clone(), c.layout.overlap_interior)
            stage[r] = "close"
            c.close()
            stage[r] = "done"

    th = [threading.Thread(target=rank, args=(r,), daemon=True) for r in range(4)]
    for t in th:
        t.start()
    for t in th:
        t.join(60)
    if any(t.is_alive() for t in th):
        print(f"iteration {it}: STALL, stages {stage}", flush=True)
        faulthandler.dump_traceback(all_threads=True)
        os._exit(3)
    Z, Y = torch.full_like(V, complex("nan")), torch.full_like(V, complex("nan"))
    for pl, z, y, ov in res:
        sl = (slice(pl["owned_j0"] - 1, pl["owned_j1"] - 1), slice(pl["owned_i0"] - 1, pl["owned_i1"] - 1))
        shape = (pl["owned_j1"] - pl["owned_j0"], pl["owned_i1"] - pl["owned_i0"])
        Z[sl], Y[sl] = z.view(shape), y.view(shape)
    ok = torch.equal(Z.view(-1), z_ref) and torch.equal(Y.view(-1), y_ref)
    print(f"iteration {it}: ok={ok} overlap={[r[3] for r in res]}", flush=True)

"""Small end-to-end runs of every kernel family (for compute-sanitizer): P1 plain and cluster-split apply, Q1 cluster
factorisation + split apply, ramp PoU, Richardson, GMRES."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2602_00735_b200 import Context  # noqa: E402
from paper_2602_00735_b200.helm import POU_RAMP, paper_params  # noqa: E402
from paper_2602_00735_b200.workloads import paper_source, probe_vector, sources, CONFIGS  # noqa: E402

for kw in [dict(k=20.0, nsub_x=2, nsub_y=2), dict(k=100.0, nsub_x=4, nsub_y=4, pou=POU_RAMP),
           dict(k=100.0, nsub_x=4, nsub_y=4, local_bc=1), paper_params(60.0, 2, 4, 2), paper_params(80.0, 1, 4, 2),
           dict(k=400.0, nsub_x=16, nsub_y=16)]:
    ctx = Context(**kw)
    ctx.factor()
    v = torch.from_numpy(probe_vector(ctx.n, 1)).cuda()
    z = ctx.precond_apply(v)
    y = ctx.matvec(z)
    if "n_cells" in kw:
        xy, amp, s = paper_source(kw["k"])
    else:
        xy, amp, s = sources(CONFIGS["c0"])
    b = ctx.rhs(xy, amp, s)
    ctx.gmres(b, restart=20, rtol=1e-6, maxit=30)
    ctx.richardson(b, rtol=1e-6, maxit=5)
    torch.cuda.synchronize()
    print("ok", kw.get("k"), kw.get("nsub_x"), flush=True)
    ctx.close()

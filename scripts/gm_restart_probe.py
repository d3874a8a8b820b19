import os, sys
sys.path.insert(0, '/root/repo')
import torch
from paper_2602_00735_b200 import Context
from paper_2602_00735_b200.helm import paper_params
from paper_2602_00735_b200.workloads import paper_source
for k, P, pml, ov, grid in [(300., 2, 8, 4, 600), (600., 4, 11, 5, 1200), (1200., 8, 15, 6, 2400)]:
    for bc in (1, 0):
        ctx = Context(**paper_params(k, P, pml, ov, n_cells=grid, local_bc=bc))
        ctx.factor()
        xy, amp, s = paper_source(k)
        b = ctx.rhs(xy, amp, s)
        out = []
        for rs in (10, 20, 30, 50):
            _, info, _ = ctx.gmres(b, restart=rs, rtol=1e-10, maxit=500)
            out.append((rs, info.iterations))
        print(k, 'imp' if bc else 'drch', out, flush=True)
        ctx.close(); torch.cuda.empty_cache()

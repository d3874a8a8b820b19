"""Profiling driver: a few cluster-split applies on one paper workload (argv[1], default t300)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2602_00735_b200 import Context  # noqa: E402
from paper_2602_00735_b200.helm import paper_params  # noqa: E402
from paper_2602_00735_b200.workloads import PAPER_CONFIGS, probe_vector  # noqa: E402

c = PAPER_CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "t300"]
ctx = Context(**paper_params(c.k, c.nsub, c.pml, c.ovlp, n_cells=c.n_cells))
ctx.factor()
v = torch.from_numpy(probe_vector(ctx.n, 5)).cuda()
z = ctx.precond_apply(v)
for _ in range(3):
    ctx.precond_apply(v, z)
torch.cuda.synchronize()
print("ok", ctx.layout.apply_bytes)

"""Profiling driver: one factorisation (argv[1] = BJ config c0..c4 or paper config t300..)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2602_00735_b200 import Context  # noqa: E402
from paper_2602_00735_b200.helm import paper_params  # noqa: E402
from paper_2602_00735_b200.workloads import CONFIGS, PAPER_CONFIGS  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "c2"
if name in CONFIGS:
    c = CONFIGS[name]
    ctx = Context(c.k, c.nsub, c.nsub)
else:
    c = PAPER_CONFIGS[name]
    ctx = Context(**paper_params(c.k, c.nsub, c.pml, c.ovlp, n_cells=c.n_cells))
torch.cuda.synchronize()
t = time.time()
ctx.factor()
print(name, "factor %.3f s" % (time.time() - t), "bytes %.2f GB" % (ctx.layout.factor_bytes / 1e9))

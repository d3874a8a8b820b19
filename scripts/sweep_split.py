"""Development sweep: cluster-split apply time vs G on the paper workloads."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2602_00735_b200 import Context  # noqa: E402
from paper_2602_00735_b200.helm import paper_params  # noqa: E402
from paper_2602_00735_b200.workloads import PAPER_CONFIGS, probe_vector  # noqa: E402

for name in sys.argv[1].split(","):
    c = PAPER_CONFIGS[name]
    for G in sys.argv[2].split(","):
        if G == "auto":
            os.environ.pop("HELM_SPLIT_G", None)
        else:
            os.environ["HELM_SPLIT_G"] = G
        ctx = Context(**paper_params(c.k, c.nsub, c.pml, c.ovlp, n_cells=c.n_cells))
        ctx.factor()
        v = torch.from_numpy(probe_vector(ctx.n, 5)).cuda()
        z = ctx.precond_apply(v)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            ctx.precond_apply(v, z)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        print(name, "G", G, "apply %.3f ms %.0f GB/s" % (ms, ctx.layout.apply_bytes / ms / 1e6), flush=True)
        ctx.close()
        del ctx, v, z
        torch.cuda.empty_cache()

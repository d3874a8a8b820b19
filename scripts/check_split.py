"""Development check: cluster-split apply vs the one-CTA-per-subdomain apply (bitwise) on a few workloads."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2602_00735_b200 import Context  # noqa: E402
from paper_2602_00735_b200.helm import paper_params  # noqa: E402
from paper_2602_00735_b200.workloads import probe_vector  # noqa: E402

cases = [dict(k=20.0, nsub_x=2, nsub_y=2), dict(k=100.0, nsub_x=4, nsub_y=4),
         paper_params(100.0, 2, 6, 3), paper_params(150.0, 3, 6, 3, local_bc=0), paper_params(300.0, 2, 8, 4)]
for kw in cases:
    out = {}
    for G in ("0", ""):
        if G:
            os.environ["HELM_SPLIT_G"] = G
        else:
            os.environ.pop("HELM_SPLIT_G", None)
        ctx = Context(**kw)
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
        out[G] = (z.clone(), e0.elapsed_time(e1) / 5, ctx.layout.apply_bytes)
        ctx.close()
    a, b = out["0"][0], out[""][0]
    print(kw.get("k"), kw.get("nsub_x"), "bitwise" if torch.equal(a, b) else "DIFF %.3e" % (
        (a - b).abs().max().item() / a.abs().max().item()),
        "plain %.3f ms split %.3f ms (%.0f GB/s)" % (out["0"][1], out[""][1], out[""][2] / out[""][1] / 1e6), flush=True)

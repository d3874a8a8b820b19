"""Factorisation time (CUDA events around helm_factor, best of 3 contexts) per config, with the default 8-wide panels;
HELM_LIB_PATH times another build of libhelm (A/B of compile-time variants).  python scripts/factor_time.py c2 c3"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_00735_b200 import build  # noqa: E402

if os.environ.get("HELM_LIB_PATH"):      # time another build of libhelm (A/B of compile-time variants)
    build.LIB = os.environ["HELM_LIB_PATH"]
import torch  # noqa: E402

from paper_2602_00735_b200 import helm  # noqa: E402
from paper_2602_00735_b200 import Context  # noqa: E402

helm.load(build_if_missing=False)
from paper_2602_00735_b200.workloads import CONFIGS  # noqa: E402

for name in sys.argv[1:] or ["c3"]:
    c = CONFIGS[name]
    for look, panel in (("1", "8"),):
        os.environ["HELM_FACTOR_PANEL"] = panel
        best = None
        for _ in range(3):
            ctx = Context(c.k, c.nsub, c.nsub)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            torch.cuda.synchronize()
            e0.record()
            ctx.factor()
            e1.record()
            torch.cuda.synchronize()
            t = e0.elapsed_time(e1) / 1e3
            best = t if best is None else min(best, t)
            ctx.close()
            del ctx
            torch.cuda.empty_cache()
        print(f"{name} panel={panel} lookahead={look} factor {best:.4f} s", flush=True)

"""Phase profile of the shared-memory factorisation (k_factor_chains, CTA 0) from libhelm_prof.so, a build with
-DHELM_FACTOR_PROF:  HELM_NVCC_EXTRA=-DHELM_FACTOR_PROF (LIB -> libhelm_prof.so) then  python scripts/factor_phases.py c3"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_00735_b200 import build  # noqa: E402

build.LIB = build.LIB.replace("libhelm.so", "libhelm_prof.so")
import torch  # noqa: E402

from paper_2602_00735_b200 import helm  # noqa: E402
from paper_2602_00735_b200.workloads import CONFIGS  # noqa: E402

helm.load(build_if_missing=False)
for name in sys.argv[1:] or ["c3"]:
    c = CONFIGS[name]
    for look, panel in (("1", "8"),):
        os.environ["HELM_FACTOR_LOOKAHEAD"] = look
        os.environ["HELM_FACTOR_PANEL"] = panel
        ctx = helm.Context(c.k, c.nsub, c.nsub)
        ctx.factor()
        torch.cuda.synchronize()
        print(name, "panel", panel, "lookahead", look, flush=True)
        ctx.close()

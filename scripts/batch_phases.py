"""Phase profile of the tensor-core apply (k_apply_batch, CTA 0, thread 0) from libhelm_prof.so, a build with
-DHELM_BATCH_PROF:  HELM_NVCC_EXTRA=-DHELM_BATCH_PROF with LIB -> libhelm_prof.so, then
python scripts/batch_phases.py c3   (prints one BPROF line per apply)"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2602_00735_b200 import build  # noqa: E402

build.LIB = build.LIB.replace("libhelm.so", "libhelm_prof.so")
if len(sys.argv) > 1 and sys.argv[1] == "--build":
    os.environ["HELM_NVCC_EXTRA"] = "-DHELM_BATCH_PROF"
    build.build(force=True)
    sys.exit(0)
import torch  # noqa: E402

from paper_2602_00735_b200 import helm  # noqa: E402
from paper_2602_00735_b200.workloads import CONFIGS, probe_vector  # noqa: E402

helm.load(build_if_missing=False)
for name in sys.argv[1:] or ["c3"]:
    c = CONFIGS[name]
    ctx = helm.Context(c.k, c.nsub, c.nsub)
    ctx.factor()
    v = torch.from_numpy(probe_vector(ctx.n, 7)).cuda()
    for _ in range(2):
        ctx.precond_apply(v)
    torch.cuda.synchronize()
    ctx.close()

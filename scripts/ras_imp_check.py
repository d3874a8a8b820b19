"""RAS-Imp (the paper's third column in Tables 1-2: no local PML, impedance directly on the subdomain faces) on the
GPU path: Richardson and GMRES counts at k = 300 / 600 / 1200 (development check)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2602_00735_b200 import Context  # noqa: E402
from paper_2602_00735_b200.helm import paper_params  # noqa: E402
from paper_2602_00735_b200.workloads import paper_source  # noqa: E402

for k, P, ov in [(300.0, 2, 4), (600.0, 4, 5), (1200.0, 8, 6)]:
    ctx = Context(**paper_params(k, P, 0, ov, n_cells=int(2 * k)))
    ctx.factor()
    b = ctx.rhs(*paper_source(k))
    _, ri, _ = ctx.richardson(b, rtol=1e-10, maxit=500)
    _, gi, _ = ctx.gmres(b, restart=50, rtol=1e-10, maxit=500)
    print(f"k={k:g} RAS-Imp richardson its {ri.iterations} relres {ri.relres:.2e} status {ri.status} | "
          f"gmres its {gi.iterations} relres {gi.relres_true:.2e}", flush=True)
    ctx.close()
    torch.cuda.empty_cache()

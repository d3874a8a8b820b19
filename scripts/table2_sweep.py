"""Table 2 ("GMRES ... with slightly thin PML thickness"): GMRES(50) iteration counts to rtol 1e-10 for
local PML widths below the printed ones, RAS-PML-Imp and -Drch, at the Table 2 rows that fit one GPU.  Prints one line
per (k, pml): the widths whose counts match the printed 11/12, 19/19, 48/49 would be the caption's set-up."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2602_00735_b200 import Context  # noqa: E402
from paper_2602_00735_b200.helm import paper_params  # noqa: E402
from paper_2602_00735_b200.workloads import paper_source  # noqa: E402

ROWS = [(300.0, 600, 2, 8, 4, (11, 12)), (600.0, 1200, 4, 11, 5, (19, 19)), (1200.0, 2400, 8, 15, 6, (48, 49))]
for k, grid, P, pml_p, ov, printed in ROWS:
    for pml in range(1, pml_p + 1):
        its = []
        for bc in (1, 0):
            ctx = Context(**paper_params(k, P, pml, ov, n_cells=grid, local_bc=bc))
            ctx.factor()
            b = ctx.rhs(*paper_source(k))
            _, info, _ = ctx.gmres(b, restart=50, rtol=1e-10, maxit=500)
            its.append(info.iterations)
            ctx.close()
            del ctx, b
            torch.cuda.empty_cache()
        print(f"k={k:g} pml={pml} ovlp={ov}: imp {its[0]} drch {its[1]}   (printed at pml={pml_p}: {printed})",
              flush=True)

"""Run every Richardson / GMRES row of tests/golden/paper_iterations.txt that fits one GPU (k <= 1200) on the GPU path
and print a markdown table: printed iterations (paper, line cited) vs ours, with our final relative residual."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2602_00735_b200 import Context  # noqa: E402
from paper_2602_00735_b200.helm import paper_params  # noqa: E402
from paper_2602_00735_b200.workloads import paper_source  # noqa: E402

GOLDEN = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests", "golden",
                      "paper_iterations.txt")
rows = []
for line in open(GOLDEN):
    if line.startswith("#") or not line.strip():
        continue
    t, ln, k, grid, P, pml, ov, bc, solver, its, rr = line.split()
    if float(k) <= 1200:
        rows.append((t, int(ln), float(k), int(grid), int(P), int(pml), int(ov), bc, solver, int(its), rr))
print("| table (PAPER.md line) | k | grid | N | pml | ovlp | local BC | solver | printed its | ours | ours - printed | our relres |")
print("|---|---|---|---|---|---|---|---|---|---|---|---|")
for t, ln, k, grid, P, pml, ov, bc, solver, its, rr in rows:
    ctx = Context(**paper_params(k, P, 0 if bc == "rasimp" else pml, ov, n_cells=grid, local_bc=0 if bc == "drch" else 1))
    ctx.factor()
    xy, amp, s = paper_source(k)
    b = ctx.rhs(xy, amp, s)
    if solver == "richardson":
        _, info, _ = ctx.richardson(b, rtol=1e-10, maxit=500)
        got, res = info.iterations, info.relres
        if info.status == 4:
            got = f"div@{info.iterations}"
    else:
        _, info, _ = ctx.gmres(b, restart=50, rtol=1e-10, maxit=500)
        got, res = info.iterations, info.relres_true
    diff = f"{got - its:+d}" if isinstance(got, int) else "-"
    print(f"| {t} (P:{ln}) | {k:g} | {grid}^2 | {P * P} | {pml if bc != 'rasimp' else 0} | {ov} | {bc} | {solver} | {its} | "
          f"{got} | {diff} | {res:.2e} |", flush=True)
    ctx.close()
    del ctx, b
    torch.cuda.empty_cache()

# Sweep of the cluster-split apply's G (CTAs per chain) on t300 / t600 (HELM_SPLIT_G forces it; 0 = the automatic choice).
#   bash scripts/split_g_sweep.sh   -- measured r01: t300 auto(G=8) 1.47 ms, G=6 1.61, G=4 1.93; t600 auto(G=3) 3.24, G=4 4.66
for g in 0 2 3 4 5 6 8; do
  if [ $g = 0 ]; then unset HELM_SPLIT_G; else export HELM_SPLIT_G=$g; fi
  HELM_DEBUG_CONFIG=1 python - <<'PY' 2>&1 | grep -E "helm rank|apply ms"
import torch, sys, os
sys.path.insert(0, ".")
from paper_2602_00735_b200 import Context
from paper_2602_00735_b200.helm import paper_params
from paper_2602_00735_b200.workloads import PAPER_CONFIGS
for name in ("t300", "t600"):
    c = PAPER_CONFIGS[name]
    ctx = Context(**paper_params(c.k, c.nsub, c.pml, c.ovlp, n_cells=c.n_cells)); ctx.factor()
    v = torch.randn(ctx.n, dtype=torch.complex128, device="cuda")
    for _ in range(2): ctx.precond_apply(v)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): ctx.precond_apply(v)
    e1.record(); torch.cuda.synchronize()
    print(name, "G", os.environ.get("HELM_SPLIT_G", "auto"), "apply ms", round(e0.elapsed_time(e1) / 10, 3), flush=True)
    ctx.close()
PY
done

# Sweep of k_apply_split's ring (HELM_SPLIT_SLOTS cap, HELM_SPLIT_SLOTB slot bytes) on the paper workloads.
#   bash scripts/split_ring_sweep.sh
for cfg in "16 16384" "16 32000" "16 48000" "16 80000" "16 16384" "16 32000" "16 48000" "16 80000"; do set -- $cfg; HELM_SPLIT_SLOTS=$1 HELM_SPLIT_SLOTB=$2 python - <<'PY'
import os, torch
from paper_2602_00735_b200 import Context
from paper_2602_00735_b200.helm import paper_params
from paper_2602_00735_b200.workloads import PAPER_CONFIGS
out = []
for name in ("t300", "t600", "t1200"):
    c = PAPER_CONFIGS[name]
    ctx = Context(**paper_params(c.k, c.nsub, c.pml, c.ovlp, n_cells=c.n_cells)); ctx.factor()
    torch.manual_seed(0)
    v = torch.randn(ctx.n, dtype=torch.complex128, device="cuda")
    for _ in range(2): ctx.precond_apply(v)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): ctx.precond_apply(v)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    out.append(f"{name} {ms:.3f} ms {ctx.layout.apply_bytes / ms / 1e6:.0f} GB/s")
    ctx.close(); del ctx; torch.cuda.empty_cache()
print("cfg", os.environ["HELM_SPLIT_SLOTS"], os.environ["HELM_SPLIT_SLOTB"], " | ".join(out), flush=True)
PY
done

# Sweep of k_apply's ring (HELM_APPLY_SLOTS slots of ~HELM_APPLY_SLOTB bytes) at c3 on one GPU, configurations
# interleaved; every configuration must give bitwise the same z (checked at the end against the first one).
#   bash scripts/apply_ring_sweep.sh
for cfg in "2 20000" "8 12288" "6 8192" "3 12288" "2 26000" "2 20000" "8 12288" "6 8192" "3 12288" "2 26000"; do set -- $cfg; HELM_APPLY_SLOTS=$1 HELM_APPLY_SLOTB=$2 python - <<'PY'
import os, torch
from paper_2602_00735_b200 import Context
from paper_2602_00735_b200.workloads import CONFIGS
cfg=CONFIGS["c3"]; c=Context(cfg.k,cfg.nsub,cfg.nsub); c.factor()
torch.manual_seed(0)
v=torch.randn(c.n,dtype=torch.complex128,device="cuda")
z0=c.precond_apply(v).clone()
for _ in range(2): c.precond_apply(v)
torch.cuda.synchronize()
e0,e1=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
best=1e9
for rep in range(3):
    e0.record()
    for _ in range(10): c.precond_apply(v)
    e1.record(); torch.cuda.synchronize()
    best=min(best, e0.elapsed_time(e1)/10)
tag=os.environ["HELM_APPLY_SLOTS"]+"_"+os.environ["HELM_APPLY_SLOTB"]
print("cfg", tag, "apply ms", round(best,3), "GB/s", round(c.layout.apply_bytes/(best*1e-3)/1e9), flush=True)
torch.save(z0.cpu(), f"/tmp/z_{tag}.pt")
PY
done
python -c "
import torch, glob
a=torch.load('/tmp/z_2_20000.pt')
for f in sorted(glob.glob('/tmp/z_*.pt')): print(f, torch.equal(a, torch.load(f)))
"

"""c4 (k = 3200, 16384 subdomains) apply on one GPU, CUDA events over 10 applies (development aid)."""
import os, sys, time
sys.path.insert(0, os.getcwd())
import torch
from paper_2602_00735_b200 import Context
from paper_2602_00735_b200.workloads import CONFIGS, probe_vector
cfg = CONFIGS["c4"]
ctx = Context(cfg.k, cfg.nsub, cfg.nsub); ctx.factor()
v = torch.from_numpy(probe_vector(ctx.n, 7)).cuda(); z = torch.empty_like(v)
for _ in range(3): ctx.precond_apply(v, z)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10): ctx.precond_apply(v, z)
e1.record(); torch.cuda.synchronize()
print("c4 apply", e0.elapsed_time(e1)/10, "ms", ctx.factor_classes(), flush=True)

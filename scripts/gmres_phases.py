"""Live per-phase times of the GMRES(50) Arnoldi step at c3 (HELM_GMRES_PHASES=1: CUDA events between the phases,
totals printed to stderr when the context closes).  HELM_GMRES_PHASES=1 python scripts/gmres_phases.py"""
import os, sys, time, torch
sys.path.insert(0, '.')
from paper_2602_00735_b200 import Context
from paper_2602_00735_b200.workloads import CONFIGS, sources
cfg = CONFIGS["c3"]
s = torch.cuda.Stream(); torch.cuda.set_stream(s)
ctx = Context(cfg.k, cfg.nsub, cfg.nsub, stream=s); ctx.factor()
b = ctx.rhs(*sources(cfg))
x = torch.zeros_like(b)
ctx.gmres(b, x, restart=50, rtol=0.0, maxit=5)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
x.zero_(); e0.record(s)
ctx.gmres(b, x, restart=50, rtol=0.0, maxit=100)
e1.record(s); torch.cuda.synchronize()
print("total ms", e0.elapsed_time(e1), flush=True)
ctx.close()

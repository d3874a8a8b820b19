"""GPU-only timing probe for one config (development aid)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2602_00735_b200 import Context
from paper_2602_00735_b200.workloads import CONFIGS, probe_vector, sources

name = sys.argv[1] if len(sys.argv) > 1 else "c3"
cfg = CONFIGS[name]
t0 = time.time()
ctx = Context(cfg.k, cfg.nsub, cfg.nsub)
torch.cuda.synchronize(); t1 = time.time()
ctx.factor(); t2 = time.time()
L = ctx.layout
print(name, "setup %.3fs factor %.3fs" % (t1 - t0, t2 - t1), L.as_dict(), flush=True)
v = torch.from_numpy(probe_vector(ctx.n, int(cfg.k) + 1)).cuda()
z = torch.empty_like(v)
for _ in range(3): ctx.precond_apply(v, z)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(10): ctx.precond_apply(v, z)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
print("apply %.3f ms -> %.1f GB/s algorithmic, %.1f GB/s band-equivalent" % (ms, L.apply_bytes / ms / 1e6, L.band_bytes / ms / 1e6), flush=True)
e0.record()
for _ in range(10): ctx.matvec(v, z)
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 10
print("spmv %.3f ms -> %.1f GB/s" % (ms, L.spmv_bytes / ms / 1e6), flush=True)
xy, amp, sig = sources(cfg)
b = ctx.rhs(xy, amp, sig)
torch.cuda.synchronize(); t = time.time()
x, info, hist = ctx.gmres(b, history=True)
torch.cuda.synchronize(); tts = time.time() - t
print("gmres its %d restarts %d status %d relres %.3e applies %d TTS %.3fs (%.2f ms/it)" % (
    info.iterations, info.restarts, info.status, info.relres_true, info.applies, tts, 1e3 * tts / max(1, info.iterations)), flush=True)
print("hist", [float("%.3e" % h) for h in hist[::10]])

"""Predict strong scaling of the apply at N GPUs from one GPU: every rank's shard of a config (communication-free
`_ext` entry point, the ghost frame supplied by the caller) is factored and its apply timed alone with CUDA events.
max over ranks vs (full apply) / N gives the load-balance part of the scaling efficiency (no communication)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2602_00735_b200 import Context  # noqa: E402
from paper_2602_00735_b200.workloads import CONFIGS  # noqa: E402


def timed(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


name = sys.argv[1] if len(sys.argv) > 1 else "c3"
Ns = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [2, 4, 8]
cfg = CONFIGS[name]
if name == "c4":   # 198 GB of factors: no one-GPU reference; the shards alone (ideal = sum of shard bytes at the mean)
    probe = Context(cfg.k, cfg.nsub, cfg.nsub, rank=0, nranks=Ns[0])
    nf = probe.layout.N_cells - 1
    probe.close()
    V = torch.randn(nf * nf, dtype=torch.complex128, device="cuda").view(nf, nf)
    t1 = None
else:
    full = Context(cfg.k, cfg.nsub, cfg.nsub)
    full.factor()
    v = torch.randn(full.n, dtype=torch.complex128, device="cuda")
    t1 = timed(lambda: full.precond_apply(v))
    nf = full.layout.N_cells - 1
    V = v.view(nf, nf)
    full.close()
    del full
    torch.cuda.empty_cache()
    print(f"{name} N=1 apply {t1:.3f} ms", flush=True)
for N in Ns:
    ts = []
    for r in range(N):
        c = Context(cfg.k, cfg.nsub, cfg.nsub, rank=r, nranks=N)
        c.factor()
        pl = c.plan
        ext = V[pl["ext_j0"] - 1:pl["ext_j1"] - 1, pl["ext_i0"] - 1:pl["ext_i1"] - 1].contiguous().view(-1)
        ts.append(timed(lambda: c.precond_apply_ext(ext)))
        c.close()
        del c
        torch.cuda.empty_cache()
    ideal = t1 / N if t1 else sum(ts) / N
    print(f"{name} N={N} shard apply ms: max {max(ts):.3f} mean {sum(ts) / N:.3f} ideal {ideal:.3f} "
          f"-> balance efficiency {ideal / max(ts):.3f}  {['%.3f' % t for t in ts]}", flush=True)

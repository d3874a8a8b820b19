"""GPU-only timing probe for the paper's workloads (Table 4 / Table 1 rows; development aid)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2602_00735_b200 import Context  # noqa: E402
from paper_2602_00735_b200.helm import paper_params  # noqa: E402
from paper_2602_00735_b200.workloads import PAPER_CONFIGS, paper_source, probe_vector  # noqa: E402

for name in sys.argv[1:]:
    cfg = PAPER_CONFIGS[name]
    torch.cuda.synchronize()
    t0 = time.time()
    ctx = Context(**paper_params(cfg.k, cfg.nsub, cfg.pml, cfg.ovlp, n_cells=cfg.n_cells, local_bc=cfg.local_bc))
    torch.cuda.synchronize()
    t1 = time.time()
    ctx.factor()
    t2 = time.time()
    L = ctx.layout
    print(name, "setup %.3fs factor %.3fs m_max %d factor %.2f GB apply_bytes %.2f GB" % (
        t1 - t0, t2 - t1, L.m_max, L.factor_bytes / 1e9, L.apply_bytes / 1e9), flush=True)
    v = torch.from_numpy(probe_vector(ctx.n, 7)).cuda()
    z = torch.empty_like(v)
    for _ in range(2):
        ctx.precond_apply(v, z)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        ctx.precond_apply(v, z)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print("  apply %.3f ms -> %.1f GB/s algorithmic" % (ms, L.apply_bytes / ms / 1e6), flush=True)
    xy, amp, s = paper_source(cfg.k)
    b = ctx.rhs(xy, amp, s)
    torch.cuda.synchronize()
    t = time.time()
    x, info, _ = ctx.richardson(b, rtol=cfg.rtol, maxit=cfg.maxit)
    torch.cuda.synchronize()
    tr = time.time() - t
    t = time.time()
    x, ginfo, _ = ctx.gmres(b, restart=50, rtol=cfg.rtol, maxit=cfg.maxit)
    torch.cuda.synchronize()
    tg = time.time() - t
    print("  richardson its %d relres %.2e  %.3fs | gmres its %d relres %.2e %.3fs" % (
        info.iterations, info.relres, tr, ginfo.iterations, ginfo.relres_true, tg), flush=True)
    ctx.close()
    del ctx, v, z, b, x
    torch.cuda.empty_cache()

"""Shared-factor apply (D28) vs the per-subdomain streaming apply on the same seeded vector: classes, factor time,
apply time, relative difference, and a GMRES(50) solve with each (development aid, one GPU).

    python scripts/batch_check.py c2 c3 [--gmres]
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2602_00735_b200 import Context  # noqa: E402
from paper_2602_00735_b200.workloads import CONFIGS, probe_vector, sources  # noqa: E402

names = [a for a in sys.argv[1:] if not a.startswith("--")] or ["c3"]
do_gmres = "--gmres" in sys.argv
for name in names:
    cfg = CONFIGS[name]
    out = {}
    for mode in ("0", "1"):
        os.environ["HELM_APPLY_BATCH"] = mode
        ctx = Context(cfg.k, cfg.nsub, cfg.nsub)
        torch.cuda.synchronize()
        t0 = time.time()
        ctx.factor()
        torch.cuda.synchronize()
        tf = time.time() - t0
        info = ctx.factor_classes()
        v = torch.from_numpy(probe_vector(ctx.n, int(cfg.k) + 1)).cuda()
        z = torch.empty_like(v)
        for _ in range(3):
            ctx.precond_apply(v, z)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            ctx.precond_apply(v, z)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 10
        out[mode] = z.clone()
        line = f"{name} batch={mode} {info} factor {tf:.3f} s apply {ms:.3f} ms"
        if do_gmres:
            xy, amp, sigma = sources(cfg)
            b = ctx.rhs(xy, amp, sigma)
            torch.cuda.synchronize()
            e0.record()
            x, ginfo, _ = ctx.gmres(b, restart=50, rtol=1e-6)
            e1.record()
            torch.cuda.synchronize()
            line += f" gmres {ginfo.iterations} its {e0.elapsed_time(e1) / 1e3:.3f} s relres {ginfo.relres_true:.2e}"
            out[mode + "x"] = x.clone()
        print(line, flush=True)
        ctx.close()
        del ctx
        torch.cuda.empty_cache()
    d = ((out["0"] - out["1"]).norm() / out["0"].norm()).item()
    line = f"{name} apply rel diff batch vs streaming {d:.3e}"
    if do_gmres:
        line += f"; x rel diff {((out['0x'] - out['1x']).norm() / out['0x'].norm()).item():.3e}"
    print(line, flush=True)

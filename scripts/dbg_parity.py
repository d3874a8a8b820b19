"""Quick parity / timing print-out (development aid; imports the oracle, so test-side only)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from oracle.oracle import Oracle, gmres
from paper_2602_00735_b200 import Context
from paper_2602_00735_b200.workloads import CONFIGS, probe_vector, sources

for name in sys.argv[1:] or ["c0", "c1", "c2"]:
    cfg = CONFIGS[name]
    t0 = time.time()
    ctx = Context(cfg.k, cfg.nsub, cfg.nsub)
    torch.cuda.synchronize(); t1 = time.time()
    ctx.factor(); t2 = time.time()
    print(name, "setup %.3fs factor %.3fs" % (t1 - t0, t2 - t1), ctx.layout.as_dict(), flush=True)
    o = Oracle.from_config(k=cfg.k, nsub_x=cfg.nsub, nsub_y=cfg.nsub)
    A = ctx.export_stencil().cpu().numpy(); R = o.stencil().T
    print("  stencil max rel", np.max(np.abs(A - R)) / np.max(np.abs(R)), flush=True)
    v = probe_vector(o.nfree, int(cfg.k) + 1)
    y = ctx.matvec(torch.from_numpy(v).cuda()).cpu().numpy()
    print("  matvec", np.linalg.norm(y - o.matvec(v)) / np.linalg.norm(o.matvec(v)), flush=True)
    o.factor()
    z = ctx.precond_apply(torch.from_numpy(v).cuda()).cpu().numpy()
    zo = o.apply(v)
    print("  apply", np.linalg.norm(z - zo) / np.linalg.norm(zo), flush=True)
    xy, amp, sig = sources(cfg)
    b = o.rhs(xy, amp, sig)
    bg = ctx.rhs(xy, amp, sig).cpu().numpy()
    print("  rhs", np.linalg.norm(bg - b) / np.linalg.norm(b), flush=True)
    x, info, _ = ctx.gmres(torch.from_numpy(b).cuda())
    ref = gmres(o.matvec, o.apply, b)
    print("  gmres its", info.iterations, ref.iterations, "relres", info.relres_true, ref.relres_true,
          "x err", np.linalg.norm(x.cpu().numpy() - ref.x) / np.linalg.norm(ref.x), flush=True)
    # timing of apply
    r = torch.from_numpy(v).cuda(); zz = torch.empty_like(r)
    for _ in range(3): ctx.precond_apply(r, zz)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): ctx.precond_apply(r, zz)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    print("  apply %.3f ms  -> %.1f GB/s algorithmic" % (ms, ctx.layout.apply_bytes / ms / 1e6), flush=True)
    ctx.close()

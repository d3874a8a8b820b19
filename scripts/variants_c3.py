"""GMRES(50) to 1e-6 at a BJ config (argv[1], default c3) for the four local-BC / PoU variants (development aid)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2602_00735_b200 import Context  # noqa: E402
from paper_2602_00735_b200.helm import BC_DIRICHLET, BC_IMPEDANCE, POU_OWNER, POU_RAMP  # noqa: E402
from paper_2602_00735_b200.workloads import CONFIGS, sources  # noqa: E402

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3"]
for bc, pou in [(BC_DIRICHLET, POU_OWNER), (BC_IMPEDANCE, POU_OWNER), (BC_DIRICHLET, POU_RAMP), (BC_IMPEDANCE, POU_RAMP)]:
    torch.cuda.synchronize()
    t0 = time.time()
    ctx = Context(cfg.k, cfg.nsub, cfg.nsub, local_bc=bc, pou=pou)
    ctx.factor()
    torch.cuda.synchronize()
    t1 = time.time()
    b = ctx.rhs(*sources(cfg))
    torch.cuda.synchronize()
    t2 = time.time()
    x, info, _ = ctx.gmres(b, restart=cfg.restart, rtol=cfg.rtol, maxit=5000)
    torch.cuda.synchronize()
    t3 = time.time()
    print(f"bc={'imp' if bc else 'drch'} pou={'ramp' if pou else 'owner'} setup+factor {t1 - t0:.2f}s its {info.iterations} "
          f"TTS {t3 - t2:.2f}s relres {info.relres_true:.2e} apply_GB {ctx.layout.apply_bytes / 1e9:.1f}", flush=True)
    ctx.close()
    del ctx, b, x
    torch.cuda.empty_cache()

"""Observed GPU-vs-oracle agreement at full size against the oracle-only golden records (c0..c3): iteration counts,
the largest relative difference of the residual-estimate histories, and ||S (x - x_orc)|| / ||S x_orc||."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402

from golden_util import load_golden, sketch_rel  # noqa: E402
from paper_2602_00735_b200 import Context  # noqa: E402
from paper_2602_00735_b200.workloads import CONFIGS, sources  # noqa: E402

rows = []
for name in ("c0", "c1", "c2", "c3"):
    g = load_golden(name)
    cfg = CONFIGS[name]
    ctx = Context(cfg.k, cfg.nsub, cfg.nsub)
    ctx.factor()
    b = ctx.rhs(*sources(cfg))
    x, info, hist = ctx.gmres(b, restart=cfg.restart, rtol=cfg.rtol, maxit=g["maxit"], history=True)
    ho = np.asarray(g["history"])
    n = min(len(hist), len(ho))
    rows.append({"config": name, "iterations_gpu": info.iterations, "iterations_oracle": g["iterations"],
                 "history_max_rel_diff": float(np.max(np.abs(hist[:n] - ho[:n]) / ho[:n])),
                 "x_sketch_rel_diff": sketch_rel(x.cpu().numpy(), g), "relres_true_gpu": info.relres_true,
                 "relres_true_oracle": g["relres_true"]})
    ctx.close()
print(json.dumps(rows, indent=1))

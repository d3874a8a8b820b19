"""Collectives per Arnoldi step on a c3 rank grid: c3 on N loopback ranks in one process (the
multi-rank code path with NCCL replaced by device copies; timings are not meaningful here, the counts are exact),
one GMRES(50) cycle per rank, then helm_comm_counters: allreduces, halo messages and complex elements per step.

    python scripts/shard_collectives.py [N=8]
"""
import itertools
import json
import os
import sys
import threading

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2602_00735_b200 import Context  # noqa: E402
from paper_2602_00735_b200.workloads import CONFIGS, sources  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 8
GRID = {2: (2, 1), 4: (2, 2), 8: (4, 2)}[N]
cfg = CONFIGS["c3"]
kw = dict(k=cfg.k, nsub_x=cfg.nsub, nsub_y=cfg.nsub)
res = [None] * N


def rank(r):
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        c = Context(**kw, gpu_grid=GRID, rank=r, nranks=N, stream=s, loopback_group=4242)
        c.factor()
        b = c.rhs(*sources(cfg))
        c.gmres(b, restart=cfg.restart, rtol=0.0, maxit=2)            # warm-up (allocations)
        c.comm_counters(reset=True)
        _, info, _ = c.gmres(b, restart=cfg.restart, rtol=0.0, maxit=cfg.restart)
        cnt = c.comm_counters(reset=True)
        lay = c.layout
        s.synchronize()
        res[r] = {"rank": r, "iterations": info.iterations, "applies": info.applies, "counters": cnt,
                  "n_local": lay.n_local, "subdomains": lay.n_sub_local, "overlap_interior": lay.overlap_interior,
                  "comm": c.comm_info()}
        c.close()


th = [threading.Thread(target=rank, args=(r,)) for r in range(N)]
for t in th:
    t.start()
for t in th:
    t.join()
out = []
for r in res:
    st = r["applies"]
    c = r["counters"]
    out.append({**r, "per_step": {"allreduces": c["allreduces"] / st, "halo_msgs": c["msgs"] / st,
                                  "halo_recv_elems": c["recv"] / st, "halo_recv_MB": 16 * c["recv"] / st / 1e6}})
print(json.dumps({"config": "c3", "ranks": N, "grid": GRID, "cycle": "one GMRES(50) cycle, rtol 0", "per_rank": out},
                 indent=1))

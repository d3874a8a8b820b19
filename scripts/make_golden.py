"""Write tests/golden/<cfg>_gmres.json from the CPU ORACLE ONLY (no libhelm, no GPU).

    python scripts/make_golden.py c3            # full MGS GMRES(50) solve to rtol 1e-6 (~1 h on 8 cores)
    python scripts/make_golden.py c4 --maxit 100   # first two cycles of the c4 solve (status 2 = maxit)

The golden holds what the GPU must reproduce at the full size of the config (north_star: "GPU solutions
matching the oracle ... on all five configs"; GMRES P:240-242, B^-1 P:143-147):
  * iterations, restarts, status, relres_est / relres_true and the per-iteration residual-estimate history of
    right-preconditioned MGS GMRES(50) (oracle.gmres, O9) from x0 = 0;
  * ||b||, ||x|| and a seeded 64-row complex Gaussian sketch S x (S_i = workloads.probe_vector(n, SKETCH_SEED + i),
    unconjugated dot products), plus the sketch of b;
  * the oracle's own timings on this host (dedup-mode factorisation, apply median of 3, matvec, GMRES TTS) with the
    host description, keyed by the oracle source hash, for bench.py's cpu_baseline.full_oracle.
It imports only oracle/ and the seeded input generators of paper_2602_00735_b200/workloads.py (which hold no
method arithmetic).  The oracle runs in dedup mode (SURVEY 8(d) memory fallback, exact).
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import platform
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from oracle.oracle import Oracle, gmres  # noqa: E402
from paper_2602_00735_b200.workloads import CONFIGS, probe_vector, sources  # noqa: E402

SKETCH_SEED = 77_000
SKETCH_ROWS = 64


def oracle_hash() -> str:
    h = hashlib.sha256()
    for f in ("orc.c", "oracle.py"):
        with open(os.path.join(ROOT, "oracle", f), "rb") as fh:
            h.update(fh.read())
    return h.hexdigest()[:16]


def sketch(x: np.ndarray, rows: int = SKETCH_ROWS) -> np.ndarray:
    """s_i = sum_g S_ig x_g with S_i = probe_vector(n, SKETCH_SEED + i) (unconjugated)."""
    return np.array([np.dot(probe_vector(x.size, SKETCH_SEED + i), x) for i in range(rows)])


def host_info() -> dict:
    model = ""
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    ram = None
    try:
        with open("/proc/meminfo") as f:
            ram = int(f.readline().split()[1]) / 2 ** 20
    except (OSError, ValueError, IndexError):
        pass
    return {"cores": len(os.sched_getaffinity(0)), "omp_threads": int(os.environ.get("OMP_NUM_THREADS", "0")) or None,
            "cpu_model": model, "ram_GiB": ram, "machine": platform.node()}


def cz(a):
    return [[float(v.real), float(v.imag)] for v in np.asarray(a).ravel()]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("config")
    ap.add_argument("--maxit", type=int, default=5000)
    ap.add_argument("--out", default=None)
    ap.add_argument("--pou", default="owner", choices=["owner", "ramp"],
                    help="partition of unity: the owner write (D10, the hot path) or the paper's linear ramps (P:225)")
    args = ap.parse_args()
    os.environ.setdefault("OMP_NUM_THREADS", str(len(os.sched_getaffinity(0))))
    cfg = CONFIGS[args.config]
    ohash = oracle_hash()          # before the (long) run: the source the numbers come from
    pou = 1 if args.pou == "ramp" else 0
    o = Oracle.from_config(k=cfg.k, nsub_x=cfg.nsub, nsub_y=cfg.nsub, pou=pou)
    t = time.perf_counter()
    ncls = o.factor_dedup()
    factor_s = time.perf_counter() - t
    v = probe_vector(o.nfree, int(cfg.k) + 1)
    o.matvec(v)                        # first call assembles the global stencil (untimed)
    ta = []
    for _ in range(3):
        t = time.perf_counter()
        o.apply(v)
        ta.append(time.perf_counter() - t)
    t = time.perf_counter()
    o.matvec(v)
    matvec_s = time.perf_counter() - t
    b = o.rhs(*sources(cfg))
    hist_t = []

    def A(x):
        return o.matvec(x)

    def M(x):
        z = o.apply(x)
        hist_t.append(time.perf_counter())
        if len(hist_t) % 10 == 0:
            print(f"[{args.config}] apply {len(hist_t)}", flush=True)
        return z

    t = time.perf_counter()
    res = gmres(A, M, b, restart=cfg.restart, rtol=cfg.rtol, maxit=args.maxit)
    tts = time.perf_counter() - t
    out = {
        "config": cfg.name, "k": cfg.k, "nsub": cfg.nsub, "seed": cfg.seed, "nsrc": cfg.nsrc, "n_free": o.nfree,
        "restart": cfg.restart, "rtol": cfg.rtol, "maxit": args.maxit, "x0": "zero", "pou": args.pou,
        "solver": "oracle.gmres: right-preconditioned GMRES(50), MGS, Hermitian inner products (O9, P:240-242)",
        "iterations": res.iterations, "restarts": res.restarts, "status": res.status,
        "relres_est": res.relres_est, "relres_true": res.relres_true, "history": [float(h) for h in res.history],
        "norm_b": float(np.linalg.norm(b)), "norm_x": float(np.linalg.norm(res.x)),
        "sketch_seed": SKETCH_SEED, "sketch_rows": SKETCH_ROWS,
        "sketch_x": cz(sketch(res.x)), "sketch_b": cz(sketch(b)),
        "oracle_hash": ohash,
        "oracle_timing": {"factor_dedup_s": factor_s, "classes": ncls, "apply_s_median3": statistics.median(ta),
                          "matvec_s": matvec_s, "gmres_s": tts, "gmres_applies": len(hist_t),
                          "host": host_info(), "when": time.strftime("%Y-%m-%dT%H:%M:%SZ", time.gmtime())},
        "written_by": "scripts/make_golden.py (imports oracle/ and workloads only)",
    }
    suffix = "" if args.pou == "owner" else "_ramp"
    path = args.out or os.path.join(ROOT, "tests", "golden", f"{cfg.name}{suffix}_gmres.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print(json.dumps({k: out[k] for k in ("config", "iterations", "restarts", "status", "relres_true", "norm_x")}))
    print("oracle_timing", json.dumps(out["oracle_timing"]))


if __name__ == "__main__":
    main()

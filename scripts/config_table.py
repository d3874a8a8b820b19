"""SURVEY 8(d) "Reporting" for the BASELINE.json configs on one GPU.  Per config: setup and factorisation time, apply
time (median of 20 after 3 warm-ups) as applies/s, algorithmic and band-equivalent GB/s against the measured copy
peak, SpMV, GMRES(50) to 1e-6 (iterations, restarts, time) and its roofline fraction.  Prints a markdown table
(profiles/r01_configs.md).  The oracle's timings beside it come from bench.py's cpu_baseline leg
(`python bench.py --config cX`, key cpu_baseline.full_oracle): only tests/, smoke() and that leg run the oracle.

    python scripts/config_table.py c0 c1 c2 c3
"""
import json
import os
import statistics
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2602_00735_b200 import Context  # noqa: E402
from paper_2602_00735_b200.workloads import CONFIGS, probe_vector, sources  # noqa: E402

PEAK = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]


def median_ms(fn, reps=20, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


def gpu_row(name):
    cfg = CONFIGS[name]
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    ctx = Context(cfg.k, cfg.nsub, cfg.nsub)
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    ctx.factor()
    t2 = time.perf_counter()
    L = ctx.layout
    v = torch.from_numpy(probe_vector(ctx.n, int(cfg.k) + 1)).cuda()
    z = torch.empty_like(v)
    ap = median_ms(lambda: ctx.precond_apply(v, z))
    sp = median_ms(lambda: ctx.matvec(v, z))
    b = ctx.rhs(*sources(cfg))
    ctx.gmres(b, restart=cfg.restart, rtol=cfg.rtol, maxit=1)   # untimed: allocates the Krylov workspace
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    _, info, _ = ctx.gmres(b, restart=cfg.restart, rtol=cfg.rtol, maxit=5000)
    e1.record()
    torch.cuda.synchronize()
    tts = e0.elapsed_time(e1) / 1e3
    # TTS at the roofline: the same byte model as bench.py (DCGS2), every byte at the measured copy peak
    n16, m = 16 * ctx.n, cfg.restart
    tot, left = 0, info.iterations
    for _ in range(info.restarts + 1):
        mm = min(m, left)
        for j in range(mm):
            tot += L.apply_bytes + L.spmv_bytes + n16 * (2 * (j + 1) + 4)
        tot += n16 * (2 + 2 * (mm + 1)) + L.apply_bytes + 4 * n16 + L.spmv_bytes
        left -= mm
    row = dict(cfg=name, unknowns=ctx.n, subdomains=cfg.nsub ** 2, factor_GB=L.factor_bytes / 1e9,
               setup_s=t1 - t0, factor_s=t2 - t1, apply_ms=ap, applies_per_s=1e3 / ap,
               GBps=L.apply_bytes / ap / 1e6, band_GBps=L.band_bytes / ap / 1e6, spmv_ms=sp,
               its=info.iterations, restarts=info.restarts, relres=info.relres_true, tts_s=tts,
               tts_roofline_frac=tot / (PEAK * 1e9) / tts)
    ctx.close()
    del ctx, v, z, b
    torch.cuda.empty_cache()
    return row


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    names = args or ["c0", "c1", "c2", "c3"]
    print(f"1 x {torch.cuda.get_device_name()}; copy peak {PEAK} GB/s (MEASURED_PEAKS.json)\n")
    w = Context(CONFIGS["c0"].k, CONFIGS["c0"].nsub, CONFIGS["c0"].nsub)   # untimed: CUDA context and module loading
    w.factor()
    w.close()
    print("| cfg | unknowns | subdomains | factors GB | setup s | factor s | apply ms | applies/s | GB/s (frac) | "
          "band-equiv. GB/s | SpMV ms | GMRES its / restarts | TTS s | TTS roofline frac |")
    print("|---|---|---|---|---|---|---|---|---|---|---|---|---|---|")
    for name in names:
        r = gpu_row(name)
        print(f"| {name} | {r['unknowns']:,} | {r['subdomains']} | {r['factor_GB']:.2f} | {r['setup_s']:.3f} | "
              f"{r['factor_s']:.3f} | {r['apply_ms']:.3f} | {r['applies_per_s']:.1f} | {r['GBps']:.0f} "
              f"({r['GBps'] / PEAK:.2f}) | {r['band_GBps']:.0f} | {r['spmv_ms']:.3f} | {r['its']} / {r['restarts']} | "
              f"{r['tts_s']:.3f} | {r['tts_roofline_frac']:.2f} |", flush=True)


if __name__ == "__main__":
    main()

"""bench.py -- RAS-PML hot path on B200 (driver contract: one JSON line on rank 0).

A step is one right-preconditioned GMRES(50) Arnoldi iteration over the whole hot path:
RAS-PML apply (restrict -> twisted block-tridiagonal local solves -> owner write), 7-point SpMV, CGS2
orthogonalisation with the re-orthogonalisation delayed one step (DCGS2: two sweeps over the basis per step), Givens
update on the host.  `value` = RAS-PML preconditioner applications per second over exactly K steps (one per
Arnoldi step; a cycle's solution update reuses the steps' applies, so the timed region's cycle ends add only their
vector work), all inputs resident in HBM.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3] [--impl ours|reference]

--impl reference times the CPU oracle (the only reference this paper has) on the box's host cores, on the
same config / metric / unit, each step a bounded sample of the workload.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

METRIC = "RAS-PML applies/s inside right-preconditioned GMRES(50) (1 apply + SpMV + CGS2 per Arnoldi step)"
UNIT = "applies/s"


def workload_desc(cfg, lay=None):
    d = {"workload": f"{cfg.name}: k={cfg.k:g}, {cfg.nsub}x{cfg.nsub} subdomains, P1 10 ppw, GMRES({cfg.restart}), "
                     f"seeded synthetic inputs (BASELINE.json configs[{list('01234').index(cfg.name[1])}])",
         "k": cfg.k, "subdomains": cfg.nsub * cfg.nsub, "restart": cfg.restart, "nsrc": cfg.nsrc, "seed": cfg.seed}
    if lay is not None:
        d.update({"n_free": lay["n_free_global"], "cells_per_side": lay["N_cells"], "delta": lay["n_ovlp"],
                  "kappa": lay["n_pml"], "local_unknowns": lay["local_unknowns"], "m_max": lay["m_max"],
                  "factor_GB": round(lay["factor_bytes"] / 1e9, 3)})
    return d


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            j = json.load(f)
        return float(j["hbm_gbs"]), "measured copy bandwidth, MEASURED_PEAKS.json"
    return 6650.0, "fallback (B200_PROFILING.md)"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()
            self.th.join(timeout=2)

    def summary(self):
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            try:
                sm.append(float(r[0]))
                mx.append(float(r[1]))
            except (ValueError, IndexError):
                continue
            for n, v in zip(names, r[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"], "samples": 0}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": max(mx), "reasons": sorted(reasons),
                "samples": len(sm)}


# ====================================================================================== our arm
def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2602_00735_b200 import Context
    from paper_2602_00735_b200.workloads import CONFIGS, sources

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl")
    cfg = CONFIGS[args.config]
    if args.seed is not None:   # another draw of the same workload (sources; the probe vectors keep k + 1)
        import dataclasses
        cfg = dataclasses.replace(cfg, seed=args.seed)
    # a dedicated (non-default) stream for the library and everything timed around it; torch work issued below
    # (inputs, events, the barrier's NCCL collectives) is ordered on it as the current stream
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    nccl_id = None
    if world > 1:
        # libhelm owns its NCCL communicator; rank 0 makes the id, torch.distributed only broadcasts it
        from paper_2602_00735_b200.helm import nccl_unique_id
        buf = torch.zeros(128, dtype=torch.uint8, device="cuda")
        if rank == 0:
            buf.copy_(torch.frombuffer(bytearray(nccl_unique_id()), dtype=torch.uint8))
        dist.broadcast(buf, src=0)
        nccl_id = bytes(buf.cpu().numpy().tobytes())

    t0 = time.time()
    ctx = Context(cfg.k, cfg.nsub, cfg.nsub, rank=rank, nranks=world, stream=stream, nccl_id=nccl_id)
    ctx.factor()
    if args.orth == "cgs2":
        from paper_2602_00735_b200.helm import ORTH_CGS2
        ctx.set_orthogonalisation(ORTH_CGS2)
    torch.cuda.synchronize()
    setup_s = time.time() - t0
    lay = ctx.layout.as_dict()
    xy, amp, sig = sources(cfg)
    b = ctx.rhs(xy, amp, sig)

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # ---- warm-up: W Arnoldi steps
    x = torch.zeros_like(b)
    ctx.gmres(b, x, restart=cfg.restart, rtol=0.0, maxit=max(args.warmup, 1))
    # ---- timed: exactly K Arnoldi steps in one GMRES(50) call (rtol = 0: no early exit)
    x.zero_()
    ctx.profile(True)
    ctx.profile_read()
    barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        ev0.record(stream)
        _, info, _ = ctx.gmres(b, x, restart=cfg.restart, rtol=0.0, maxit=args.steps)
        ev1.record(stream)
        barrier()
    ms = ev0.elapsed_time(ev1)
    apply_ms, apply_n, launches = ctx.profile_read()
    ctx.profile(False)
    if world > 1:
        t = torch.tensor([ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    applies = info.applies
    value = applies / (ms / 1e3)

    # ---- apply-only and SpMV-only rates (reported alongside; not the headline)
    v = torch.randn(ctx.n, dtype=torch.complex128, device="cuda")
    z = torch.empty_like(v)
    for _ in range(3):
        ctx.precond_apply(v, z)
    barrier()
    ev0.record(stream)
    for _ in range(10):
        ctx.precond_apply(v, z)
    ev1.record(stream)
    barrier()
    apply_only_ms = ev0.elapsed_time(ev1) / 10

    # ---- time to solution (rtol 1e-6), inputs resident
    x.zero_()
    barrier()
    ev0.record(stream)
    _, tinfo, _ = ctx.gmres(b, x, restart=cfg.restart, rtol=cfg.rtol, maxit=5000)
    ev1.record(stream)
    barrier()
    tts_s = ev0.elapsed_time(ev1) / 1e3

    # ---- end to end through the C ABI with host buffers (pinned), K steps, copies inside
    bh = b.cpu().pin_memory()
    xh = torch.zeros_like(bh).pin_memory()
    ctx.gmres_host(bh.numpy(), xh.numpy(), restart=cfg.restart, rtol=0.0, maxit=max(args.warmup, 1))   # warm-up
    xh.zero_()
    barrier()
    t1 = time.perf_counter()
    _, einfo = ctx.gmres_host(bh.numpy(), xh.numpy(), restart=cfg.restart, rtol=0.0, maxit=args.steps)
    barrier()
    e2e_s = time.perf_counter() - t1
    n = ctx.n
    cycles = einfo.restarts + 1
    h2d = 16 * n * 2 + 16 * args.steps                        # b, x0; y coefficients
    if args.orth == "cgs2":
        h2d += 8 * cycles                                       # per-cycle beta
    if args.orth == "cgs2":   # one Hessenberg column per step
        d2h = 16 * n + sum(16 * (min(j % cfg.restart, cfg.restart - 1) + 2) for j in range(args.steps)) + 8 * (cycles + 1)
    else:   # DCGS2: the step record (3 x 64 + 2 complex) per step, the closed column per cycle
        d2h = 16 * n + 16 * 194 * args.steps + 16 * (cfg.restart + 1) * cycles + 8 * (cycles + 1)

    hbm, peak_src = peaks()

    # TTS roofline: bytes the solve must move at the kernels' algorithmic rates (tts_bytes below).
    def tts_bytes(its, restarts):
        """Algorithmic bytes of the whole solve: per Arnoldi step the apply, the SpMV and the orthogonalisation
        sweeps (DCGS2: projection sweep over V_{j+1} and w, update sweep reading V_j, u_j, w and writing v_j,
        u_{j+1}; CGS2: three sweeps over V_{j+1} plus w traffic); per cycle u_0 = r, then for DCGS2 the closing
        projection and x += Z (R^-1 y) (no apply), for CGS2 the combination V y, one apply and x += z; then the
        true residual."""
        n16 = 16 * ctx.n
        cgs2 = args.orth == "cgs2"
        tot, left = 0, its
        for _ in range(restarts + 1):
            m = min(cfg.restart, left)
            for j in range(m):
                orth = 3 * (j + 1) + 7 if cgs2 else 2 * (j + 1) + 4
                tot += lay["apply_bytes"] + lay["spmv_bytes"] + n16 * orth
            if cgs2:   # x += B^-1 (V y): combine, one apply, axpy; then the true residual
                tot += n16 * (2 + m + 1) + lay["apply_bytes"] + 3 * n16 + lay["spmv_bytes"] + n16
            else:      # closing projection, x += Z (R^-1 y): combine + axpy (no apply); then the true residual
                tot += n16 * (2 + (m + 1) + (m + 1)) + 3 * n16 + lay["spmv_bytes"] + n16
            left -= m
        return tot

    tts_b = tts_bytes(tinfo.iterations, tinfo.restarts)
    apply_avg_ms = apply_ms / max(apply_n, 1)
    achieved = lay["apply_bytes"] / (apply_avg_ms / 1e3) / 1e9
    from paper_2602_00735_b200.helm import probe_read_bandwidth
    read_peak = probe_read_bandwidth(8 << 30, 5, 0)          # chunks interleaved over the CTAs
    read_streams = probe_read_bandwidth(16 << 30, 5, 1)      # one contiguous stream per CTA, like k_apply
    traffic = None
    prof = os.path.join(ROOT, "profiles", "k_apply_traffic.json")
    if os.path.exists(prof) and world == 1:
        with open(prof) as f:
            tj = json.load(f)
        traffic = tj.get(cfg.name, {}).get("dram_bytes_per_launch")

    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": {**workload_desc(cfg, lay), "parallelism": f"subdomain-sharded x{world}", "orth": args.orth,
                   "l2": "inputs larger than L2: %.1f GB of factor blocks streamed per apply vs 126 MB L2"
                         % (lay["apply_bytes"] / 1e9)},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                     "traffic": traffic, "kernel": "k_apply (fused restrict + twisted block solves + owner write)",
                     "algorithmic_bytes_per_launch": lay["apply_bytes"], "peak_source": peak_src,
                     "band_equivalent_GBps": lay["band_bytes"] / (apply_avg_ms / 1e3) / 1e9,
                     "read_stream_probe_GBps": read_peak, "frac_of_read_probe": achieved / read_peak,
                     "read_streams_probe_GBps": read_streams, "frac_of_read_streams_probe": achieved / read_streams,
                     "apply_kernel_ms": apply_avg_ms, "apply_share_of_step": apply_ms / ms},
        "e2e": {"value": applies_e2e(einfo, e2e_s), "unit": UNIT, "h2d_bytes_per_step": h2d / args.steps,
                "d2h_bytes_per_step": d2h / args.steps, "api": "helm_gmres_host (host b/x, copies inside)"},
        "gpu_launches": launches,
        "applies": applies, "iterations": info.iterations,
        "apply_only": {"ms": apply_only_ms, "applies_per_s": 1e3 / apply_only_ms,
                       "GBps": lay["apply_bytes"] / apply_only_ms / 1e6},
        "gmres_tts": {"seconds": tts_s, "iterations": tinfo.iterations, "restarts": tinfo.restarts,
                      "relres_true": tinfo.relres_true, "status": tinfo.status, "rtol": cfg.rtol,
                      "algorithmic_bytes": tts_b, "roofline_s": tts_b / (hbm * 1e9),
                      "roofline_frac": tts_b / (hbm * 1e9) / tts_s},
        "setup_factor_s": setup_s,
        "clocks": clk.summary(),
    }
    if world == 1 and not args.no_paper:
        out["paper_table4"] = paper_table4(stream)
        out["gmres_tts_ramp_pou"] = ramp_pou_tts(cfg, stream, xy, amp, sig)
    if rank == 0 and args.gpus == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(cfg, steps=1)
    if rank == 0:
        print(json.dumps(out), flush=True)
    ctx.close()
    if world > 1:
        dist.destroy_process_group()


# The paper's timed runs (Table 4: RAS-PML-Imp Richardson to rtol 1e-10, one processor per subdomain;
# the paper names no hardware).  Context only: another machine, another discretisation code.
PAPER_TABLE4 = {"t300": {"k": 300, "procs": 4, "iter": 7, "setup_s": 0.95, "solve_s": 0.27, "line": 322},
                "t600": {"k": 600, "procs": 16, "iter": 14, "setup_s": 1.12, "solve_s": 0.68, "line": 323},
                "t1200": {"k": 1200, "procs": 64, "iter": 31, "setup_s": 1.40, "solve_s": 1.87, "line": 324}}


def paper_table4(stream, names=("t300", "t600")):
    """The paper's own workload end to end on this GPU: setup (assembly) + factorisation, then Algorithm 1 to 1e-10
    from u = 0, each timed with CUDA events on the library stream."""
    import torch

    from paper_2602_00735_b200 import Context
    from paper_2602_00735_b200.helm import paper_params
    from paper_2602_00735_b200.workloads import PAPER_CONFIGS, paper_source

    # untimed warm-up on a small paper-type problem: the Q1 assembly, cluster factorisation and cluster-split apply
    # kernels are loaded lazily by the CUDA runtime on first launch
    for kw, nsw in ((60.0, 2), (100.0, 1)):   # m < 112 (shared-memory factorisation) and m > 112 (clusters)
        w = Context(**paper_params(kw, nsw, 4, 2), stream=stream)
        w.factor()
        w.richardson(w.rhs(*paper_source(kw)), rtol=1e-6, maxit=3)
        w.close()
    rows = []
    for name in names:
        c = PAPER_CONFIGS[name]
        best = None
        for _ in range(2):   # best of two: these runs last 0.1-0.3 s, where clock ramp-up and allocator noise show
            torch.cuda.synchronize()
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
            ev[0].record(stream)
            ctx = Context(**paper_params(c.k, c.nsub, c.pml, c.ovlp, n_cells=c.n_cells, local_bc=c.local_bc),
                          stream=stream)
            ctx.factor()
            ev[1].record(stream)
            xy, amp, s = paper_source(c.k)
            b = ctx.rhs(xy, amp, s)
            ev[2].record(stream)
            _, info, _ = ctx.richardson(b, rtol=c.rtol, maxit=c.maxit)
            ev[3].record(stream)
            torch.cuda.synchronize()
            lay = ctx.layout
            row = {"config": name, "k": c.k, "grid": c.n_cells, "subdomains": c.nsub ** 2, "pml": c.pml,
                   "ovlp": c.ovlp, "m_max": lay.m_max, "factor_GB": round(lay.factor_bytes / 1e9, 2),
                   "setup_factor_s": ev[0].elapsed_time(ev[1]) / 1e3, "solve_s": ev[2].elapsed_time(ev[3]) / 1e3,
                   "iterations": info.iterations, "relres": info.relres, "timing": "best of 2 runs",
                   "paper": PAPER_TABLE4[name]}
            if best is None or row["setup_factor_s"] + row["solve_s"] < best["setup_factor_s"] + best["solve_s"]:
                best = row
            ctx.close()
            del ctx, b
            torch.cuda.empty_cache()
        rows.append(best)
    return rows


def ramp_pou_tts(cfg, stream, xy, amp, sig):
    """The same GMRES(50) solve with the paper's linear-ramp partition of unity instead of the north_star's
    owner write: reported beside the headline, not as it (one rank only)."""
    import torch

    from paper_2602_00735_b200 import Context
    from paper_2602_00735_b200.helm import POU_RAMP

    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    ev[0].record(stream)
    ctx = Context(cfg.k, cfg.nsub, cfg.nsub, pou=POU_RAMP, stream=stream)
    ctx.factor()
    ev[1].record(stream)
    b = ctx.rhs(xy, amp, sig)
    ev[2].record(stream)
    _, info, _ = ctx.gmres(b, restart=cfg.restart, rtol=cfg.rtol, maxit=5000)
    ev[3].record(stream)
    torch.cuda.synchronize()
    res = {"setup_factor_s": ev[0].elapsed_time(ev[1]) / 1e3, "seconds": ev[2].elapsed_time(ev[3]) / 1e3,
           "iterations": info.iterations, "restarts": info.restarts, "relres_true": info.relres_true,
           "apply_bytes": ctx.layout.apply_bytes}
    ctx.close()
    del ctx, b
    torch.cuda.empty_cache()
    return res


def applies_e2e(info, seconds):
    return info.applies / seconds if seconds > 0 else None


# ====================================================================================== oracle arm
def _oracle_step_model(cfg):
    """Set up the oracle on this config and return a callable timing one bounded-sample step."""
    import numpy as np

    from oracle.oracle import Oracle
    from paper_2602_00735_b200.workloads import probe_vector

    o = Oracle.from_config(k=cfg.k, nsub_x=cfg.nsub, nsub_y=cfg.nsub)
    # stratified sample of subdomains: interior, edge and corner classes, at most 48
    P = cfg.nsub
    cand = sorted({0, P - 1, P * (P - 1), P * P - 1, 1, P, P * (P // 2) + P // 2, P * (P // 3) + (2 * P) // 3})
    rng = np.random.default_rng(cfg.seed)
    extra = rng.choice(P * P, size=min(48, P * P), replace=False).tolist()
    sample = sorted(set(cand + extra))[:48] if P * P > 48 else list(range(P * P))

    def cost(j):
        s = o.subdomain(j)
        mx, my = s["m"]
        return mx * my * (mx + 1)          # band solve work ~ n * p

    total = sum(cost(j) for j in range(o.nsub)) if o.nsub <= 20000 else None
    scale = total / sum(cost(j) for j in sample)
    t = time.perf_counter()
    o.factor(sample)
    factor_s = time.perf_counter() - t
    v = probe_vector(o.nfree, int(cfg.k) + 1)
    V = [v / np.linalg.norm(v)]
    jdepth = cfg.restart // 2            # a cycle orthogonalises against ~restart/2 vectors on average
    jsample = min(4, jdepth)             # time MGS against 4 of them, scale linearly
    for i in range(jsample - 1):
        w = probe_vector(o.nfree, 1000 + i)
        V.append(w / np.linalg.norm(w))

    def step():
        t0 = time.perf_counter()
        z = o.apply(V[0], subs=sample)
        t1 = time.perf_counter()
        w = o.matvec(z)
        t2 = time.perf_counter()
        for i in range(len(V)):               # MGS (O9)
            h = np.vdot(V[i], w)
            w = w - h * V[i]
        np.linalg.norm(w)
        t3 = time.perf_counter()
        return (t1 - t0) * scale + (t2 - t1) + (t3 - t2) * jdepth / jsample

    desc = (f"oracle GMRES step on {cfg.name}: band-LU RAS apply on {len(sample)} of {o.nsub} subdomains "
            f"(scaled by band work x{scale:.1f}) + full matvec + MGS against {jsample} vectors scaled to {jdepth}; "
            f"sample factor time {factor_s:.1f}s untimed")
    return step, desc


def cpu_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def cpu_baseline(cfg, steps=1):
    os.environ.setdefault("OMP_NUM_THREADS", str(cpu_threads()))
    step, desc = _oracle_step_model(cfg)
    ts = [step() for _ in range(max(1, steps))]
    per = sum(ts) / len(ts)
    out = {"value": 1.0 / per, "unit": UNIT, "cores": int(os.environ["OMP_NUM_THREADS"]), "kind": "oracle",
           "sample": desc, "seconds_per_step": per}
    if cfg.name in ("c0", "c1", "c2"):   # small enough to time the whole oracle solve (SURVEY 8(d) reporting)
        out["full_oracle"] = _oracle_full(cfg)
    return out


def _oracle_full(cfg):
    """The oracle on the whole workload: band-LU factorisation, apply (median of 3), MGS GMRES(50) to rtol."""
    import statistics

    from oracle.oracle import Oracle, gmres
    from paper_2602_00735_b200.workloads import probe_vector, sources
    o = Oracle.from_config(k=cfg.k, nsub_x=cfg.nsub, nsub_y=cfg.nsub)
    t = time.perf_counter()
    o.factor()
    fs = time.perf_counter() - t
    v = probe_vector(o.nfree, int(cfg.k) + 1)
    ts = []
    for _ in range(3):
        t = time.perf_counter()
        o.apply(v)
        ts.append(time.perf_counter() - t)
    b = o.rhs(*sources(cfg))
    t = time.perf_counter()
    res = gmres(o.matvec, o.apply, b, restart=cfg.restart, rtol=cfg.rtol)
    tts = time.perf_counter() - t
    o.close()
    return {"factor_s": fs, "apply_s": statistics.median(ts), "gmres_iterations": res.iterations, "gmres_s": tts}


def run_reference(args):
    from paper_2602_00735_b200.workloads import CONFIGS
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    os.environ.setdefault("OMP_NUM_THREADS", str(cpu_threads()))
    cfg = CONFIGS[args.config]
    if args.seed is not None:   # another draw of the same workload (sources; the probe vectors keep k + 1)
        import dataclasses
        cfg = dataclasses.replace(cfg, seed=args.seed)
    step, desc = _oracle_step_model(cfg)
    for _ in range(args.warmup):
        step()
    ts = [step() for _ in range(args.steps)]
    total = sum(ts)
    value = args.steps / total
    out = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
           "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": workload_desc(cfg),
           "cpu_baseline": {"value": value, "unit": UNIT, "cores": int(os.environ["OMP_NUM_THREADS"]),
                            "kind": "oracle", "sample": desc},
           "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=100)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="c3")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-paper", action="store_true", help="skip the paper Table 4 comparison rows")
    ap.add_argument("--seed", type=int, default=None, help="source draw seed (default: the config's, = k)")
    ap.add_argument("--orth", default="dcgs2", choices=["dcgs2", "cgs2"],
                    help="GMRES orthogonalisation (DESIGN.md 5.6); cgs2 = the undelayed form, for A/B")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()

"""bench.py -- RAS-PML hot path on B200 (driver contract: one JSON line on rank 0).

A step is one whole right-preconditioned GMRES(50) restart cycle over the hot path: 50 Arnoldi
iterations, each one RAS-PML apply (restrict -> twisted block-tridiagonal local solves -> owner write), one 7-point
SpMV and CGS2 orthogonalisation with the re-orthogonalisation delayed one step (DCGS2), Givens updates on the host,
then the cycle end (closing projection, x += Z R^-1 y, true residual).  `value` = RAS-PML preconditioner applications
(= Arnoldi iterations) per second over exactly K cycles, all inputs resident in HBM: a whole cycle, so the Krylov
depth averages over 0..49 exactly as in a real solve (time to solution = cycles x cycle time).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config c3] [--impl ours|reference]

--gpus N > 1 without torchrun's environment re-launches itself under torch.distributed.run (one rank per GPU).
--impl reference times the CPU oracle (the only reference this paper has) on the box's host cores, on the same
config / metric / unit: each step one full-size oracle Arnoldi step (apply over every subdomain, matvec, MGS) at
depths spread evenly over a GMRES(50) cycle.
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
STEP_DESC = ("one GMRES(50) restart cycle: 50 Arnoldi steps (RAS-PML apply + SpMV + orthogonalisation) + cycle end; "
             "value = Arnoldi steps (one apply each) per second")


def workload_desc(cfg, world: int):
    """The workload, identical in both arms (no implementation or layout keys)."""
    return {"workload": f"{cfg.name}: k={cfg.k:g}, {cfg.nsub}x{cfg.nsub} subdomains, P1 10 ppw, GMRES({cfg.restart}), "
                        f"seeded synthetic inputs (BASELINE.json configs[{list('01234').index(cfg.name[1])}])",
            "k": cfg.k, "subdomains": cfg.nsub * cfg.nsub, "restart": cfg.restart, "nsrc": cfg.nsrc, "seed": cfg.seed,
            "rtol": cfg.rtol, "step": STEP_DESC, "parallelism": f"subdomain-sharded x{world}",
            "l2": "inputs larger than L2: every apply streams all factor blocks (GBs at c2-c4) vs the 126 MB L2"}


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


def nccl_init_lines(path_glob):
    """NCCL INIT lines of this job (NCCL_DEBUG=INFO, NCCL_DEBUG_SUBSYS=INIT written to per-process files)."""
    import glob
    out = []
    for f in sorted(glob.glob(path_glob)):
        try:
            with open(f) as fh:
                for line in fh:
                    if "Init COMPLETE" in line or "NVLS" in line or "nranks" in line:
                        out.append(line.strip()[-200:])
        except OSError:
            pass
    return out[:64]


# ====================================================================================== our arm
def run_ours(args):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    # NCCL's own record of the communicators (rank 0 reports the INIT lines: N ranks, NVLS or not)
    tag = os.environ.get("TORCHELASTIC_RUN_ID", str(os.getppid()))
    nccl_log = f"/tmp/helm_nccl_{tag}"
    if world > 1:
        os.environ.setdefault("NCCL_DEBUG", "INFO")
        os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
        os.environ.setdefault("NCCL_DEBUG_FILE", nccl_log + ".%h.%p.log")

    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2602_00735_b200 import Context
    from paper_2602_00735_b200.workloads import CONFIGS, sources

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

    def barrier():
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    def max_over_ranks(v: float) -> float:
        if world == 1:
            return v
        t = torch.tensor([v], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def gather(v: float) -> list:
        if world == 1:
            return [v]
        t = torch.zeros(world, device="cuda", dtype=torch.float64)
        t[rank] = v
        dist.all_reduce(t)
        return t.cpu().tolist()

    # untimed warm-up of the setup kernels on a small problem (lazy module loading, clocks ramping up from idle)
    wctx = Context(100.0, 4, 4, stream=stream)
    wctx.factor()
    wctx.close()
    del wctx
    barrier()
    t0 = time.time()
    ctx = Context(cfg.k, cfg.nsub, cfg.nsub, rank=rank, nranks=world, stream=stream, nccl_id=nccl_id)
    fe0, fe1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fe0.record(stream)
    ctx.factor()
    fe1.record(stream)
    if args.orth == "cgs2":
        from paper_2602_00735_b200.helm import ORTH_CGS2
        ctx.set_orthogonalisation(ORTH_CGS2)
    torch.cuda.synchronize()
    setup_s = max_over_ranks(time.time() - t0)
    factor_s = max_over_ranks(fe0.elapsed_time(fe1) / 1e3)
    lay = ctx.layout.as_dict()
    fcls = ctx.factor_classes()
    comm = ctx.comm_info()
    xy, amp, sig = sources(cfg)
    b = ctx.rhs(xy, amp, sig)
    x = torch.zeros_like(b)
    R = cfg.restart

    def cycles(k):
        its = 0
        for _ in range(k):
            x.zero_()
            _, inf, _ = ctx.gmres(b, x, restart=R, rtol=0.0, maxit=R)
            its += inf.iterations
        return its

    # ---- warm-up: W cycles; timed: exactly K cycles (rtol = 0: no early exit), CUDA events on the library stream
    cycles(args.warmup)
    ctx.profile(True)
    ctx.profile_read()
    barrier()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        ev0.record(stream)
        its = cycles(args.steps)
        ev1.record(stream)
        barrier()
    ms = max_over_ranks(ev0.elapsed_time(ev1))
    apply_ms, apply_n, launches = ctx.profile_read()
    ctx.profile(False)
    value = its / (ms / 1e3)

    # ---- apply-only rate (reported alongside; not the headline)
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
    apply_only_ms = max_over_ranks(ev0.elapsed_time(ev1) / 10)

    # ---- time to solution (rtol 1e-6), inputs resident
    x.zero_()
    barrier()
    ev0.record(stream)
    _, tinfo, _ = ctx.gmres(b, x, restart=R, rtol=cfg.rtol, maxit=5000)
    ev1.record(stream)
    barrier()
    tts_s = max_over_ranks(ev0.elapsed_time(ev1) / 1e3)

    # ---- end to end through the C ABI with host buffers (pinned), K cycles, copies inside every call
    bh = b.cpu().pin_memory()
    xh = torch.zeros_like(bh).pin_memory()
    xh_np = xh.numpy()
    for _ in range(max(1, min(args.warmup, 2))):
        xh.zero_()
        ctx.gmres_host(bh.numpy(), xh_np, restart=R, rtol=0.0, maxit=R)   # warm-up (staging buffers on first use)
    barrier()
    t1 = time.perf_counter()
    e_its = 0
    for _ in range(args.steps):
        xh.zero_()
        _, einfo = ctx.gmres_host(bh.numpy(), xh_np, restart=R, rtol=0.0, maxit=R)
        e_its += einfo.iterations
    barrier()
    e2e_s = max_over_ranks(time.perf_counter() - t1)
    n = ctx.n
    h2d = 16 * n * 2 + 16 * R                                 # b, x0; the cycle's y coefficients
    if args.orth == "cgs2":
        h2d += 8
        d2h = 16 * n + sum(16 * (j + 2) for j in range(R)) + 8 * 2
    else:   # DCGS2: the step record (3 x 64 + 2 complex) per step, the closed column, the norms
        d2h = 16 * n + 16 * 194 * R + 16 * (R + 1) + 8 * 2

    hbm, peak_src = peaks()

    def tts_cost(its, restarts):
        """(algorithmic bytes, roofline seconds) of a solve.  The vector work (SpMV, orthogonalisation, cycle ends)
        is HBM-bound: its bytes at the HBM peak.  The apply: with per-subdomain factors its bytes at the HBM peak too;
        with the tensor-core apply (D28) its algorithmic flops at the measured DMMA peak."""
        tot = tts_bytes(its, restarts)
        if not fcls["batched"]:
            return tot, tot / (hbm * 1e9)
        vec = tot - its * lay["apply_bytes"]
        return vec, vec / (hbm * 1e9) + its * fcls["apply_flop"] / (dmma_peak * 1e12)

    def tts_bytes(its, restarts):
        """Algorithmic bytes of a solve: per Arnoldi step the apply, the SpMV and the orthogonalisation sweeps
        (DCGS2: projection sweep over V_{j+1} and w, update sweep reading V_j, u_j, w and writing v_j, u_{j+1};
        CGS2: three sweeps over V_{j+1} plus w traffic); per cycle u_0 = r, then for DCGS2 the closing projection and
        x += Z (R^-1 y) (no apply), for CGS2 the combination V y, one apply and x += z; then the true residual."""
        n16 = 16 * ctx.n
        cgs2 = args.orth == "cgs2"
        tot, left = 0, its
        for _ in range(restarts + 1):
            m = min(R, left)
            for j in range(m):
                orth = 3 * (j + 1) + 7 if cgs2 else 2 * (j + 1) + 4
                tot += lay["apply_bytes"] + lay["spmv_bytes"] + n16 * orth
            if cgs2:
                tot += n16 * (2 + m + 1) + lay["apply_bytes"] + 3 * n16 + lay["spmv_bytes"] + n16
            else:
                tot += n16 * (2 + (m + 1) + (m + 1)) + 3 * n16 + lay["spmv_bytes"] + n16
            left -= m
        return tot

    from paper_2602_00735_b200.helm import probe_fp64_tflops
    dmma_peak = probe_fp64_tflops(0)
    tts_b, tts_roof_s = tts_cost(tinfo.iterations, tinfo.restarts)
    cyc_b = tts_bytes(R, 0)
    apply_avg_ms = apply_ms / max(apply_n, 1)
    # per GPU: this rank's algorithmic apply bytes over its own mean apply time; the line reports the slowest rank
    ach_r = gather(lay["apply_bytes"] / (apply_avg_ms / 1e3) / 1e9)
    ms_r = gather(apply_avg_ms)
    slow = max(range(world), key=lambda q: ms_r[q])
    achieved = ach_r[slow]
    from paper_2602_00735_b200.helm import probe_read_bandwidth
    read_peak = probe_read_bandwidth(8 << 30, 5, 0)          # chunks interleaved over the CTAs
    read_streams = probe_read_bandwidth(16 << 30, 5, 1)      # one contiguous stream per CTA, like k_apply
    traffic = None
    prof = os.path.join(ROOT, "profiles", "k_apply_traffic.json")
    if os.path.exists(prof):
        with open(prof) as f:
            tj = json.load(f)
        key = cfg.name if world == 1 else f"{cfg.name}/{world}"
        traffic = tj.get(key, {}).get("dram_bytes_per_launch")
    launches_tot = int(sum(gather(float(launches))))
    if fcls["batched"]:
        # D28: the shared-factor apply is a batch of complex GEMMs on the FP64 tensor cores -- tensor-bound; achieved =
        # algorithmic flops (8 m^2 per block step of every subdomain, SURVEY 8(d)'s GEMV work in flops) / kernel time
        fl_r = gather(float(fcls["apply_flop"]))
        tf_r = [fl_r[q] / (ms_r[q] / 1e3) / 1e12 for q in range(world)]
        slow_t = max(range(world), key=lambda q: ms_r[q])
        tprof = os.path.join(ROOT, "profiles", "k_apply_batch_traffic.json")
        btraffic = None
        if os.path.exists(tprof):
            with open(tprof) as f:
                btraffic = json.load(f).get(cfg.name if world == 1 else f"{cfg.name}/{world}", {}).get(
                    "dram_bytes_per_launch")
        roofline = {"bound": "tensor", "achieved": tf_r[slow_t], "peak": dmma_peak, "unit": "TFLOP/s",
                    "frac": tf_r[slow_t] / dmma_peak, "traffic": btraffic,
                    "kernel": "k_apply_batch (shared-factor twisted block solves as complex GEMMs on DMMA, D28)",
                    "algorithmic_flop_per_launch": fcls["apply_flop"], "issued_flop_per_launch": fcls["apply_flop_issued"],
                    "issued_frac": fcls["apply_flop_issued"] / (ms_r[slow_t] / 1e3) / 1e12 / dmma_peak,
                    "peak_source": "helm_probe_fp64_tflops(DMMA), measured on this GPU: MEASURED_PEAKS.json has no FP64 "
                                   "figure (its bf16 1671.8 x the nominal FP64/bf16 ratio 40/2250 = 29.7, below the probe)",
                    "classes": fcls["classes"], "tiles": fcls["tiles"],
                    "per_gpu": world > 1, "slowest_rank": slow_t, "achieved_per_rank": tf_r,
                    "apply_kernel_ms": ms_r[slow_t], "apply_share_of_step": apply_ms / ms}
    else:
        roofline = {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                    "traffic": traffic, "kernel": "k_apply (fused restrict + twisted block solves + owner write)",
                    "algorithmic_bytes_per_launch": lay["apply_bytes"], "peak_source": peak_src,
                    "per_gpu": world > 1, "slowest_rank": slow, "achieved_per_rank": ach_r,
                    "band_equivalent_GBps": lay["band_bytes"] / (apply_avg_ms / 1e3) / 1e9,
                    "read_stream_probe_GBps": read_peak, "frac_of_read_probe": achieved / read_peak,
                    "read_streams_probe_GBps": read_streams, "frac_of_read_streams_probe": achieved / read_streams,
                    "apply_kernel_ms": ms_r[slow], "apply_share_of_step": apply_ms / ms,
                    "cycle_algorithmic_bytes": cyc_b, "cycle_frac": cyc_b / (hbm * 1e9) / (ms / args.steps / 1e3)}

    out = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms / args.steps, "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": workload_desc(cfg, world),
        "layout": {"n_free": lay["n_free_global"], "cells_per_side": lay["N_cells"], "delta": lay["n_ovlp"],
                   "kappa": lay["n_pml"], "local_unknowns_rank0": lay["local_unknowns"], "m_max": lay["m_max"],
                   "factor_GB_rank0": round(lay["factor_bytes"] / 1e9, 3),
                   "apply_GB_rank0": round(lay["apply_bytes"] / 1e9, 3), "orth": args.orth},
        "roofline": roofline,
        "factor_sharing": {"classes": fcls["classes"], "batched_apply": fcls["batched"], "tiles": fcls["tiles"],
                           "factor_bytes_on_device": fcls["factor_bytes"],
                           "note": "D28: subdomains with bitwise-equal local operators share one factorisation"},
        "e2e": {"value": e_its / e2e_s, "unit": UNIT, "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                "api": "helm_gmres_host (host b/x, copies inside every call), one call per cycle"},
        "gpu_launches": launches_tot,
        "iterations": its, "applies": its,
        "apply_only": ({"ms": apply_only_ms, "applies_per_s": 1e3 / apply_only_ms,
                        "TFLOPs": fcls["apply_flop"] / apply_only_ms / 1e9} if fcls["batched"] else
                       {"ms": apply_only_ms, "applies_per_s": 1e3 / apply_only_ms,
                        "GBps": lay["apply_bytes"] / apply_only_ms / 1e6}),
        "gmres_tts": {"seconds": tts_s, "iterations": tinfo.iterations, "restarts": tinfo.restarts,
                      "relres_true": tinfo.relres_true, "status": tinfo.status, "rtol": cfg.rtol,
                      "applies_per_s": tinfo.iterations / tts_s,
                      "algorithmic_bytes": tts_b, "roofline_s": tts_roof_s, "roofline_frac": tts_roof_s / tts_s,
                      "roofline_note": ("vector work (SpMV, orthogonalisation) at the HBM peak + the apply's flops at "
                                        "the measured DMMA peak" if fcls["batched"] else
                                        "all algorithmic bytes at the HBM peak")},
        "setup_factor_s": setup_s,
        "factor": factor_roofline(lay, factor_s, gather),
        "comm": comm,
        "clocks": clk.summary(),
    }
    if world == 1 and not args.no_paper:
        out["per_subdomain_factors"] = per_subdomain_factors(cfg, stream, hbm, peak_src, read_streams)
    if world == 1 and not args.no_tts:
        out["tts_vs_k"] = tts_vs_k(stream, cfg, tts_s, tinfo, factor_s, apply_only_ms)
    if world == 1 and not args.no_paper:
        out["paper_table4"] = paper_table4(stream)
        out["gmres_tts_ramp_pou"] = ramp_pou_tts(cfg, stream, xy, amp, sig)
    if world > 1:
        out["nccl_init"] = nccl_init_lines(nccl_log + ".*.log") if rank == 0 else []
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        out["cpu_baseline"] = cpu_baseline(cfg)
    if rank == 0:
        print(json.dumps(out), flush=True)
    ctx.close()
    if world > 1:
        dist.destroy_process_group()


def tts_vs_k(stream, cfg_main, tts_main, tinfo_main, factor_main, apply_main_ms):
    """BASELINE.json's 'GMRES time-to-solve vs k; local-solve HBM GB/s': every single-GPU config c0..c3 solved to 1e-6
    on this GPU (factorisation, solve and the apply alone timed with CUDA events; the bench config's own numbers
    reused), beside the oracle's solve of the same system from the golden records (another host: context).  c4
    (k = 3200, 26 M unknowns; one GPU since the shared factors, D28) runs the golden record's first six GMRES(50)
    cycles (maxit 300: the oracle solve to 1e-6 would take many hours), reported with its status and residual."""
    import torch

    from paper_2602_00735_b200 import Context
    from paper_2602_00735_b200.workloads import CONFIGS, sources
    rows = []
    for name in ("c0", "c1", "c2", "c3", "c4"):
        c = CONFIGS[name]
        gold = os.path.join(ROOT, "tests", "golden", f"{name}_gmres.json")
        orc, maxit = None, 5000
        if os.path.exists(gold):
            with open(gold) as f:
                g = json.load(f)
            orc = {"iterations": g["iterations"], "gmres_s": g["oracle_timing"]["gmres_s"],
                   "cores": g["oracle_timing"]["host"]["cores"], "relres": g["relres_true"], "maxit": g["maxit"]}
            if name == "c4":
                maxit = g["maxit"]
        if name == cfg_main.name:
            rows.append({"config": name, "k": c.k, "subdomains": c.nsub ** 2, "factor_s": factor_main,
                         "solve_s": tts_main, "iterations": tinfo_main.iterations, "relres_true": tinfo_main.relres_true,
                         "apply_ms": apply_main_ms, "oracle": orc})
            continue
        torch.cuda.synchronize()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
        # first setup of this shape (includes the lazy loading of its kernel instances), then the one reported
        ctx = Context(c.k, c.nsub, c.nsub, stream=stream)
        ev[0].record(stream)
        ctx.factor()
        ev[1].record(stream)
        torch.cuda.synchronize()
        factor_first_s = ev[0].elapsed_time(ev[1]) / 1e3
        ctx.close()
        ctx = Context(c.k, c.nsub, c.nsub, stream=stream)
        ev[0].record(stream)
        ctx.factor()
        ev[1].record(stream)
        b = ctx.rhs(*sources(c))
        ctx.gmres(b, restart=c.restart, rtol=c.rtol, maxit=min(maxit, 2 * c.restart))   # warm-up (first launches)
        ev[2].record(stream)
        _, info, _ = ctx.gmres(b, restart=c.restart, rtol=c.rtol, maxit=maxit)
        ev[3].record(stream)
        torch.cuda.synchronize()
        factor_s_row, solve_s_row = ev[0].elapsed_time(ev[1]) / 1e3, ev[2].elapsed_time(ev[3]) / 1e3
        v = torch.randn(ctx.n, dtype=torch.complex128, device="cuda")
        z = torch.empty_like(v)
        for _ in range(3):
            ctx.precond_apply(v, z)
        ev[0].record(stream)
        for _ in range(20):
            ctx.precond_apply(v, z)
        ev[1].record(stream)
        torch.cuda.synchronize()
        apply_ms = ev[0].elapsed_time(ev[1]) / 20
        lay = ctx.layout
        rows.append({"config": name, "k": c.k, "subdomains": c.nsub ** 2, "factor_s": factor_s_row,
                     "factor_first_call_s": factor_first_s, "solve_s": solve_s_row, "iterations": info.iterations,
                     "relres_true": info.relres_true, "status": info.status, "maxit": maxit, "apply_ms": apply_ms,
                     "tensor_core_apply": ctx.factor_classes()["batched"], "oracle": orc})
        ctx.close()
        del ctx, b
        torch.cuda.empty_cache()
    return rows


def per_subdomain_factors(cfg, stream, hbm, peak_src, read_streams):
    """The general path of the method (every subdomain factored and its inverse blocks streamed from HBM per apply:
    HELM_SHARE_FACTORS=0, what a variable wave speed needs) on the same workload: factorisation, apply alone and its
    HBM roofline -- BASELINE.json's 'local-solve HBM GB/s'."""
    import torch

    from paper_2602_00735_b200 import Context
    old = os.environ.get("HELM_SHARE_FACTORS")
    os.environ["HELM_SHARE_FACTORS"] = "0"
    try:
        ctx = Context(cfg.k, cfg.nsub, cfg.nsub, stream=stream)
    finally:
        if old is None:
            del os.environ["HELM_SHARE_FACTORS"]
        else:
            os.environ["HELM_SHARE_FACTORS"] = old
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    ev[0].record(stream)
    ctx.factor()
    ev[1].record(stream)
    v = torch.randn(ctx.n, dtype=torch.complex128, device="cuda")
    z = torch.empty_like(v)
    for _ in range(3):
        ctx.precond_apply(v, z)
    ev[2].record(stream)
    for _ in range(10):
        ctx.precond_apply(v, z)
    ev[3].record(stream)
    torch.cuda.synchronize()
    lay = ctx.layout
    ms = ev[2].elapsed_time(ev[3]) / 10
    gbps = lay.apply_bytes / ms / 1e6
    res = {"factor_s": ev[0].elapsed_time(ev[1]) / 1e3, "factor_GB": round(lay.factor_bytes / 1e9, 3),
           "apply_ms": ms, "applies_per_s": 1e3 / ms, "algorithmic_bytes_per_launch": lay.apply_bytes,
           "achieved_GBps": gbps, "peak_GBps": hbm, "peak_source": peak_src, "frac": gbps / hbm,
           "frac_of_read_streams_probe": gbps / read_streams, "kernel": "k_apply", "classes": ctx.factor_classes()["classes"]}
    ctx.close()
    del ctx, v, z
    torch.cuda.empty_cache()
    return res


def factor_roofline(lay, factor_s, gather):
    """Setup factorisation (s3) against the FP64 tensor-core peak MEASURED on this GPU (helm_probe_fp64_tflops: DMMA
    issue rate; MEASURED_PEAKS.json has no FP64 figure): flops = sum over blocks of 8 m^3 (Gauss-Jordan inversions)."""
    from paper_2602_00735_b200.helm import probe_fp64_tflops
    dmma = probe_fp64_tflops(0)
    dfma = probe_fp64_tflops(1)
    flop = sum(gather(float(lay["factor_flop"])))
    ach = flop / factor_s / 1e12
    return {"seconds": factor_s, "tflop": flop / 1e12, "achieved_tflops": ach, "bound": "tensor",
            "peak_dmma_tflops_measured": dmma, "peak_dfma_tflops_measured": dfma, "frac": ach / dmma,
            "kernel": "k_factor_chains + k_factor_twist (8-wide blocked Gauss-Jordan, DMMA)"}


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


# ====================================================================================== oracle arm
def cpu_threads():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count() or 1


def host_info():
    model, ram = "", None
    try:
        with open("/proc/cpuinfo") as f:
            model = next((ln.split(":", 1)[1].strip() for ln in f if ln.startswith("model name")), "")
        with open("/proc/meminfo") as f:
            ram = round(int(f.readline().split()[1]) / 2 ** 20, 1)
    except (OSError, ValueError, IndexError):
        pass
    return {"cores": cpu_threads(), "cpu_model": model, "ram_GiB": ram}


class OracleSteps:
    """The oracle at the full size of the workload, as it stands: dedup-mode factorisation (SURVEY 8(d) memory
    fallback: one band LU per bitwise-distinct A_j, exact), then full oracle Arnoldi steps -- w = A(B^-1 v) over every
    subdomain and every row, MGS against the first j + 1 basis vectors (oracle.mgs, O9 step 2), ||w||."""

    def __init__(self, cfg):
        import numpy as np

        from oracle.oracle import Oracle
        from paper_2602_00735_b200.workloads import probe_vector
        self.np = np
        t = time.perf_counter()
        self.o = Oracle.from_config(k=cfg.k, nsub_x=cfg.nsub, nsub_y=cfg.nsub)
        self.classes = self.o.factor_dedup()
        self.factor_s = time.perf_counter() - t
        n = self.o.nfree
        # a basis of restart + 1 unit vectors (the MGS cost does not depend on their content)
        self.V = []
        for i in range(cfg.restart + 1):
            v = probe_vector(n, 1000 + i)
            self.V.append(v / np.linalg.norm(v))
        self.o.matvec(self.V[0])                      # first call assembles the global stencil (untimed)

    def step(self, j: int) -> float:
        from oracle.oracle import mgs
        t = time.perf_counter()
        w = self.o.matvec(self.o.apply(self.V[j]))
        w, _ = mgs(self.V[:j + 1], w)
        self.np.linalg.norm(w)
        return time.perf_counter() - t

    def apply_s(self, reps: int = 3) -> float:
        ts = []
        for _ in range(reps):
            t = time.perf_counter()
            self.o.apply(self.V[0])
            ts.append(time.perf_counter() - t)
        return statistics.median(ts)


def depths(k_steps: int, restart: int):
    """Krylov depths of the reference arm's steps: spread evenly over one cycle (cycle-average cost)."""
    return [min(restart - 1, int((s + 0.5) * restart / k_steps)) for s in range(k_steps)]


def oracle_golden_timing(cfg):
    """The full oracle GMRES(50) solve of this config as recorded by scripts/make_golden.py (oracle only, hours of
    host time at c3/c4: run once and cached, keyed by config, seed and oracle source hash)."""
    path = os.path.join(ROOT, "tests", "golden", f"{cfg.name}_gmres.json")
    if not os.path.exists(path):
        return None
    with open(path) as f:
        g = json.load(f)
    sys.path.insert(0, os.path.join(ROOT, "scripts"))
    try:
        from make_golden import oracle_hash
        cur = oracle_hash()
    except Exception:
        cur = None
    t = g.get("oracle_timing", {})
    return {"gmres_s": t.get("gmres_s"), "iterations": g.get("iterations"), "restarts": g.get("restarts"),
            "maxit": g.get("maxit"), "status": g.get("status"), "seed": g.get("seed"),
            "host": t.get("host"), "when": t.get("when"), "oracle_hash": g.get("oracle_hash"),
            "oracle_hash_current": cur, "cached": True}


def cpu_baseline(cfg):
    """Rank 0, N = 1: the oracle timed on this box's host cores on a bounded sample -- ONE full-size oracle Arnoldi
    step at the cycle-average depth (restart / 2) -- plus the full oracle's factorisation and apply (median of 3)
    timed here and its whole GMRES solve from the cached golden record."""
    os.environ.setdefault("OMP_NUM_THREADS", str(cpu_threads()))
    st = OracleSteps(cfg)
    j = cfg.restart // 2
    sec = st.step(j)
    return {"value": 1.0 / sec, "unit": UNIT, "cores": int(os.environ["OMP_NUM_THREADS"]), "kind": "oracle",
            "sample": f"one full-size oracle GMRES Arnoldi step on {cfg.name} at Krylov depth {j} (the cycle average): "
                      f"band-LU RAS apply over all {st.o.nsub} subdomains (dedup mode, {st.classes} factor classes), "
                      f"full matvec, MGS against {j + 1} vectors",
            "seconds_per_step": sec, "host": host_info(),
            "full_oracle": {"factor_dedup_s": st.factor_s, "classes": st.classes, "apply_s_median3": st.apply_s(),
                            "gmres": oracle_golden_timing(cfg)}}


def run_reference(args):
    from paper_2602_00735_b200.workloads import CONFIGS
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    os.environ.setdefault("OMP_NUM_THREADS", str(cpu_threads()))
    cfg = CONFIGS[args.config]
    if args.seed is not None:
        import dataclasses
        cfg = dataclasses.replace(cfg, seed=args.seed)
    st = OracleSteps(cfg)
    for _ in range(args.warmup):
        st.step(0)
    ds = depths(args.steps, cfg.restart)
    ts = [st.step(j) for j in ds]
    total = sum(ts)
    value = args.steps / total
    cores = int(os.environ["OMP_NUM_THREADS"])
    desc = (f"each step one full-size oracle GMRES Arnoldi step on {cfg.name} (band-LU RAS apply over all "
            f"{st.o.nsub} subdomains in dedup mode, full matvec, MGS, norm) at Krylov depths spread evenly over a "
            f"GMRES({cfg.restart}) cycle ({min(ds)}..{max(ds)}); warm-up steps at depth 0; setup "
            f"{st.factor_s:.1f} s untimed")
    out = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * total / args.steps,
           "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": workload_desc(cfg, args.gpus),
           "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle", "sample": desc,
                            "host": host_info()},
           "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def relaunch_distributed(args):
    """--gpus N > 1 without torchrun's environment: run this script under torch.distributed.run, one rank per GPU
    (rendezvous on 127.0.0.1), and pass its output through."""
    import socket
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c3")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-paper", action="store_true", help="skip the paper Table 4 comparison rows")
    ap.add_argument("--no-tts", action="store_true", help="skip the time-to-solve-vs-k rows (c0..c4)")
    ap.add_argument("--seed", type=int, default=None, help="source draw seed (default: the config's, = k)")
    ap.add_argument("--orth", default="dcgs2", choices=["dcgs2", "cgs2"],
                    help="GMRES orthogonalisation (DESIGN.md 5.6); cgs2 = the undelayed form, for A/B")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    elif args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        sys.exit(relaunch_distributed(args))
    else:
        run_ours(args)


if __name__ == "__main__":
    main()

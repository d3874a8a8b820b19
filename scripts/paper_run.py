"""Run one of the paper's workloads (Tables 1-4 rows) end to end on N GPUs and print one JSON line.

    python scripts/paper_run.py --config t1200                       # one GPU
    torchrun --nproc-per-node 2 --master-addr 127.0.0.1 scripts/paper_run.py --config t2400 --gpus 2

Setup (assembly) + factorisation, then Algorithm 1 (Richardson, the paper's solver for Tables 1/3/4) or GMRES to
rtol 1e-10, timed with CUDA events on the library stream, max over ranks.  RAS-PML-Imp with the linear-ramp PoU, as in
the paper; --drch for RAS-PML-Drch.  k >= 2400 needs >= 2 GPUs (factor storage > 180 GB on one).
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="t1200")
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--solver", default="richardson", choices=["richardson", "gmres"])
    ap.add_argument("--drch", action="store_true")
    ap.add_argument("--warmup", type=int, default=1, help="untimed warm-up on a small paper-type problem (0: off)")
    args = ap.parse_args()

    import torch
    import torch.distributed as dist

    from paper_2602_00735_b200 import Context
    from paper_2602_00735_b200.helm import BC_DIRICHLET, nccl_unique_id, paper_params
    from paper_2602_00735_b200.workloads import PAPER_CONFIGS, paper_source

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", "0")))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    nccl_id = None
    if world > 1:
        dist.init_process_group("nccl")
        buf = torch.zeros(128, dtype=torch.uint8, device="cuda")
        if rank == 0:
            buf.copy_(torch.frombuffer(bytearray(nccl_unique_id()), dtype=torch.uint8))
        dist.broadcast(buf, src=0)
        nccl_id = bytes(buf.cpu().numpy().tobytes())
    if args.warmup:   # untimed: CUDA context, lazily loaded kernels and clocks, through the same code paths
        for kw_, ns_ in ((60.0, 2), (100.0, 1)):
            w = Context(**paper_params(kw_, ns_, 4, 2), rank=0, nranks=1)
            w.factor()
            w.richardson(w.rhs(*paper_source(kw_)), rtol=1e-6, maxit=3)
            w.close()
    c = PAPER_CONFIGS[args.config]
    kw = paper_params(c.k, c.nsub, c.pml, c.ovlp, n_cells=c.n_cells)
    if args.drch:
        kw["local_bc"] = BC_DIRICHLET
    stream = torch.cuda.Stream()   # dedicated library stream (NCCL on a non-default stream)
    torch.cuda.set_stream(stream)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    ev[0].record(stream)
    ctx = Context(**kw, rank=rank, nranks=world, stream=stream, nccl_id=nccl_id)
    ctx.factor()
    ev[1].record(stream)
    b = ctx.rhs(*paper_source(c.k))
    ev[2].record(stream)
    if args.solver == "richardson":
        _, info, _ = ctx.richardson(b, rtol=c.rtol, maxit=c.maxit)
        its, res, status = info.iterations, info.relres, info.status
    else:
        _, info, _ = ctx.gmres(b, restart=50, rtol=c.rtol, maxit=c.maxit)
        its, res, status = info.iterations, info.relres_true, info.status
    ev[3].record(stream)
    torch.cuda.synchronize()
    t = torch.tensor([ev[0].elapsed_time(ev[1]), ev[2].elapsed_time(ev[3])], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    lay = ctx.layout
    out = {"config": args.config, "k": c.k, "grid": c.n_cells, "subdomains": c.nsub ** 2, "pml": c.pml,
           "ovlp": c.ovlp, "local_bc": "drch" if args.drch else "imp", "pou": "ramp", "solver": args.solver,
           "n_gpus": world, "setup_factor_s": float(t[0]) / 1e3, "solve_s": float(t[1]) / 1e3, "iterations": its,
           "relres": res, "status": status, "factor_GB_per_rank": lay.factor_bytes / 1e9}
    if rank == 0:
        print(json.dumps(out), flush=True)
    ctx.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()

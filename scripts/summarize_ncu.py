"""Summarise ncu outputs into profiles/ (tracked): per-kernel launch shares and the top kernel's traffic."""
import csv, json, os, subprocess, sys
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def launches(path, out_md, title):
    rows = [r for r in csv.reader(open(path)) if len(r) > 10]
    h = rows[0]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    agg = defaultdict(lambda: [0, 0.0])
    for r in rows[1:]:
        if r[h.index("Metric Name")] != "gpu__time_duration.sum":
            continue
        name = r[ki].split("(")[0].replace("<unnamed>::", "")
        v = float(r[vi].replace(",", ""))
        scale = {"ns": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0}.get(r[ui], 1e-6)
        agg[name][0] += 1
        agg[name][1] += v * scale
    tot = sum(v[1] for v in agg.values())
    with open(out_md, "w") as f:
        f.write(f"# {title}\n\nncu `--metrics gpu__time_duration.sum --clock-control none` over every launch of the command "
                "(cold-cache, serialised: compare shares, not absolutes).\n\n| kernel | launches | total ms | share | avg ms |\n|---|---|---|---|---|\n")
        for k, (n, ms) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
            f.write(f"| {k} | {n} | {ms:.3f} | {100 * ms / tot:.1f}% | {ms / n:.4f} |\n")
        f.write(f"| **total** | {sum(v[0] for v in agg.values())} | {tot:.3f} | 100% | |\n")
    return agg


def full(rep, key, out_json, keep):
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(raw.splitlines()))
    h, u = rows[0], rows[1]
    res = {}
    for row in rows[2:]:
        d = {k: (un, v) for k, un, v in zip(h, u, row)}
        def val(name):
            un, v = d[name]
            v = float(v.replace(",", ""))
            return v * {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12, "ns": 1e-9, "us": 1e-6,
                        "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "s": 1.0}.get(un, 1.0)
        rd, wr, t = val("dram__bytes_read.sum"), val("dram__bytes_write.sum"), val("gpu__time_duration.sum")
        res = {"kernel": d["Kernel Name"][1], "dram_read_bytes": rd, "dram_write_bytes": wr,
               "dram_bytes_per_launch": rd + wr, "duration_s": t, "dram_GBps": (rd + wr) / t / 1e9,
               "metrics": {k: d[k][0] + " " + d[k][1] for k in keep if k in d}}
    j = json.load(open(out_json)) if os.path.exists(out_json) else {}
    j[key] = res
    json.dump(j, open(out_json, "w"), indent=1)
    return res


if __name__ == "__main__":
    cmd = sys.argv[1]
    if cmd == "launches":
        launches(sys.argv[2], sys.argv[3], sys.argv[4])
    else:
        keep = ["dram__throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
                "launch__registers_per_thread", "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block",
                "launch__occupancy_limit_shared_mem", "sm__warps_active.avg.pct_of_peak_sustained_active",
                "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
                "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
                "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
                "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
                "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
                "lts__t_sector_hit_rate.pct",
                "smsp__average_warps_issue_stalled_math_pipe_throttle_per_issue_active.ratio",
                "smsp__pipe_tensor_subpipe_dmma_cycles_active.avg", "sm__cycles_active.avg", "sm__cycles_elapsed.avg",
                "sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
                "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum"]
        print(json.dumps(full(sys.argv[2], sys.argv[3], sys.argv[4], keep), indent=1))

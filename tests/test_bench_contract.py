"""bench.py's reference arm (the oracle: the only reference this paper has) runs on CPU and prints one contract line
with the same config dict as the GPU arm; the relaunch command for --gpus N is torch.distributed.run.  -m "not gpu"."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_line_c0():
    out = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--config", "c0",
                          "--steps", "2", "--warmup", "3"], capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "applies/s" and d["steps"] == 2
    assert d["higher_is_better"] is True and d["dtype"] == "f64" and d["vs_baseline"] is None
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] >= 1
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["value"] == d["value"]
    sys.path.insert(0, ROOT)
    import bench
    from paper_2602_00735_b200.workloads import CONFIGS
    assert d["config"] == json.loads(json.dumps(bench.workload_desc(CONFIGS["c0"], 1)))   # the GPU arm's dict
    assert abs(d["ms_per_step"] * d["steps"] / 1e3 - d["steps"] / d["value"]) <= 1e-9 * d["steps"] / d["value"] + 1e-9


def test_depths_spread_over_a_cycle():
    sys.path.insert(0, ROOT)
    import bench
    ds = bench.depths(20, 50)
    assert len(ds) == 20 and min(ds) >= 0 and max(ds) <= 49
    assert abs(sum(ds) / len(ds) - 24.5) <= 1.0          # the cycle-average depth


def test_relaunch_command_for_several_gpus(monkeypatch):
    """--gpus N without torchrun's environment re-launches bench.py under torch.distributed.run: one process per GPU,
    rendezvous on 127.0.0.1, the same arguments."""
    sys.path.insert(0, ROOT)
    import argparse

    import bench
    seen = {}
    monkeypatch.setattr(bench.subprocess, "call", lambda cmd: seen.setdefault("cmd", cmd) and 0)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "4", "--steps", "7"])
    bench.relaunch_distributed(argparse.Namespace(gpus=4))
    cmd = seen["cmd"]
    assert cmd[1:3] == ["-m", "torch.distributed.run"] and "--nproc-per-node=4" in cmd and "--nnodes=1" in cmd
    assert cmd[cmd.index("--master-addr") + 1] == "127.0.0.1"
    assert cmd[-4:] == ["--gpus", "4", "--steps", "7"] and cmd[-5].endswith("bench.py")

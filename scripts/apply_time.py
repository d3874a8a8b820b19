"""Time the preconditioner apply alone on one config (default c3): best of 3 x 10 applies, CUDA events."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2602_00735_b200 import Context  # noqa: E402
from paper_2602_00735_b200.workloads import CONFIGS  # noqa: E402

cfg = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "c3"]
c = Context(cfg.k, cfg.nsub, cfg.nsub)
c.factor()
torch.manual_seed(0)
v = torch.randn(c.n, dtype=torch.complex128, device="cuda")
for _ in range(2):
    c.precond_apply(v)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
best = 1e9
for _ in range(3):
    e0.record()
    for _ in range(10):
        c.precond_apply(v)
    e1.record()
    torch.cuda.synchronize()
    best = min(best, e0.elapsed_time(e1) / 10)
print(f"{cfg.name} apply {best:.3f} ms {c.layout.apply_bytes / best / 1e6:.0f} GB/s", flush=True)

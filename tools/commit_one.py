"""Commit one large tensor a few times (for ncu captures of the SHA-256 kernels)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2502_19405_b200 as R
n = int(sys.argv[1]) if len(sys.argv) > 1 and sys.argv[1].isdigit() else 256 * 1024 * 1024
torch.manual_seed(0)
x = torch.rand(n, device="cuda")
d = torch.empty((1, 32), dtype=torch.uint8, device="cuda")
plan = R.CommitPlan([x], d)
for _ in range(3):
    plan.run()
torch.cuda.synchronize()
if "--time" in sys.argv:
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(10):
        plan.run()
    e.record()
    torch.cuda.synchronize()
    ms = s.elapsed_time(e) / 10
    print(f"commit {4 * n / 2**20:.0f} MiB: {ms:.3f} ms  {4 * n / ms / 1e6:.1f} GB/s  digest {d[0, :8].cpu().numpy().tobytes().hex()}")

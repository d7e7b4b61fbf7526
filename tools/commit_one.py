"""Commit one large tensor a few times (for ncu captures of the SHA-256 kernels)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2502_19405_b200 as R
n = int(sys.argv[1]) if len(sys.argv) > 1 else 256 * 1024 * 1024
x = torch.rand(n, device="cuda")
d = torch.empty((1, 32), dtype=torch.uint8, device="cuda")
plan = R.CommitPlan([x], d)
for _ in range(3):
    plan.run()
torch.cuda.synchronize()

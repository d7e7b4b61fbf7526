"""Run one R-GEMM launch configuration a few times (for ncu captures)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2502_19405_b200 as R
M, N, K = (int(x) for x in sys.argv[1].split("x"))
ta, tb, cfg = int(sys.argv[2]), int(sys.argv[3]), int(sys.argv[4])
cfg = None if cfg < 0 else cfg
A = torch.rand((K, M) if ta else (M, K), device="cuda") * 2 - 1
B = torch.rand((N, K) if tb else (K, N), device="cuda") * 2 - 1
C = torch.empty(M, N, device="cuda")
for _ in range(3):
    R.repops_gemm(A, B, transA=bool(ta), transB=bool(tb), out=C, cfg=cfg)
torch.cuda.synchronize()

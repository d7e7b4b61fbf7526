"""Run torch.mm (cuBLAS FP32 SGEMM, TF32 off) a few times -- for ncu captures of the
library kernel next to the R-GEMM (context: what the non-reproducible library does)."""
import sys
import torch
torch.backends.cuda.matmul.allow_tf32 = False
M, N, K = (int(x) for x in sys.argv[1].split("x"))
ta, tb = int(sys.argv[2]), int(sys.argv[3])
A = torch.rand((K, M) if ta else (M, K), device="cuda") * 2 - 1
B = torch.rand((N, K) if tb else (K, N), device="cuda") * 2 - 1
Ab = A.t() if ta else A
Bb = B.t() if tb else B
for _ in range(4):
    C = torch.mm(Ab, Bb)
torch.cuda.synchronize()

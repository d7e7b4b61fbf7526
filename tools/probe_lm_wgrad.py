import sys, os
sys.path.insert(0, os.getcwd())
import torch
import paper_2502_19405_b200 as R
b, M, N, K = 8, 50257, 768, 512
A = torch.rand((b, K, 50260), device="cuda")[:, :, :M]
B = torch.rand((b, K, N), device="cuda")
Cr = torch.empty((b, M, N), device="cuda")
def run(cfg=None):
    if cfg is not None:
        from paper_2502_19405_b200._lib import lib
        lib().repops_gemm_force_cfg(cfg)
    R.repops_gemm_strided_batched(A, B, Cr, M=M, N=N, K=K, lda=A.stride(1), ldb=N, ldc=N, sA=(A.stride(0), 0), sB=(K*N, 0), sC=(M*N, 0), batch=(b, 1), transA=True)
for cfg in (-1, 20, 6, 22):
    for _ in range(2): run(cfg)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(5): run(cfg)
    e.record(); torch.cuda.synchronize()
    print("cfg", cfg, 2*b*M*N*K/(s.elapsed_time(e)/5)/1e9)

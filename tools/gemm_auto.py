import sys, os
sys.path.insert(0, os.getcwd())
import torch
import paper_2502_19405_b200 as R
def t_ms(fn, iters=5, warm=2):
    for _ in range(warm): fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / iters
shapes = [(8192,8192,8192),(4096,4096,4096),(2048,2048,2048),(1024,1024,1024),(4096,2304,768),(4096,3072,768),(4096,768,3072),(4096,768,768),(4096,50304,768),(768,2304,4096)]
for ta in (1, 0):
    for (M,N,K) in shapes:
        A = torch.rand((K, M) if ta else (M, K), device="cuda") * 2 - 1
        B = torch.rand((K, N), device="cuda") * 2 - 1
        C = torch.empty(M, N, device="cuda")
        ms = t_ms(lambda: R.repops_gemm(A, B, transA=bool(ta), out=C))
        torch.backends.cuda.matmul.allow_tf32 = False
        Ab = A.t() if ta else A
        mc = t_ms(lambda: torch.mm(Ab, B))
        print(f"{'TN' if ta else 'NN'} {M}x{N}x{K}: auto {2*M*N*K/ms/1e9:6.1f}  cublas {2*M*N*K/mc/1e9:6.1f} TFLOP/s", flush=True)

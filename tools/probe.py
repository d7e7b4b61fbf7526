"""Quick device timing of the main kernels (CUDA events, not a bench number)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import sys, time
import torch
import paper_2502_19405_b200 as R

def t_ms(fn, iters=10, warm=3):
    for _ in range(warm): fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / iters

torch.manual_seed(0)
for n in (1024, 2048, 4096, 8192):
    A = torch.rand(n, n, device="cuda") * 2 - 1
    B = torch.rand(n, n, device="cuda") * 2 - 1
    C = torch.empty(n, n, device="cuda")
    for cfg in (0, 1):
        ms = t_ms(lambda: R.repops_gemm(A, B, out=C, cfg=cfg))
        print(f"repops_gemm n={n} cfg={cfg}: {ms:.3f} ms  {2*n**3/ms/1e9:.1f} TFLOP/s", flush=True)
    for ta, tb in ((0, 1), (1, 0)):
        ms = t_ms(lambda: R.repops_gemm(A, B, transA=bool(ta), transB=bool(tb), out=C))
        print(f"repops_gemm n={n} tA={ta} tB={tb}: {ms:.3f} ms  {2*n**3/ms/1e9:.1f} TFLOP/s", flush=True)
    torch.backends.cuda.matmul.allow_tf32 = False
    ms = t_ms(lambda: torch.mm(A, B, out=C))
    print(f"cublas sgemm n={n}: {ms:.3f} ms  {2*n**3/ms/1e9:.1f} TFLOP/s", flush=True)
x = torch.rand(96 * 512 * 8, 512, device="cuda")
ms = t_ms(lambda: R.repops_softmax(x, causal=True, out=x))
print(f"softmax 393216x512 causal: {ms:.3f} ms {x.numel()*8/ms/1e6:.0f} GB/s")
x = torch.rand(4096 * 8, 768, device="cuda"); g = torch.rand(768, device="cuda"); b = torch.rand(768, device="cuda")
y = torch.empty_like(x)
ms = t_ms(lambda: R.repops_layernorm(x, g, b, out=y))
print(f"layernorm 32768x768: {ms:.3f} ms {x.numel()*8/ms/1e6:.0f} GB/s")
x = torch.rand(256 * 1024 * 1024, device="cuda")
ms = t_ms(lambda: R.repops_exp(x, out=x))
print(f"exp 256M: {ms:.3f} ms {x.numel()*8/ms/1e6:.0f} GB/s")
ws = R.CommitWorkspace()
ms = t_ms(lambda: R.verde_commit_tensors([x], ws=ws), iters=3, warm=1)
print(f"commit 1 GiB: {ms:.3f} ms {x.numel()*4/ms/1e6:.0f} GB/s")

"""Do independent GEMMs of the GPT-2 backward (dgrad N=768 output: 384 tiles on 444
CTA slots; per-shard wgrad batch) gain from running on two streams?"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2502_19405_b200 as R

torch.manual_seed(0)
M, d, F, T, S = 4096, 768, 3072, 512, 8
dY = torch.rand(M, d, device="cuda") - 0.5       # d fc2 out
W2T = torch.rand(d, F, device="cuda") - 0.5      # fc2.w^T (d x F)
G = torch.rand(M, F, device="cuda") - 0.5        # gelu activations
dG = torch.empty(M, F, device="cuda")
dW = torch.empty(S, F, d, device="cuda")
dX = torch.empty(M, d, device="cuda")
W1T = torch.rand(F, d, device="cuda") - 0.5
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def dgrad(st):  # dX = dfc . W_fc^T : N = 768
    R.repops_gemm(G, W1T, out=dX, stream=st)


def wgrad(st):  # per shard dW_s = G_s^T dY_s  (TN batched)
    R.repops_gemm_strided_batched(G, dY, dW, M=F, N=d, K=T, lda=F, ldb=d, ldc=d, sA=(T * F, 0), sB=(T * d, 0),
                                  sC=(F * d, 0), batch=(S, 1), transA=True, stream=st)


def timed(fn, n=10):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n


def serial():
    st = torch.cuda.current_stream()
    dgrad(st)
    wgrad(st)


def concurrent():
    cur = torch.cuda.current_stream()
    e = torch.cuda.Event()
    e.record(cur)
    s1.wait_event(e)
    s2.wait_event(e)
    dgrad(s1)
    wgrad(s2)
    e1, e2 = torch.cuda.Event(), torch.cuda.Event()
    e1.record(s1)
    e2.record(s2)
    cur.wait_event(e1)
    cur.wait_event(e2)


print(f"dgrad alone {timed(lambda: dgrad(torch.cuda.current_stream())):.3f} ms  "
      f"wgrad alone {timed(lambda: wgrad(torch.cuda.current_stream())):.3f} ms  "
      f"serial {timed(serial):.3f} ms  two streams {timed(concurrent):.3f} ms")

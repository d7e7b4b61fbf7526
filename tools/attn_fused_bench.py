"""Fused attention forward vs the three unfused launches at the GPT-2 layer shape."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2502_19405_b200 as R  # noqa: E402

S_, H, T, hd = 8, 12, 512, 64
d = H * hd
qkv = torch.rand(S_ * T, 3 * d, device="cuda") - 0.5
Sb = torch.empty(S_ * H * T, T, device="cuda")
Pb = torch.empty_like(Sb)
O = torch.empty(S_ * T, d, device="cuda")


def fused():
    R.repops_attention_fwd(qkv, T, hd, 3 * d, (T * 3 * d, hd), 0, d, 2 * d, (S_, H), O, d, (T * d, hd), S=Sb, P=Pb,
                           sp=(H * T * T, T * T), scale=0.125)


def unfused():
    R.repops_gemm_strided_batched(qkv, qkv, Sb, M=T, N=T, K=hd, lda=3 * d, ldb=3 * d, ldc=T, sA=(T * 3 * d, hd),
                                  sB=(T * 3 * d, hd), sC=(H * T * T, T * T), batch=(S_, H), transB=True,
                                  epi=R.EPI_SCALE, scale=0.125, offB=d)
    R.repops_softmax(Sb, causal=True, out=Pb)
    R.repops_gemm_strided_batched(Pb, qkv, O, M=T, N=hd, K=T, lda=T, ldb=3 * d, ldc=d, sA=(H * T * T, T * T),
                                  sB=(T * 3 * d, hd), sC=(T * d, hd), batch=(S_, H), offB=2 * d)


def t(fn, n=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n


fl = 4 * S_ * H * T * T * hd
for name, fn in (("fused", fused), ("unfused", unfused)):
    ms = t(fn)
    print(f"{name:8s} {ms * 1e3:8.1f} us  {fl / ms / 1e9:6.1f} TFLOP/s")

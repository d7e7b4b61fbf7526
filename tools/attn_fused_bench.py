"""Fused attention forward (causal, scores scratch: S not stored, P stored for the
backward) vs the unfused launches the GPT-2 step runs (causal score-tile skip, softmax,
full PV), one GPT-2 layer (8 shards x 12 heads, T 512, hd 64); every variant, bits checked."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2502_19405_b200 as R  # noqa: E402

S_, H, T, hd = 8, 12, 512, 64
d = H * hd
torch.manual_seed(0)
qkv = torch.rand(S_ * T, 3 * d, device="cuda") - 0.5
Sb = torch.empty(S_ * H * T, T, device="cuda")
Pb = torch.empty_like(Sb)
Pf = torch.empty_like(Sb)
O = torch.empty(S_ * T, d, device="cuda")
Ou = torch.empty(S_ * T, d, device="cuda")


def fused():
    R.repops_attention_fwd(qkv, T, hd, 3 * d, (T * 3 * d, hd), 0, d, 2 * d, (S_, H), O, d, (T * d, hd), P=Pf,
                           sp=(H * T * T, T * T), scale=0.125)


def unfused():
    R.repops_gemm_strided_batched(qkv, qkv, Sb, M=T, N=T, K=hd, lda=3 * d, ldb=3 * d, ldc=T, sA=(T * 3 * d, hd),
                                  sB=(T * 3 * d, hd), sC=(H * T * T, T * T), batch=(S_, H), transB=True,
                                  epi=R.EPI_SCALE, scale=0.125, offB=d, causal=1)
    R.repops_softmax(Sb, causal=True, out=Pb)
    R.repops_gemm_strided_batched(Pb, qkv, Ou, M=T, N=hd, K=T, lda=T, ldb=3 * d, ldc=d, sA=(H * T * T, T * T),
                                  sB=(T * 3 * d, hd), sC=(T * d, hd), batch=(S_, H), offB=2 * d)


def probs_pv():
    R.repops_attention_probs(qkv, T, hd, 3 * d, (T * 3 * d, hd), 0, d, (S_, H), Pf, (H * T * T, T * T), scale=0.125)
    R.repops_gemm_strided_batched(Pf, qkv, O, M=T, N=hd, K=T, lda=T, ldb=3 * d, ldc=d, sA=(H * T * T, T * T),
                                  sB=(T * 3 * d, hd), sC=(T * d, hd), batch=(S_, H), offB=2 * d)


def probs_only():
    R.repops_attention_probs(qkv, T, hd, 3 * d, (T * 3 * d, hd), 0, d, (S_, H), Pf, (H * T * T, T * T), scale=0.125)


dO = torch.rand(S_ * T, d, device="cuda") - 0.5
dPb = torch.empty_like(Sb)
dSb = torch.empty_like(Sb)
dSf = torch.empty_like(Sb)


def bwd_unfused():
    R.repops_gemm_strided_batched(dO, qkv, dPb, M=T, N=T, K=hd, lda=d, ldb=3 * d, ldc=T, sA=(T * d, hd),
                                  sB=(T * 3 * d, hd), sC=(H * T * T, T * T), batch=(S_, H), transB=True, offB=2 * d)
    R.repops_softmax_backward(Pb, dPb, scale=0.125, out=dSb)


def bwd_fused():
    R.repops_attention_dscores(dO, qkv, T, hd, d, (T * d, hd), 0, 3 * d, (T * 3 * d, hd), 2 * d, Pb,
                               (H * T * T, T * T), dSf, (H * T * T, T * T), (S_, H), scale=0.125)


def t(fn, n=50):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n


fl = 4 * S_ * H * T * T * hd // 2   # causal half of QK^T and PV
ms = t(unfused)
print(f"unfused      {ms * 1e3:8.1f} us  {fl / ms / 1e9:6.1f} TFLOP/s (causal-half flops)")
for name, fn in (("probs+PV", probs_pv), ("probs only", probs_only)):
    ms = t(fn)
    same = torch.equal(O.view(torch.int32), Ou.view(torch.int32)) and torch.equal(Pf.view(torch.int32),
                                                                                  Pb.view(torch.int32))
    print(f"{name:12s} {ms * 1e3:8.1f} us  bits {'same' if same else 'DIFFER'}")
for v in (sys.argv[1:] or ["0", "1", "2", "3"]):
    os.environ["REPOPS_ATTN_VARIANT"] = v
    ms = t(fused)
    same = torch.equal(O.view(torch.int32), Ou.view(torch.int32)) and torch.equal(Pf.view(torch.int32),
                                                                                  Pb.view(torch.int32))
    print(f"fused v{v}     {ms * 1e3:8.1f} us  {fl / ms / 1e9:6.1f} TFLOP/s  bits {'same' if same else 'DIFFER'}")
ms = t(bwd_unfused)
print(f"bwd dP GEMM + softmax_bwd  {ms * 1e3:8.1f} us")
ms = t(bwd_fused)
same = torch.equal(dSf.view(torch.int32), dSb.view(torch.int32))
print(f"bwd dscores fused          {ms * 1e3:8.1f} us  bits {'same' if same else 'DIFFER'}")

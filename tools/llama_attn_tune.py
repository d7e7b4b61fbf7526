"""Llama-3-8B prefill attention R-GEMMs (8 blocks x 4 q-heads, T 2048, hd 128) per forced
tile configuration: causal scores (NT, mode 1) and causal PV (NN, mode 2); bits checked equal."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2502_19405_b200 as R  # noqa: E402
from paper_2502_19405_b200._lib import lib  # noqa: E402

nbl, qh, T, hd = 8, 4, 2048, 128
W2, Wb = (qh + 1) * hd, (qh + 2) * hd
qk = torch.rand(nbl, T, W2, device="cuda") - 0.5
qkv = torch.rand(nbl, T, Wb, device="cuda") - 0.5
S = torch.empty(nbl, qh * T, T, device="cuda")
P = torch.rand(nbl, qh * T, T, device="cuda")
P = P.view(-1, T)
P = R.repops_softmax(P, causal=True).view(nbl, qh * T, T)
o = torch.empty(nbl, T, qh * hd, device="cuda")
fl = torch.empty((nbl, T + 1, hd), dtype=torch.uint8, device="cuda")
R.repops_causal_suffix_flags(qkv, T, hd, Wb, (T * Wb, 0), (nbl, 1), out=fl, ldf=hd, sF=((T + 1) * hd, 0),
                             offB=(qh + 1) * hd)


def t_ms(fn, iters=5):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / iters


def run(name, fn, out, flops, cfgs, mask=None):
    res, ref = [], None
    for cfg in cfgs:
        lib().repops_gemm_force_cfg(cfg)
        try:
            ms = t_ms(fn)
        except Exception as e:  # noqa: BLE001
            res.append(f"cfg{cfg} err {str(e)[:40]}")
            continue
        torch.cuda.synchronize()
        c = out.clone()
        if mask is not None:   # causal mode 1: entries above the diagonal are never computed
            c = c.view(-1, T, T) * 0 + torch.where(mask, c.view(-1, T, T), torch.zeros_like(c.view(-1, T, T)))
        tag = ""
        if ref is None:
            ref = c
        elif not torch.equal(ref.view(torch.int32), c.view(torch.int32)):
            tag = " MISMATCH"
        res.append(f"cfg{cfg} {ms * 1e3:6.0f}us {flops / ms / 1e9:5.1f}{tag}")
    lib().repops_gemm_force_cfg(-1)
    print(name, " | ".join(res), flush=True)


half = 2 * nbl * qh * T * T * hd / 2
run("scores NT causal1", lambda: R.repops_gemm_strided_batched(
    qk, qk, S, M=T, N=T, K=hd, lda=W2, ldb=W2, ldc=T, sA=(T * W2, hd), sB=(T * W2, 0), sC=(qh * T * T, T * T),
    batch=(nbl, qh), transB=True, epi=R.EPI_SCALE, scale=0.088, offB=qh * hd, causal=1),
    S, half, [-1, 0, 1, 3, 4, 5, 6, 9, 2], mask=torch.ones(T, T, dtype=torch.bool, device="cuda").tril())
run("PV NN causal2", lambda: R.repops_gemm_strided_batched(
    P, qkv, o, M=T, N=hd, K=T, lda=T, ldb=Wb, ldc=qh * hd, sA=(qh * T * T, T * T), sB=(T * Wb, 0),
    sC=(T * qh * hd, hd), batch=(nbl, qh), offB=(qh + 1) * hd, causal=2, kflags=fl, ldf=hd,
    sF=((T + 1) * hd, 0)), o, half, [-1, 0, 1, 3, 5, 6, 10, 11, 13, 2])

# the fused scores + softmax kernel against the two launches it replaces
P2 = torch.empty_like(P)


def unfused():
    R.repops_gemm_strided_batched(qk, qk, S, M=T, N=T, K=hd, lda=W2, ldb=W2, ldc=T, sA=(T * W2, hd),
                                  sB=(T * W2, 0), sC=(qh * T * T, T * T), batch=(nbl, qh), transB=True,
                                  epi=R.EPI_SCALE, scale=0.088, offB=qh * hd, causal=1)
    R.repops_softmax(S.view(-1, T), causal=True, out=P.view(-1, T))


def fused():
    R.repops_attention_probs(qk, T, hd, W2, (T * W2, hd), 0, qh * hd, (nbl, qh), P2, (qh * T * T, T * T),
                             scale=0.088, causal=True, sk=(T * W2, 0))


mu, mf = t_ms(unfused), t_ms(fused)
same = torch.equal(P.view(torch.int32), P2.view(torch.int32))
print(f"scores+softmax unfused {mu * 1e3:6.0f} us | fused probs {mf * 1e3:6.0f} us | bits {'same' if same else 'DIFFER'}")

"""Batched attention-shaped R-GEMMs of the GPT-2 step (96 = 8 shards x 12 heads) per tile
configuration: scores as NT (Q, K row-major inside qkv) and as TN (Q^T, K^T slices of a
transposed qkv), dV / dK as TN with N = 64, PV / dQ as NN.  Bits are checked equal."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2502_19405_b200 as R
from paper_2502_19405_b200._lib import lib

S, H, T, hd, d = 8, 12, 512, 64, 768
qkv = torch.rand(S * T, 3 * d, device="cuda") - 0.5
qkvT = R.repops_transpose(qkv)  # [3d, S*T]
P = torch.rand(S * H * T, T, device="cuda")
dO = torch.rand(S * T, d, device="cuda") - 0.5


def t_ms(fn, iters=10):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / iters


def run(name, fn, flops, cfgs):
    outs = []
    for cfg in cfgs:
        lib().repops_gemm_force_cfg(cfg)
        ms = t_ms(fn)
        C = fn()
        torch.cuda.synchronize()
        outs.append(f"cfg{cfg} {flops / ms / 1e9:5.1f}")
        if cfg == cfgs[0]:
            ref = C.clone()
        elif not torch.equal(ref.view(torch.int32), C.view(torch.int32)):
            outs[-1] += " MISMATCH"
    lib().repops_gemm_force_cfg(-1)
    print(f"{name:28s}", " | ".join(outs), flush=True)


Sc = torch.empty(S * H * T, T, device="cuda")
fl = 2 * S * H * T * T * hd
run("scores NT (current)", lambda: R.repops_gemm_strided_batched(
    qkv, qkv, Sc, M=T, N=T, K=hd, lda=3 * d, ldb=3 * d, ldc=T, sA=(T * 3 * d, hd), sB=(T * 3 * d, hd),
    sC=(H * T * T, T * T), batch=(S, H), transB=True, epi=R.EPI_SCALE, scale=0.125, offB=d), fl, [-1, 6, 5, 2])
run("scores TN (qkv^T slices)", lambda: R.repops_gemm_strided_batched(
    qkvT, qkvT, Sc, M=T, N=T, K=hd, lda=S * T, ldb=S * T, ldc=T, sA=(T, hd * S * T), sB=(T, hd * S * T),
    sC=(H * T * T, T * T), batch=(S, H), transA=True, epi=R.EPI_SCALE, scale=0.125, offB=d * S * T), fl,
    [-1, 20, 22, 24, 6])
dV = torch.empty(S * T, 3 * d, device="cuda")
run("dV TN N=64", lambda: R.repops_gemm_strided_batched(
    P, dO, dV, M=T, N=hd, K=T, lda=T, ldb=d, ldc=3 * d, sA=(H * T * T, T * T), sB=(T * d, hd),
    sC=(T * 3 * d, hd), batch=(S, H), transA=True, offC=2 * d), fl, [-1, 5, 24, 22, 1])
att = torch.empty(S * T, d, device="cuda")
run("PV NN N=64", lambda: R.repops_gemm_strided_batched(
    P, qkv, att, M=T, N=hd, K=T, lda=T, ldb=3 * d, ldc=d, sA=(H * T * T, T * T), sB=(T * 3 * d, hd),
    sC=(T * d, hd), batch=(S, H), offB=2 * d), fl, [-1, 5, 11, 1, 13])

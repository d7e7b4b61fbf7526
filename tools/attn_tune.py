"""Time the GPT-2 step's six attention GEMMs (batched over 8 shards x 12 heads)
for every tile configuration in CFGS and check bit-identity across configs."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2502_19405_b200 as R
from paper_2502_19405_b200._lib import lib

S_loc, H, T, d = 8, 12, 512, 768
hd = d // H
torch.manual_seed(0)
qkv = torch.rand(S_loc * T, 3 * d, device="cuda") - 0.5
att = torch.rand(S_loc * T, d, device="cuda") - 0.5
P = torch.rand(S_loc * H * T, T, device="cuda")
out_S = torch.empty(S_loc * H * T, T, device="cuda")
out_o = torch.empty(S_loc * T, d, device="cuda")
out_q = torch.empty(S_loc * T, 3 * d, device="cuda")

CALLS = {
    "S=QK^T (NT)": lambda cfg: R.repops_gemm_strided_batched(
        qkv, qkv, out_S, M=T, N=T, K=hd, lda=3 * d, ldb=3 * d, ldc=T, sA=(T * 3 * d, hd), sB=(T * 3 * d, hd),
        sC=(H * T * T, T * T), batch=(S_loc, H), transB=True, epi=R.EPI_SCALE, scale=0.125, offB=d),
    "O=PV (NN)": lambda cfg: R.repops_gemm_strided_batched(
        P, qkv, out_o, M=T, N=hd, K=T, lda=T, ldb=3 * d, ldc=d, sA=(H * T * T, T * T), sB=(T * 3 * d, hd),
        sC=(T * d, hd), batch=(S_loc, H), offB=2 * d),
    "dP=dO V^T (NT)": lambda cfg: R.repops_gemm_strided_batched(
        att, qkv, out_S, M=T, N=T, K=hd, lda=d, ldb=3 * d, ldc=T, sA=(T * d, hd), sB=(T * 3 * d, hd),
        sC=(H * T * T, T * T), batch=(S_loc, H), transB=True, offB=2 * d),
    "dV=P^T dO (TN)": lambda cfg: R.repops_gemm_strided_batched(
        P, att, out_q, M=T, N=hd, K=T, lda=T, ldb=d, ldc=3 * d, sA=(H * T * T, T * T), sB=(T * d, hd),
        sC=(T * 3 * d, hd), batch=(S_loc, H), transA=True, offC=2 * d),
    "dQ=dS K (NN)": lambda cfg: R.repops_gemm_strided_batched(
        P, qkv, out_q, M=T, N=hd, K=T, lda=T, ldb=3 * d, ldc=3 * d, sA=(H * T * T, T * T), sB=(T * 3 * d, hd),
        sC=(T * 3 * d, hd), batch=(S_loc, H), offB=d),
}
cfgs = [int(x) for x in os.environ.get("CFGS", "-1,1,5,6,10,11,13").split(",")]
flops = 2 * S_loc * H * T * T * hd
for name, fn in CALLS.items():
    res, ref = [], None
    for cfg in cfgs:
        lib().repops_gemm_force_cfg(cfg)
        c = None
        for _ in range(2):
            fn(c)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(10):
            fn(c)
        b.record()
        torch.cuda.synchronize()
        ms = a.elapsed_time(b) / 10
        outbuf = out_S if "S" in name.split("=")[0] or name.startswith("dP") else (out_o if "O=" in name else out_q)
        h = outbuf.view(torch.int32).sum().item()
        ref = h if ref is None else ref
        res.append(f"{'auto' if cfg < 0 else 'cfg%d' % cfg} {ms * 1e3:6.1f}us {flops / ms / 1e9:5.1f}"
                   + ("" if h == ref else " MISMATCH"))
    print(f"{name:16s} " + " | ".join(res), flush=True)

"""The GPT-2 step's batched attention GEMMs (96 = 8 shards x 12 heads) a few times each,
for ncu captures: scores (NT, causal tile skip), PV (NN), dV (TN)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2502_19405_b200 as R

S, H, T, hd = 8, 12, 512, 64
d = H * hd
qkv = torch.rand(S * T, 3 * d, device="cuda") - 0.5
Sc = torch.empty(S * H * T, T, device="cuda")
P = torch.rand(S * H * T, T, device="cuda")
att = torch.empty(S * T, d, device="cuda")
dq = torch.empty(S * T, 3 * d, device="cuda")
for _ in range(3):
    R.repops_gemm_strided_batched(qkv, qkv, Sc, M=T, N=T, K=hd, lda=3 * d, ldb=3 * d, ldc=T, sA=(T * 3 * d, hd),
                                  sB=(T * 3 * d, hd), sC=(H * T * T, T * T), batch=(S, H), transB=True,
                                  epi=R.EPI_SCALE, scale=0.125, offB=d, causal=1)
    R.repops_gemm_strided_batched(P, qkv, att, M=T, N=hd, K=T, lda=T, ldb=3 * d, ldc=d, sA=(H * T * T, T * T),
                                  sB=(T * 3 * d, hd), sC=(T * d, hd), batch=(S, H), offB=2 * d)
    R.repops_gemm_strided_batched(P, att, dq, M=T, N=hd, K=T, lda=T, ldb=d, ldc=3 * d, sA=(H * T * T, T * T),
                                  sB=(T * d, hd), sC=(T * 3 * d, hd), batch=(S, H), transA=True, offC=2 * d)
torch.cuda.synchronize()

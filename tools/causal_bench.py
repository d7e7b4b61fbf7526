"""GPT-2 / Llama attention launches with and without the exact causal structure (R31):
scores (mode 1), V suffix flags, PV (mode 2) -- per-launch device times."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2502_19405_b200 as R


def t_us(fn, iters=20):
    for _ in range(3): fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(iters): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / iters * 1e3


for (S, H, T, hd) in ((8, 12, 512, 64), (1, 32, 2048, 128)):
    d = H * hd
    qkv = torch.rand(S * T, 3 * d, device="cuda") - 0.5
    Sc = torch.empty(S * H * T, T, device="cuda")
    P = torch.empty(S * H * T, T, device="cuda")
    att = torch.empty(S * T, d, device="cuda")
    fl = torch.empty((S * H, T + 1, hd), dtype=torch.uint8, device="cuda")
    sc = lambda c: R.repops_gemm_strided_batched(qkv, qkv, Sc, M=T, N=T, K=hd, lda=3 * d, ldb=3 * d, ldc=T,  # noqa
                                                 sA=(T * 3 * d, hd), sB=(T * 3 * d, hd), sC=(H * T * T, T * T),
                                                 batch=(S, H), transB=True, epi=R.EPI_SCALE, scale=0.125, offB=d,
                                                 causal=c)
    flags = lambda: R.repops_causal_suffix_flags(qkv, T, hd, 3 * d, (T * 3 * d, hd), (S, H), out=fl, ldf=hd,  # noqa
                                                 sF=(H * (T + 1) * hd, (T + 1) * hd), offB=2 * d)
    pv = lambda c: R.repops_gemm_strided_batched(P, qkv, att, M=T, N=hd, K=T, lda=T, ldb=3 * d, ldc=d,  # noqa
                                                 sA=(H * T * T, T * T), sB=(T * 3 * d, hd), sC=(T * d, hd),
                                                 batch=(S, H), offB=2 * d, causal=c, kflags=fl, ldf=hd,
                                                 sF=(H * (T + 1) * hd, (T + 1) * hd))
    sc(0)
    R.repops_softmax(Sc, causal=True, out=P)
    flags()
    print(f"S={S} H={H} T={T} hd={hd}: scores full {t_us(lambda: sc(0)):7.1f} us, causal {t_us(lambda: sc(1)):7.1f} us;"
          f" flags {t_us(flags):6.1f} us; PV full {t_us(lambda: pv(0)):7.1f} us, causal {t_us(lambda: pv(2)):7.1f} us",
          flush=True)

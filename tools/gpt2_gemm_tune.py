"""Time every R-GEMM tile configuration on the GEMM shapes of the GPT-2 step
(batched shapes as in the step), check bits-neutrality, print the best cfg."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2502_19405_b200 as R  # noqa: E402
from paper_2502_19405_b200._lib import check, lib  # noqa: E402

NCFG = int(os.environ.get("NCFG", "7"))
T, d, F, V, Vld, H, hd, S = 512, 768, 3072, 50257, 50304, 12, 64, 8
M = S * T
# name, M, N, K, tA, tB, lda, ldb, ldc, batch(b0,b1), strides
SHAPES = [
    ("qkv fwd", M, 3 * d, d, 0, 0, d, 3 * d, 3 * d, (1, 1)),
    ("proj fwd", M, d, d, 0, 0, d, d, d, (1, 1)),
    ("fc fwd", M, F, d, 0, 0, d, F, F, (1, 1)),
    ("fc2 fwd", M, d, F, 0, 0, F, d, d, (1, 1)),
    ("lm head", M, V, d, 0, 1, d, d, Vld, (1, 1)),
    ("lm dgrad", M, d, V, 0, 0, Vld, d, d, (1, 1)),
    ("lm wgrad x8", V, d, T, 1, 0, Vld, d, d, (S, 1)),
    ("fc2 dgrad", M, F, d, 0, 1, d, d, F, (1, 1)),
    ("fc2 wgrad x8", F, d, T, 1, 0, F, d, d, (S, 1)),
    ("fc dgrad", M, d, F, 0, 1, F, F, d, (1, 1)),
    ("fc wgrad x8", d, F, T, 1, 0, d, F, F, (S, 1)),
    ("proj dgrad", M, d, d, 0, 1, d, d, d, (1, 1)),
    ("proj wgrad x8", d, d, T, 1, 0, d, d, d, (S, 1)),
    ("qkv dgrad", M, d, 3 * d, 0, 1, 3 * d, 3 * d, d, (1, 1)),
    ("qkv wgrad x8", d, 3 * d, T, 1, 0, d, 3 * d, 3 * d, (S, 1)),
    ("scores NT x96", T, T, hd, 0, 1, 3 * d, 3 * d, T, (S, H)),
    ("pv NN x96", T, hd, T, 0, 0, T, 3 * d, d, (S, H)),
    ("dP NT x96", T, T, hd, 0, 1, d, 3 * d, T, (S, H)),
    ("dV TN x96", T, hd, T, 1, 0, T, d, 3 * d, (S, H)),
    ("dQ NN x96", T, hd, T, 0, 0, T, 3 * d, 3 * d, (S, H)),
]


def t_ms(fn, iters=5, warm=2):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(iters):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / iters


total_best, total_auto = 0.0, 0.0
for name, m, n, k, ta, tb, lda, ldb, ldc, (b0, b1) in SHAPES:
    # operand storage sized generously for the strided batch
    a_rows = (k if ta else m)
    b_rows = (n if tb else k)
    sA = (a_rows * lda * b1, 0) if b1 == 1 else (T * lda, hd)
    sB = (b_rows * ldb * b1, 0) if b1 == 1 else (T * ldb, hd)
    sC = (m * ldc, 0) if b1 == 1 else (H * T * T if ldc == T else T * ldc, T * T if ldc == T else hd)
    A = torch.rand(b0 * b1 * a_rows * lda + lda * a_rows, device="cuda")
    B = torch.rand(b0 * b1 * b_rows * ldb + ldb * b_rows, device="cuda")
    C = torch.empty(b0 * b1 * m * ldc + m * ldc, device="cuda")
    res = []

    def run(cfg):
        if cfg is None:
            return R.repops_gemm_strided_batched(A, B, C, m, n, k, lda, ldb, ldc, sA, sB, sC, (b0, b1),
                                                 transA=bool(ta), transB=bool(tb))
        # forced configuration through the test hook, one problem at a time is not
        # representative; use the batched entry with cfg via environment
        os.environ["REPOPS_GEMM_CFG"] = str(cfg)
        return R.repops_gemm_strided_batched(A, B, C, m, n, k, lda, ldb, ldc, sA, sB, sC, (b0, b1),
                                             transA=bool(ta), transB=bool(tb))
    flops = 2 * m * n * k * b0 * b1
    auto = t_ms(lambda: run(None))
    best = (1e9, -1)
    for cfg in range(NCFG):
        check(lib().repops_gemm_force_cfg(cfg), "force")
        ms = t_ms(lambda: run(None))
        check(lib().repops_gemm_force_cfg(-1), "force")
        res.append(f"c{cfg} {flops / ms / 1e9:5.1f}")
        best = min(best, (ms, cfg))
    total_best += best[0]
    total_auto += auto
    print(f"{name:15s} auto {flops / auto / 1e9:5.1f} | " + " ".join(res) + f" | best c{best[1]}", flush=True)
print(f"sum over one instance of each shape: auto {total_auto:.2f} ms, best {total_best:.2f} ms")

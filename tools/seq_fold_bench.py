"""R-SEQ column folds at the GPT-2 step's shapes (bias / LayerNorm parameter gradients
per shard): CUDA-event time per launch and effective GB/s."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2502_19405_b200 as R  # noqa: E402


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


for cols in (768, 2304, 3072):
    x = torch.rand(4096, cols, device="cuda")
    out = torch.empty(8, cols, device="cuda")
    ms = t(lambda: R.repops_sum_cols_seq(x, nseg=8, out=out))
    print(f"sum_cols_seq 4096x{cols}: {ms * 1e3:7.1f} us  {x.numel() * 4 / ms / 1e6:7.1f} GB/s")
dy = torch.rand(4096, 768, device="cuda")
x = torch.rand(4096, 768, device="cuda")
mu, rs = torch.rand(4096, device="cuda"), torch.rand(4096, device="cuda")
dg, db = torch.empty(8, 768, device="cuda"), torch.empty(8, 768, device="cuda")
ms = t(lambda: R.repops_layernorm_backward_params(dy, x, mu, rs, nseg=8, dgamma=dg, dbeta=db))
print(f"layernorm_params 4096x768: {ms * 1e3:7.1f} us  {2 * dy.numel() * 4 / ms / 1e6:7.1f} GB/s")

# row operators of the GPT-2 step: causal softmax over the [8 x 12 x 512, 512] scores
S = torch.rand(8 * 12 * 512, 512, device="cuda") * 8 - 4
Pm = torch.empty_like(S)
ms = t(lambda: R.repops_softmax(S, causal=True, out=Pm))
print(f"softmax causal 49152x512: {ms * 1e3:7.1f} us  {2 * S.numel() * 4 / ms / 1e6:7.1f} GB/s (algorithmic)")
X = torch.rand(4096, 768, device="cuda")
g_, b_ = torch.rand(768, device="cuda"), torch.rand(768, device="cuda")
ms = t(lambda: R.repops_layernorm(X, g_, b_))
print(f"layernorm 4096x768: {ms * 1e3:7.1f} us  {2 * X.numel() * 4 / ms / 1e6:7.1f} GB/s (algorithmic)")
logits = torch.rand(4096, 50304, device="cuda") * 8 - 4
labels = torch.randint(0, 50257, (4096,), dtype=torch.int32, device="cuda")
dl = torch.empty_like(logits)
lo = torch.empty(4096, device="cuda")
ms = t(lambda: R.repops_cross_entropy(logits, labels, scale=2.0 ** -12, loss=lo, dlogits=dl, V=50257), n=5)
print(f"cross_entropy 4096x50257: {ms * 1e3:7.1f} us  {2 * 4096 * 50257 * 4 / ms / 1e6:7.1f} GB/s (algorithmic)")
for rows, cols in ((4096, 768), (4096, 3072), (4096, 2304)):
    X = torch.rand(rows, cols, device="cuda")
    Y = torch.empty(cols, rows, device="cuda")
    ms = t(lambda: R.repops_transpose(X, out=Y))
    print(f"transpose {rows}x{cols}: {ms * 1e3:7.1f} us  {2 * X.numel() * 4 / ms / 1e6:7.1f} GB/s")

"""Cross entropy at the GPT-2 head shape: the shared-memory-row kernel (16-byte aligned
rows) against the three-pass CTA kernel (taken for unaligned rows)."""
import os
import sys, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2502_19405_b200 as R
def t(fn, n=5):
    for _ in range(2): fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n): fn()
    b.record(); torch.cuda.synchronize()
    return a.elapsed_time(b) / n
big = torch.rand(4096, 50305, device="cuda") * 8 - 4
al = big[:, :50304]          # aligned rows? ld 50305 -> not 16B aligned -> old kernel
lab = torch.randint(0, 50257, (4096,), dtype=torch.int32, device="cuda")
dl = torch.empty(4096, 50304, device="cuda"); lo = torch.empty(4096, device="cuda")
print("old (unaligned ld):", t(lambda: R.repops_cross_entropy(al, lab, scale=2.0**-12, loss=lo, dlogits=dl, V=50257)) * 1e3, "us")
al2 = torch.rand(4096, 50304, device="cuda") * 8 - 4
print("new (aligned):", t(lambda: R.repops_cross_entropy(al2, lab, scale=2.0**-12, loss=lo, dlogits=dl, V=50257)) * 1e3, "us")

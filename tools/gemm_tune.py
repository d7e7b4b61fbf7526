"""Time every R-GEMM tile configuration (all bits-neutral) on the GPU and check
that their outputs are bit-identical.  Prints one line per (shape, layout, cfg)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2502_19405_b200 as R  # noqa: E402


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


shapes = [(8192, 8192, 8192), (4096, 4096, 4096), (4096, 2304, 768), (768, 2304, 512), (4096, 768, 3072),
          (512, 512, 64)]
if len(sys.argv) > 1:
    shapes = [tuple(int(x) for x in s.split("x")) for s in sys.argv[1].split(",")]
ncfg = int(os.environ.get("NCFG", "6"))
cfgs = [int(x) for x in os.environ["CFGS"].split(",")] if "CFGS" in os.environ else list(range(ncfg))
layouts = [tuple(int(c) for c in x) for x in os.environ.get("LAYOUTS", "00,01,10").split(",")]
torch.manual_seed(0)
for (M, N, K) in shapes:
    for ta, tb in layouts:
        A = (torch.rand((K, M) if ta else (M, K), device="cuda") * 2 - 1)
        B = (torch.rand((N, K) if tb else (K, N), device="cuda") * 2 - 1)
        C0 = torch.empty(M, N, device="cuda")
        R.repops_gemm(A, B, transA=bool(ta), transB=bool(tb), out=C0, cfg=0)
        res = []
        for cfg in cfgs:
            C = torch.empty(M, N, device="cuda")
            ms = t_ms(lambda: R.repops_gemm(A, B, transA=bool(ta), transB=bool(tb), out=C, cfg=cfg))
            same = torch.equal(C.view(torch.int32), C0.view(torch.int32))
            res.append(f"cfg{cfg} {2 * M * N * K / ms / 1e9:6.1f}{'' if same else ' MISMATCH'}")
        torch.backends.cuda.matmul.allow_tf32 = False
        Ab = A.t() if ta else A
        Bb = B.t() if tb else B
        ms = t_ms(lambda: torch.mm(Ab, Bb))
        print(f"{M}x{N}x{K} tA{ta} tB{tb}: " + " | ".join(res) + f" | cublas {2 * M * N * K / ms / 1e9:6.1f} TFLOP/s",
              flush=True)

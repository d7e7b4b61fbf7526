"""Per-shape R-GEMM time inside the GPT-2 step (commit off): which GEMMs are below the
FP32 roofline.  Wraps the GEMM entry points the step program calls and brackets each
launch with CUDA events on the current stream.  Usage: python tools/gpt2_gemm_shapes.py"""
import collections
import inspect
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2502_19405_b200 as R  # noqa: E402
import paper_2502_19405_b200.gpt2 as G  # noqa: E402

REC = []


def wrap(fn, kind):
    def f(*a, **kw):
        if kind == "gemm":
            A, B = a[0], a[1]
            tA, tB = kw.get("transA", False), kw.get("transB", False)
            M = A.shape[1] if tA else A.shape[0]
            K = A.shape[0] if tA else A.shape[1]
            N = B.shape[0] if tB else B.shape[1]
            key, fl = (f"{'T' if tA else 'N'}{'T' if tB else 'N'} {M}x{N}x{K}"), 2 * M * N * K
        else:
            ba = inspect.signature(fn).bind(*a, **kw)
            ba.apply_defaults()
            M, N, K, b = ba.arguments["M"], ba.arguments["N"], ba.arguments["K"], ba.arguments["batch"]
            tA, tB = ba.arguments["transA"], ba.arguments["transB"]
            key = f"{'T' if tA else 'N'}{'T' if tB else 'N'} {M}x{N}x{K} x{b[0] * b[1]}"
            fl = 2 * M * N * K * b[0] * b[1]
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        r = fn(*a, **kw)
        e.record()
        REC.append((key, fl, s, e))
        return r
    return f


if os.environ.get("FORCE_CFG"):
    from paper_2502_19405_b200._lib import check, lib
    check(lib().repops_gemm_force_cfg(int(os.environ["FORCE_CFG"])), "force")
G.repops_gemm = wrap(R.repops_gemm, "gemm")
G.repops_gemm_strided_batched = wrap(R.repops_gemm_strided_batched, "batched")
st = G.GPT2Step(G.GPT2Config())
st.set_tokens(0)
for _ in range(2):
    st.run(commit=False)
torch.cuda.synchronize()
REC.clear()
st.run(commit=False)
torch.cuda.synchronize()
agg = collections.defaultdict(lambda: [0.0, 0, 0])
for key, fl, s, e in REC:
    a = agg[key]
    a[0] += s.elapsed_time(e)
    a[1] += fl
    a[2] += 1
tot = sum(v[0] for v in agg.values())
print(f"{'shape':34s} {'n':>4s} {'ms':>8s} {'share':>6s} {'TFLOP/s':>8s}")
for key, (ms, fl, n) in sorted(agg.items(), key=lambda kv: -kv[1][0]):
    print(f"{key:34s} {n:4d} {ms:8.3f} {ms / tot:6.1%} {fl / ms / 1e9:8.1f}")
print(f"total {tot:.2f} ms, {sum(v[1] for v in agg.values()) / tot / 1e9:.1f} TFLOP/s")

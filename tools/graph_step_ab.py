"""GPT-2 headline step (every output committed) eager vs replayed from one captured CUDA
graph: device time per step and the step root after the same number of steps."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2502_19405_b200.gpt2 import GPT2Config, GPT2Step  # noqa: E402

N = 10


def timed(fn, n=N):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n


roots = {}
for mode in sys.argv[1:] or ["eager", "graph"]:
    st = GPT2Step(GPT2Config())
    st.set_tokens(0)
    hi = torch.cuda.Stream(priority=-1)
    with torch.cuda.stream(hi):
        for _ in range(3):
            st.run(commit=True)
        torch.cuda.synchronize()
        if mode == "eager":
            ms = timed(lambda: st.run(commit=True))
        else:
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=hi):
                st.run(commit=True)
            torch.cuda.synchronize()
            ms = timed(g.replay)
        roots[mode] = st.device_root().hex()[:16]
    print(f"{mode:6s} {ms:8.2f} ms/step  root after {3 + N} steps {roots[mode]}", flush=True)
    del st
    torch.cuda.empty_cache()

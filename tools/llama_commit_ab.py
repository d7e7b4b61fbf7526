"""Llama-3-8B-shaped prefill (config 4): where the commitments run -- side stream beside the
next phases, inline on the pass stream, or all after the last phase -- and the pass without
commitments; device time per pass (CUDA events), same root in every committed mode."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_2502_19405_b200.llama import LlamaConfig, LlamaPrefill  # noqa: E402

st = LlamaPrefill(LlamaConfig())
st.load_weights()
st.set_tokens()
hi = torch.cuda.Stream(priority=-1)
for mode in sys.argv[1:] or ["side", "inline", "end", "none"]:
    with torch.cuda.stream(hi):
        for _ in range(2):
            st.run(commit=mode != "none", commit_mode=mode if mode != "none" else "side")
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        n = 3
        for _ in range(n):
            st.run(commit=mode != "none", commit_mode=mode if mode != "none" else "side")
        b.record()
        torch.cuda.synchronize()
        root = st.device_root().hex()[:16] if mode != "none" else "-"
    print(f"{mode:7s} {a.elapsed_time(b) / n:8.1f} ms/pass  root {root}", flush=True)

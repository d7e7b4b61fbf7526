"""One Llama-3-8B-shaped prefill pass (config 4) after a warm-up pass -- for ncu launch lists."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2502_19405_b200.llama import LlamaConfig, LlamaPrefill
st = LlamaPrefill(LlamaConfig())
st.load_weights()
st.set_tokens()
for _ in range(2):
    st.run()
    st.device_root()
torch.cuda.synchronize()

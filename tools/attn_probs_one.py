"""One GPT-2 layer's repops_attention_probs launch (8 shards x 12 heads, T 512, hd 64) for ncu."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2502_19405_b200 as R  # noqa: E402

S_, H, T, hd = 8, 12, 512, 64
d = H * hd
qkv = torch.rand(S_ * T, 3 * d, device="cuda") - 0.5
P = torch.empty(S_ * H * T, T, device="cuda")
for _ in range(3):
    R.repops_attention_probs(qkv, T, hd, 3 * d, (T * 3 * d, hd), 0, d, (S_, H), P, (H * T * T, T * T), scale=0.125)
torch.cuda.synchronize()

"""Dev tool: one block-wise attention launch at a mid-size shape (for ncu)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
import paper_2507_19823_b200 as hc
n, Hq, Hkv, d, bs = 32768, 32, 8, 128, 4096
q = torch.randn((n, Hq, d), device="cuda").half() * 0.5
k = torch.randn((n, Hkv, d), device="cuda").half() * 0.5
v = torch.randn((n, Hkv, d), device="cuda").half()
for _ in range(3):
    out = hc.blockwise_attention(q, k, v, bs)
torch.cuda.synchronize()
print("ok")

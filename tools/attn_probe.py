import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2202_01306_b200 import ops
B, S, H = 4, 1024, 25
d = H * 64
qkv = torch.randn(B * S, 3 * d, device="cuda").to(torch.bfloat16)
out = torch.empty(B * S, d, device="cuda", dtype=torch.bfloat16)
lse = torch.empty(B * S, H, device="cuda")
for _ in range(3):
    ops.attn_fwd_tc(qkv, out, lse, batch=B, seq=S, heads=H, head_dim=64, causal=True)
torch.cuda.synchronize()

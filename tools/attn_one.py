import sys, torch
sys.path.insert(0, '.')
from paper_2202_01306_b200 import ops
B, S, H, DH = 4, 1024, 25, 64
d = H * DH
qkv = torch.randn(B * S, 3 * d, device="cuda").to(torch.bfloat16)
out = torch.empty(B * S, d, device="cuda", dtype=torch.bfloat16)
lse = torch.empty(B * S, H, device="cuda")
dout = torch.randn(B * S, d, device="cuda").to(torch.bfloat16)
dqkv = torch.empty_like(qkv)
for _ in range(3):
    ops.attn_fwd(qkv, out, lse, batch=B, seq=S, heads=H, head_dim=DH, causal=True)
    ops.attn_bwd(qkv, out, dout, lse, dqkv, batch=B, seq=S, heads=H, head_dim=DH, causal=True)
torch.cuda.synchronize()

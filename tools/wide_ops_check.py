import math, torch, json, sys, os
sys.path.insert(0, os.getcwd())
from paper_2202_01306_b200 import ops
torch.manual_seed(0)
def bf(*s, scale=1.0): return (torch.randn(*s, device="cuda") * scale).to(torch.bfloat16)
def rel(a, b): return ((a.float() - b.float()).norm() / b.float().norm()).item()
M, d = 256, 8192
for (N, K, epi) in [(3 * d, d, "bf16"), (d, d, "resid_f32"), (4 * d, d, "gelu_bf16"), (d, 4 * d, "resid_f32"), (1024, d, "f32")]:
    a, b = bf(M, K), bf(N, K, scale=0.02)
    bias = torch.randn(N, device="cuda") * 0.1
    acc = a.float() @ b.float().t()
    out = {}
    if epi == "bf16":
        dd = torch.empty(M, N, device="cuda", dtype=torch.bfloat16); ops.gemm(a, b, dd, epi="bf16", bias=bias); ref = acc + bias
    elif epi == "f32":
        dd = torch.empty(M, N, device="cuda"); ops.gemm(a, b, dd, epi="f32"); ref = acc
    elif epi == "resid_f32":
        r = torch.randn(M, N, device="cuda"); dd = torch.empty(M, N, device="cuda"); ops.gemm(a, b, dd, epi="resid_f32", bias=bias, aux=r); ref = r + acc + bias
    else:
        p = torch.empty(M, N, device="cuda", dtype=torch.bfloat16); dd = torch.empty_like(p); ops.gemm(a, b, dd, epi="gelu_bf16", bias=bias, aux=p); ref = torch.nn.functional.gelu(acc + bias, approximate="tanh")
    torch.cuda.synchronize()
    print(json.dumps({"gemm": [M, N, K, epi], "tile": ops.gemm_tile(M, N, K, epi), "rel": rel(dd, ref)}))
# dgrad / wgrad shapes
for (Mx, N, K, amn, bmn, epi) in [(256, d, 3 * d, 0, 1, "f32"), (256, d, 4 * d, 0, 1, "f32"), (3 * d, d, 256, 1, 1, "acc_f32"), (d, 4 * d, 256, 1, 1, "acc_f32")]:
    a = bf(K, Mx) if amn else bf(Mx, K)
    b = bf(K, N) if bmn else bf(N, K)
    A = a.float().t() if amn else a.float(); B = b.float() if bmn else b.float().t()
    dd = torch.randn(Mx, N, device="cuda") if epi == "acc_f32" else torch.empty(Mx, N, device="cuda")
    ref = (dd.clone() if epi == "acc_f32" else 0) + A @ B
    ops.gemm(a, b, dd, a_mn=bool(amn), b_mn=bool(bmn), epi=epi)
    torch.cuda.synchronize()
    print(json.dumps({"gemm": [Mx, N, K, amn, bmn, epi], "tile": ops.gemm_tile(Mx, N, K, epi), "rel": rel(dd, ref)}))
# attention
B, S, H, DH = 1, 256, 64, 128
qkv = bf(B * S, 3 * H * DH)
o = torch.empty(B * S, H * DH, device="cuda", dtype=torch.bfloat16); lse = torch.empty(B * S, H, device="cuda")
ops.attn_fwd(qkv, o, lse, batch=B, seq=S, heads=H, head_dim=DH, causal=True)
q, k, v = qkv.float().view(B, S, 3, H, DH).permute(2, 0, 3, 1, 4)
s = (q @ k.transpose(-1, -2)) / math.sqrt(DH)
s = s.masked_fill(torch.triu(torch.ones(S, S, device="cuda", dtype=torch.bool), 1), float("-inf"))
ref = (torch.softmax(s, -1) @ v).permute(0, 2, 1, 3).reshape(B * S, H * DH)
torch.cuda.synchronize()
print(json.dumps({"attn": [B, S, H, DH], "rel": rel(o, ref)}))
# layernorm
x = torch.randn(M, d, device="cuda"); g = torch.randn(d, device="cuda"); bb = torch.randn(d, device="cuda")
y = torch.empty(M, d, device="cuda", dtype=torch.bfloat16); mu = torch.empty(M, device="cuda"); rs = torch.empty(M, device="cuda")
ops.layernorm_fwd(x, g, bb, y, mu, rs) if hasattr(ops, "layernorm_fwd") else None
print(json.dumps({"ln": rel(y, torch.nn.functional.layer_norm(x, (d,), g, bb, 1e-5))}))

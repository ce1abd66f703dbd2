"""Numerics of the sm_100a kernels against plain PyTorch fp32 references of
the same op (run on the B200 box: pytest -m gpu)."""

import math

import numpy as np

import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ops():
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2202_01306_b200 import ops as O
    return O


def _bf(*shape, scale=1.0):
    return (torch.randn(*shape, device="cuda") * scale).to(torch.bfloat16)


def _rel(a, b):
    return ((a.float() - b.float()).norm() / (b.float().norm() + 1e-30)).item()


@pytest.mark.parametrize("M,N,K", [(128, 128, 64), (256, 256, 128), (512, 1600, 1600), (4096, 4800, 1600),
                                   (384, 4096, 256), (200, 136, 192), (1024, 50304, 256)])
def test_gemm_fwd_kk(ops, M, N, K):
    torch.manual_seed(0)
    a, b = _bf(M, K), _bf(N, K)
    d = torch.empty(M, N, device="cuda")
    ops.gemm(a, b, d, epi="f32")
    ref = a.float() @ b.float().t()
    torch.cuda.synchronize()
    assert _rel(d, ref) < 1e-5


@pytest.mark.parametrize("M,N,K", [(256, 128, 128), (512, 1600, 6400), (4096, 1600, 1600), (320, 192, 128)])
def test_gemm_dgrad_k_mn(ops, M, N, K):
    """dX[M,N] = dY[M,K] . W[K,N]  (W stored [out=K, in=N], B MN-major)."""
    torch.manual_seed(1)
    dy, w = _bf(M, K), _bf(K, N)
    d = torch.empty(M, N, device="cuda")
    ops.gemm(dy, w, d, b_mn=True, epi="f32")
    assert _rel(d, dy.float() @ w.float()) < 1e-5


@pytest.mark.parametrize("O,I,T", [(128, 128, 128), (1600, 1600, 4096), (4800, 1600, 1024), (6400, 1600, 512),
                                   (200, 136, 256), (1000, 392, 8192)])
def test_gemm_wgrad_mn_mn_accumulate(ops, O, I, T):
    """dW[O,I] += dY[T,O]^T . X[T,I]  (both MN-major), fp32 accumulate.
    (1600, 1600, 4096) and (1000, 392, 8192) run split-K (3- and 8-way, the
    second with M/N tails): partial sums meet in the TMA reduce-add."""
    torch.manual_seed(2)
    dy, x = _bf(T, O), _bf(T, I)
    dw = torch.randn(O, I, device="cuda")
    ref = dw + dy.float().t() @ x.float()
    ops.gemm(dy, x, dw, a_mn=True, b_mn=True, epi="acc_f32")
    assert _rel(dw, ref) < 1e-5


def test_gemm_epilogues(ops):
    torch.manual_seed(3)
    M, N, K = 512, 1600, 512
    a, b = _bf(M, K), _bf(N, K, scale=0.05)
    bias = torch.randn(N, device="cuda")
    acc = a.float() @ b.float().t()
    d = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    ops.gemm(a, b, d, epi="bf16", bias=bias)
    assert _rel(d, acc + bias) < 1e-2
    r = torch.randn(M, N, device="cuda")
    d32 = torch.empty(M, N, device="cuda")
    ops.gemm(a, b, d32, epi="resid_f32", bias=bias, aux=r)
    assert _rel(d32, r + acc + bias) < 1e-5
    p = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    g = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    ops.gemm(a, b, g, epi="gelu_bf16", bias=bias, aux=p)
    pre = acc + bias
    assert _rel(p, pre) < 1e-2
    assert _rel(g, torch.nn.functional.gelu(pre, approximate="tanh")) < 1e-2
    dg = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    ops.gemm(a, b, dg, epi="dgelu_bf16", aux=p)
    x = p.float().requires_grad_(True)
    torch.nn.functional.gelu(x, approximate="tanh").backward(acc)
    assert _rel(dg, x.grad) < 1e-2


@pytest.mark.parametrize("bn,cg", [(128, 1), (192, 1), (256, 1), (128, 2), (192, 2), (256, 2)])
def test_gemm_every_tile_config(ops, bn, cg):
    """Each forced tile configuration (128/256-wide tiles, single CTA or CTA
    pair with cta_group::2 MMAs) on every operand layout and epilogue, with M,
    N and K tails, against fp32 torch."""
    torch.manual_seed(7)
    try:
        for split in (0, 3, -1):  # -1: stream-K for the accumulating (wgrad) GEMM
            ops.gemm_set_tile(bn, cg, split)
            for M, N, K in ((200, 136, 192), (640, 1600, 320), (1280, 512, 1024)):
                a, b = _bf(M, K), _bf(N, K)
                d = torch.empty(M, N, device="cuda")
                ops.gemm(a, b, d, epi="f32")
                assert _rel(d, a.float() @ b.float().t()) < 1e-5, (M, N, K)
                bt = b.t().contiguous()           # B MN-major [K, N]
                ops.gemm(a, bt, d, b_mn=True, epi="f32")
                assert _rel(d, a.float() @ b.float().t()) < 1e-5, (M, N, K)
                at = a.t().contiguous()           # A MN-major [K, M]
                acc = torch.randn(M, N, device="cuda")
                ref = acc + a.float() @ b.float().t()
                ops.gemm(at, bt, acc, a_mn=True, b_mn=True, epi="acc_f32")
                assert _rel(acc, ref) < 1e-5, (M, N, K)
            M, N, K = 384, 1600, 512
            a, b = _bf(M, K), _bf(N, K, scale=0.05)
            bias = torch.randn(N, device="cuda")
            pre = a.float() @ b.float().t() + bias
            r = torch.randn(M, N, device="cuda")
            d32 = torch.empty(M, N, device="cuda")
            ops.gemm(a, b, d32, epi="resid_f32", bias=bias, aux=r)
            assert _rel(d32, r + pre) < 1e-5
            p = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
            g = torch.empty_like(p)
            ops.gemm(a, b, g, epi="gelu_bf16", bias=bias, aux=p)
            assert _rel(p, pre) < 1e-2
            assert _rel(g, torch.nn.functional.gelu(pre, approximate="tanh")) < 1e-2
            dg = torch.empty_like(p)
            ops.gemm(a, b, dg, epi="dgelu_bf16", aux=p)
            x = p.float().requires_grad_(True)
            torch.nn.functional.gelu(x, approximate="tanh").backward(pre - bias)
            assert _rel(dg, x.grad) < 1e-2
    finally:
        ops.gemm_set_tile(0, 0, 0)


def test_gemm_tile_choice():
    from paper_2202_01306_b200 import ops as O
    bn, cg, sp = O.gemm_tile(1600, 1600, 4096, "acc_f32")
    assert sp > 1 or sp == 0  # 13 x 7 wide tiles cannot fill 148 SMs: the weight gradient splits K (0 = stream-K)
    assert O.gemm_tile(4096, 50304, 1600, "f32")[1] == 2  # big problems run on CTA pairs


def test_adam_matches_torch(ops):
    torch.manual_seed(4)
    n = 1_000_003
    w0 = torch.randn(n, device="cuda") * 0.02
    w = w0.clone()
    k = torch.zeros(2 * n, device="cuda")
    p = torch.nn.Parameter(w0.clone())
    opt = torch.optim.Adam([p], lr=1e-4, betas=(0.9, 0.999), eps=1e-8)
    for step in range(1, 6):
        g = torch.randn(n, device="cuda")
        ops.adam(w, g, k, lr=1e-4, beta1=0.9, beta2=0.999, eps=1e-8, step=step)
        p.grad = g.clone()
        opt.step()
    torch.cuda.synchronize()
    assert torch.allclose(w, p.detach(), rtol=1e-6, atol=1e-7)
    st = opt.state[p]
    for got, ref in ((k[0::2], st["exp_avg"]), (k[1::2], st["exp_avg_sq"])):
        assert ((got - ref).norm() / ref.norm()).item() < 1e-6


def _attn_ref(qkv, B, S, H, DH, causal):
    d = H * DH
    q, k, v = qkv.float().view(B, S, 3, H, DH).permute(2, 0, 3, 1, 4)  # [B,H,S,DH]
    s = (q @ k.transpose(-1, -2)) / math.sqrt(DH)
    if causal:
        s = s.masked_fill(torch.triu(torch.ones(S, S, device=s.device, dtype=torch.bool), 1), float("-inf"))
    lse = torch.logsumexp(s, -1)
    o = torch.softmax(s, -1) @ v
    return o.permute(0, 2, 1, 3).reshape(B * S, d), lse.permute(0, 2, 1).reshape(B * S, H)


@pytest.mark.parametrize("B,S,H,DH,causal", [(2, 128, 4, 64, True), (1, 512, 2, 64, False),
                                             (2, 256, 3, 64, True), (1, 256, 2, 128, True),
                                             # head_dim 64: odd 128-key block count; more
                                             # (sample-head, tile pair) / key-block items than
                                             # SMs, so persistent CTAs walk several items
                                             (3, 1024, 5, 64, True), (2, 384, 3, 64, False),
                                             (8, 1024, 25, 64, True), (4, 512, 40, 64, False),
                                             # head_dim 128 (attention_tc128.cu): odd query-tile count,
                                             # full attention, the >HBM GPT shape at 1024 tokens
                                             (2, 384, 3, 128, True), (1, 512, 2, 128, False),
                                             (1, 1024, 4, 128, True), (1, 128, 2, 128, False)])
def test_attention_fwd_bwd(ops, B, S, H, DH, causal):
    torch.manual_seed(5)
    d = H * DH
    qkv = _bf(B * S, 3 * d)
    out = torch.empty(B * S, d, device="cuda", dtype=torch.bfloat16)
    lse = torch.empty(B * S, H, device="cuda")
    ops.attn_fwd(qkv, out, lse, batch=B, seq=S, heads=H, head_dim=DH, causal=causal)
    ro, rl = _attn_ref(qkv, B, S, H, DH, causal)
    assert _rel(out, ro) < 1e-2
    assert torch.allclose(lse, rl * 1.4426950408889634, atol=2e-3, rtol=1e-3)
    dout = _bf(B * S, d)
    dqkv = torch.empty_like(qkv)
    ops.attn_bwd(qkv, out, dout, lse, dqkv, batch=B, seq=S, heads=H, head_dim=DH, causal=causal)
    x = qkv.float().requires_grad_(True)
    o2, _ = _attn_ref(x, B, S, H, DH, causal)
    o2.backward(dout.float())
    g = x.grad.view(B * S, 3, d)
    got = dqkv.float().view(B * S, 3, d)
    for i in range(3):
        assert _rel(got[:, i], g[:, i]) < 2e-2, i


@pytest.mark.parametrize("M,d", [(1000, 1600), (37, 1024), (517, 4096), (300, 8192), (64, 256), (77, 1028),
                                 (33, 2048), (45, 5124)])
def test_layernorm_fwd_bwd(ops, M, d):
    """The default backward: rows in registers (one warp per row up to d = 1024,
    rows split over 2 / 8 warps up to 2048 / 8192), ragged row counts and
    column tails."""
    torch.manual_seed(6)
    x = torch.randn(M, d, device="cuda") * 2 + 0.5
    g = torch.randn(d, device="cuda")
    b = torch.randn(d, device="cuda")
    y = torch.empty(M, d, device="cuda", dtype=torch.bfloat16)
    mean = torch.empty(M, device="cuda")
    rstd = torch.empty(M, device="cuda")
    ops.layernorm_fwd(x, g, b, y, mean, rstd)
    xr = x.clone().requires_grad_(True)
    gr = g.clone().requires_grad_(True)
    br = b.clone().requires_grad_(True)
    yr = torch.nn.functional.layer_norm(xr, (d,), gr, br, 1e-5)
    assert _rel(y, yr) < 1e-2
    dy = torch.randn(M, d, device="cuda")
    yr.backward(dy)
    resid = torch.randn(M, d, device="cuda")
    out = torch.empty(M, d, device="cuda")
    ob = torch.empty(M, d, device="cuda", dtype=torch.bfloat16)
    dg = torch.ones(d, device="cuda")
    db = torch.ones(d, device="cuda")
    ops.layernorm_bwd(dy, x, mean, rstd, g, out, dg, db, resid=resid, out_bf16=ob)
    assert _rel(out, xr.grad + resid) < 1e-5
    assert _rel(ob, xr.grad + resid) < 1e-2
    assert _rel(dg, gr.grad + 1) < 1e-5
    assert _rel(db, br.grad + 1) < 1e-5


@pytest.mark.parametrize("variant", ["a", "w"])
def test_layernorm_bwd_variants(variant):
    """The opt-in LayerNorm backward kernels (HM_LN_BWD is read once per
    process): shared-memory atomics (a, also the fallback above d = 8192) and
    two-pass warps with private partials (w); the default keeps rows in
    registers (one warp per row up to d = 1024, 2 / 8 warps per row up to 8192)."""
    import subprocess
    import sys
    here = __import__("os").path.dirname(__import__("os").path.abspath(__file__))
    cases = [(1000, 1600), (37, 1024), (517, 4096), (300, 8192), (64, 256), (77, 1028)]
    code = (f"import torch, sys; sys.path.insert(0, {here!r}); sys.path.insert(0, {here + '/..'!r}); "
            "import test_kernels_gpu as T; from paper_2202_01306_b200 import ops; "
            f"[T.test_layernorm_fwd_bwd(ops, *c) for c in {cases!r}]")
    env = dict(__import__("os").environ, HM_LN_BWD=variant)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]


def test_weight_planes_exact(ops):
    """bf16 swap payloads: the device split / join restore fp32 bits exactly and
    the weight cast equals the hi plane (host reference: model.split_planes)."""
    import sys, os
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from test_payload import _edge_floats
    from paper_2202_01306_b200.model import split_planes
    f = _edge_floats()
    f = f[: (f.size // 8) * 8]
    w = torch.from_numpy(f.copy()).cuda()
    hi = torch.empty(w.numel(), dtype=torch.int16, device="cuda")
    lo = torch.empty_like(hi)
    ops.w_split(w, hi, lo)
    back = torch.empty_like(w)
    ops.w_join(hi, lo, back)
    cast = torch.empty(w.numel(), dtype=torch.bfloat16, device="cuda")
    ops.cast_w_bf16(w, cast)
    torch.cuda.synchronize()
    assert torch.equal(back.view(torch.int32), w.view(torch.int32))
    h_ref, l_ref = split_planes(f)
    assert np.array_equal(hi.cpu().numpy().view(np.uint16), h_ref)
    assert np.array_equal(lo.cpu().numpy().view(np.uint16), l_ref)
    assert np.array_equal(cast.view(torch.int16).cpu().numpy().view(np.uint16), h_ref)


def test_embedding_fwd_bwd(ops):
    torch.manual_seed(7)
    B, S, V, d = 3, 128, 1024, 256
    tok = torch.randint(0, V, (B * S,), device="cuda", dtype=torch.int32)
    wte = torch.randn(V, d, device="cuda")
    wpe = torch.randn(S, d, device="cuda")
    out = torch.empty(B * S, d, device="cuda")
    ops.embed_fwd(tok, wte, wpe, out, batch=B, seq=S)
    ref = wte[tok.long()] + wpe.repeat(B, 1)
    assert torch.allclose(out, ref)
    dx = torch.randn(B * S, d, device="cuda")
    dwte = torch.zeros(V, d, device="cuda")
    dwpe = torch.zeros(S, d, device="cuda")
    ops.embed_bwd(tok, dx, dwte, dwpe, batch=B, seq=S)
    rwte = torch.zeros(V, d, device="cuda").index_add_(0, tok.long(), dx)
    assert torch.allclose(dwte, rwte, atol=1e-5)
    assert torch.allclose(dwpe, dx.view(B, S, d).sum(0), atol=1e-5)


@pytest.mark.parametrize("M,V,Vp", [(300, 50257, 50304), (64, 1024, 1024), (37, 30522, 30592)])
def test_cross_entropy(ops, M, V, Vp):
    torch.manual_seed(8)
    logits = torch.randn(M, Vp, device="cuda") * 3
    labels = torch.randint(0, V, (M,), device="cuda", dtype=torch.int32)
    labels[0], labels[-1] = V - 1, 0  # the vocabulary tail (V % 4 != 0) and the first column
    dl = torch.empty(M, Vp, device="cuda", dtype=torch.bfloat16)
    loss = torch.zeros(1, device="cuda", dtype=torch.float64)
    ops.cross_entropy(logits, labels, V, dl, loss, 0.5)
    x = logits[:, :V].clone().requires_grad_(True)
    ref = torch.nn.functional.cross_entropy(x, labels.long(), reduction="sum")
    (ref * 0.5).backward()
    assert abs(loss.item() - ref.item()) / ref.item() < 1e-5
    assert _rel(dl[:, :V], x.grad) < 1e-2
    if Vp > V:
        assert dl[:, V:].abs().max().item() == 0


def test_bias_grad_and_cast(ops):
    torch.manual_seed(9)
    dy = _bf(4096, 6400)
    db = torch.ones(6400, device="cuda")
    ops.bias_grad(dy, db)
    assert _rel(db, dy.float().sum(0) + 1) < 1e-5
    dyf = torch.randn(1000, 1600, device="cuda")
    db2 = torch.zeros(1600, device="cuda")
    ops.bias_grad(dyf, db2)
    assert _rel(db2, dyf.sum(0)) < 1e-5
    # ragged row blocks and the two-column fallback (n % 8 != 0, strided rows)
    for rows, n, pad, dt in ((37, 1032, 8, torch.bfloat16), (1003, 18, 2, torch.float32), (517, 4800, 2, torch.float32),
                             (77, 1600, 0, torch.float32)):
        big = torch.randn(rows, n + pad, device="cuda").to(dt)
        v = big[:, :n]
        dbx = torch.zeros(n, device="cuda")
        ops.bias_grad(v, dbx)
        assert _rel(dbx, v.float().sum(0)) < 1e-5, (rows, n, dt)
    src = torch.randn(1_000_001, device="cuda")
    dst = torch.empty(1_000_001, device="cuda", dtype=torch.bfloat16)
    ops.cast_bf16(src, dst)
    assert torch.equal(dst, src.to(torch.bfloat16))


@pytest.mark.parametrize("B,S,H,causal,DH", [(2, 128, 4, True, 64), (1, 512, 2, False, 64), (2, 1024, 3, True, 64),
                                             (1, 256, 25, True, 64), (2, 1024, 3, True, 128),
                                             (1, 640, 2, False, 128), (4, 1024, 64, True, 128)])
def test_attention_fwd_tcgen05_matches(ops, B, S, H, causal, DH):
    torch.manual_seed(11)
    d = H * DH
    qkv = _bf(B * S, 3 * d)
    out = torch.empty(B * S, d, device="cuda", dtype=torch.bfloat16)
    lse = torch.empty(B * S, H, device="cuda")
    ops.attn_fwd_tc(qkv, out, lse, batch=B, seq=S, heads=H, head_dim=DH, causal=causal)
    ro, rl = _attn_ref(qkv, B, S, H, DH, causal)
    assert _rel(out, ro) < 1e-2
    assert torch.allclose(lse, rl * 1.4426950408889634, atol=2e-3, rtol=1e-3)


@pytest.mark.parametrize("variant", ["mma", "s"])
def test_attention_bwd_tcgen05_opt_in(variant):
    """The opt-in backward kernels match autograd: the mma.sync one
    (HM_ATTN_BWD=mma) and the 64-query sub-block head_dim-64 tcgen05 one
    (s, attention_bwd64.cu); the default is attention_tc.cu's 128-query kernel."""
    import subprocess
    import sys
    here = __import__("os").path.dirname(__import__("os").path.abspath(__file__))
    code = (f"import torch, sys; sys.path.insert(0, {here!r}); sys.path.insert(0, {here + '/..'!r}); "
            "import test_kernels_gpu as T; "
            "from paper_2202_01306_b200 import ops; "
            "T.test_attention_fwd_bwd(ops, 2, 256, 3, 64, True); T.test_attention_fwd_bwd(ops, 1, 512, 2, 64, False); "
            "T.test_attention_fwd_bwd(ops, 1, 256, 2, 128, True); T.test_attention_fwd_bwd(ops, 3, 1024, 5, 64, True)")
    env = dict(__import__("os").environ, HM_ATTN_BWD=variant)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]


@pytest.mark.parametrize("mode", ["q", "t", "d"])
def test_attention_fwd_every_variant(mode):
    """Every forward variant (HM_ATTN_FWD is read once per process, so each runs
    in a subprocess) on shapes where the persistent kernel walks one item per
    CTA, several items per CTA, and a ragged last round."""
    import subprocess
    import sys
    here = __import__("os").path.dirname(__import__("os").path.abspath(__file__))
    cases = [(2, 128, 4, True, 64), (1, 512, 2, False, 64), (2, 1024, 3, True, 64), (3, 1024, 25, True, 64),
             (2, 512, 40, False, 64), (1, 256, 25, True, 64)]
    code = (f"import torch, sys; sys.path.insert(0, {here!r}); sys.path.insert(0, {here + '/..'!r}); "
            "import test_kernels_gpu as T; from paper_2202_01306_b200 import ops; "
            f"[T.test_attention_fwd_tcgen05_matches(ops, *c) for c in {cases!r}]")
    env = dict(__import__("os").environ, HM_ATTN_FWD=mode)
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]


def _conv_ref(x, w):
    import torch.nn.functional as F
    return F.conv2d(x.float().permute(0, 3, 1, 2), w.float().permute(0, 3, 1, 2), padding=1).permute(0, 2, 3, 1)


@pytest.mark.parametrize("n,h,wd,cin,cout", [(2, 8, 8, 64, 64), (3, 14, 10, 128, 64), (1, 32, 32, 64, 256),
                                            (2, 7, 9, 192, 128)])
@pytest.mark.parametrize("cfg", [(0, 0), (128, 1), (256, 2)])
def test_conv3x3_implicit_gemm(ops, n, h, wd, cin, cout, cfg):
    """Implicit-GEMM 3x3 conv (TMA im2col operands) fwd / dgrad / wgrad and the
    ReLU / residual epilogues vs torch fp32, on odd image sizes (pixel tiles
    straddle rows and images) and every tile configuration."""
    import torch.nn.functional as F
    torch.manual_seed(11)
    x = _bf(n, h, wd, cin)
    w = _bf(cout, 3, 3, cin, scale=0.05)
    bias = torch.randn(cout, device="cuda") * 0.1
    try:
        ops.gemm_set_tile(cfg[0], cfg[1], 0)
        ref = _conv_ref(x, w)
        y = torch.empty(n, h, wd, cout, device="cuda", dtype=torch.bfloat16)
        ops.conv_fwd(x, w, y)
        assert _rel(y, ref) < 1e-2
        ops.conv_fwd(x, w, y, epi="relu_bf16", bias=bias)
        assert _rel(y, torch.relu(ref + bias)) < 1e-2
        r = _bf(n, h, wd, cout)
        ops.conv_fwd(x, w, y, epi="resid_relu_bf16", bias=bias, aux=r)
        assert _rel(y, torch.relu(ref + bias + r.float())) < 1e-2
        dy = _bf(n, h, wd, cout)
        xr = x.float().permute(0, 3, 1, 2).requires_grad_(True)
        wr = w.float().permute(0, 3, 1, 2).requires_grad_(True)
        F.conv2d(xr, wr, padding=1).backward(dy.float().permute(0, 3, 1, 2))
        dx_ref = xr.grad.permute(0, 2, 3, 1)
        dx = torch.empty_like(x)
        ops.conv_dgrad(dy, w, dx)
        assert _rel(dx, dx_ref) < 1e-2
        ops.conv_dgrad(dy, w, dx, epi="drelu_bf16", aux=x)
        assert _rel(dx, dx_ref * (x.float() > 0)) < 1e-2
        ops.conv_dgrad(dy, w, dx, epi="add_bf16", aux=x)
        assert _rel(dx, dx_ref + x.float()) < 1e-2
        dw = torch.randn(cout, 3, 3, cin, device="cuda")
        dw_ref = dw + wr.grad.permute(0, 2, 3, 1)
        ops.conv_wgrad(dy, x, dw)
        assert _rel(dw, dw_ref) < 1e-4
    finally:
        ops.gemm_set_tile(0, 0, 0)

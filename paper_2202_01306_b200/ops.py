"""Torch-tensor wrappers over the exported sm_100a kernels (hm_k_* in
include/harmony_b200.h).  Tensors are plumbing here: every call goes straight
to the native kernel on the tensor's current CUDA stream; there is no torch
compute fallback -- a missing library or a CPU tensor raises.
"""

from __future__ import annotations

import ctypes as C

import torch

from . import _native as NL

EPI = {"bf16": 0, "f32": 1, "acc_f32": 2, "resid_f32": 3, "gelu_bf16": 4, "dgelu_bf16": 5,
       "relu_bf16": 6, "resid_relu_bf16": 7, "drelu_bf16": 8, "add_bf16": 9}


def _ptr(t):
    if t is None:
        return None
    if not t.is_cuda:
        raise ValueError("hm kernels take CUDA tensors only")
    return C.c_void_p(t.data_ptr())


def _stream():
    return C.c_void_p(torch.cuda.current_stream().cuda_stream)


def gemm(a, b, d, *, a_mn=False, b_mn=False, epi="f32", bias=None, aux=None):
    """d (op)= A . B^T.  K-major A is [M,K]; MN-major A is stored [K,M].
    K-major B is [N,K]; MN-major B is stored [K,N].  d is [M,N]."""
    if a_mn:
        K, M = a.shape
    else:
        M, K = a.shape
    N = b.shape[1] if b_mn else b.shape[0]
    assert d.shape == (M, N)
    lib = N_lib()
    rc = lib.hm_k_gemm(_ptr(a), _ptr(b), _ptr(d), M, N, K, a.stride(0), b.stride(0), d.stride(0),
                       int(a_mn), int(b_mn), EPI[epi], _ptr(bias), _ptr(aux),
                       aux.stride(0) if aux is not None else 0, 1, 0, 0, 0, _stream())
    NL.check(rc)
    return d


def conv_fwd(x, w, y, *, epi="bf16", bias=None, aux=None):
    """y[n,h,w,cout] = conv3x3(x[n,h,w,cin], w[cout,3,3,cin]) (+epilogue), NHWC bf16."""
    n, h, wd, cin = x.shape
    cout = w.shape[0]
    NL.check(N_lib().hm_k_conv_fwd(_ptr(x), _ptr(w), _ptr(y), n, h, wd, cin, cout, EPI[epi], _ptr(bias), _ptr(aux),
                                   _stream()))
    return y


def conv_dgrad(dy, w, dx, *, epi="bf16", aux=None):
    """dx[n,h,w,cin] = grad of conv3x3 w.r.t. its input, from dy[n,h,w,cout]."""
    n, h, wd, cout = dy.shape
    cin = w.shape[-1]
    NL.check(N_lib().hm_k_conv_dgrad(_ptr(dy), _ptr(w), _ptr(dx), n, h, wd, cin, cout, EPI[epi], _ptr(aux),
                                     _stream()))
    return dx


def conv_wgrad(dy, x, dw):
    """dw[cout,3,3,cin] (fp32) += grad of conv3x3 w.r.t. its weights."""
    n, h, wd, cin = x.shape
    cout = dy.shape[-1]
    NL.check(N_lib().hm_k_conv_wgrad(_ptr(dy), _ptr(x), _ptr(dw), n, h, wd, cin, cout, _stream()))
    return dw


def gemm_tile(M, N, K, epi="f32", b_mn=False):
    """(bn, cta_pair, splits) the GEMM picks for this problem."""
    bn, cg, sp = C.c_int32(), C.c_int32(), C.c_int32()
    NL.check(N_lib().hm_k_gemm_tile(M, N, K, EPI[epi], int(b_mn), C.byref(bn), C.byref(cg), C.byref(sp)))
    return bn.value, cg.value, sp.value


def gemm_set_tile(bn=0, cta_pair=0, splits=0):
    """Force the GEMM tile configuration process-wide (0 = automatic)."""
    NL.check(N_lib().hm_k_gemm_set_tile(bn, cta_pair, splits))


def adam(w, g, k, *, lr, beta1, beta2, eps, step, grad_scale=1.0):
    rc = N_lib().hm_k_adam(_ptr(w), _ptr(g), _ptr(k), w.numel(), lr, beta1, beta2, eps, step,
                           grad_scale, _stream())
    NL.check(rc)


def launch_count() -> int:
    return int(N_lib().hm_launch_count())


def attn_fwd(qkv, out, lse, *, batch, seq, heads, head_dim, causal=True):
    NL.check(N_lib().hm_k_attn_fwd(_ptr(qkv), _ptr(out), _ptr(lse), batch, seq, heads, head_dim,
                                   int(causal), _stream()))


def attn_fwd_tc(qkv, out, lse, *, batch, seq, heads, head_dim, causal=True):
    NL.check(N_lib().hm_k_attn_fwd_tc(_ptr(qkv), _ptr(out), _ptr(lse), batch, seq, heads, head_dim,
                                      int(causal), _stream()))


def attn_bwd(qkv, out, dout, lse, dqkv, *, batch, seq, heads, head_dim, causal=True):
    rows = batch * seq
    dvec = torch.empty(rows * heads, device=qkv.device)
    dq = torch.empty(rows, heads * head_dim, device=qkv.device)
    NL.check(N_lib().hm_k_attn_bwd(_ptr(qkv), _ptr(out), _ptr(dout), _ptr(lse), _ptr(dvec), _ptr(dq),
                                   _ptr(dqkv), batch, seq, heads, head_dim, int(causal), _stream()))


def cast_bf16(src, dst):
    NL.check(N_lib().hm_k_cast_bf16(_ptr(src), _ptr(dst), src.numel(), _stream()))


def cast_w_bf16(src, dst):
    """Weight operand cast: bf16 nearest, ties toward zero (the hi plane)."""
    NL.check(N_lib().hm_k_cast_w_bf16(_ptr(src), _ptr(dst), src.numel(), _stream()))


def w_split(w, hi, lo):
    NL.check(N_lib().hm_k_w_split(_ptr(w), _ptr(hi), _ptr(lo), w.numel(), _stream()))


def w_join(hi, lo, w):
    NL.check(N_lib().hm_k_w_join(_ptr(hi), _ptr(lo), _ptr(w), w.numel(), _stream()))


def embed_fwd(tokens, wte, wpe, out, *, batch, seq):
    NL.check(N_lib().hm_k_embed_fwd(_ptr(tokens), _ptr(wte), _ptr(wpe), _ptr(out), batch, seq,
                                    wte.shape[1], _stream()))


def embed_bwd(tokens, dx, dwte, dwpe, *, batch, seq):
    NL.check(N_lib().hm_k_embed_bwd(_ptr(tokens), _ptr(dx), _ptr(dwte), _ptr(dwpe), batch, seq,
                                    dwte.shape[1], _stream()))


def layernorm_fwd(x, g, b, y, mean, rstd):
    NL.check(N_lib().hm_k_layernorm_fwd(_ptr(x), _ptr(g), _ptr(b), _ptr(y), _ptr(mean), _ptr(rstd),
                                        x.shape[0], x.shape[1], _stream()))


def layernorm_bwd(dy, x, mean, rstd, g, out, dg, db, *, resid=None, out_bf16=None):
    NL.check(N_lib().hm_k_layernorm_bwd(_ptr(dy), _ptr(x), _ptr(mean), _ptr(rstd), _ptr(g),
                                        _ptr(resid), _ptr(out), _ptr(out_bf16), _ptr(dg), _ptr(db),
                                        x.shape[0], x.shape[1], _stream()))


def cross_entropy(logits, labels, vocab, dlogits, loss_sum, scale):
    NL.check(N_lib().hm_k_cross_entropy(_ptr(logits), _ptr(labels), logits.shape[0], logits.stride(0),
                                        vocab, _ptr(dlogits), _ptr(loss_sum), scale, _stream()))


def bias_grad(dy, db):
    NL.check(N_lib().hm_k_bias_grad(_ptr(dy), int(dy.dtype == torch.bfloat16), _ptr(db), dy.shape[0],
                                    dy.shape[1], dy.stride(0), _stream()))


def N_lib():
    return NL.lib()


def gemm_replay_us(shape, reps: int = 32) -> float:
    """The GEMM's own per-launch time (us) for one logged shape (m, n, k,
    a_major, b_major, epilogue, has_bias): back-to-back launches in a CUDA
    graph, CUDA-event timed, rotating operand sets (hm_k_gemm_replay)."""
    arr = (C.c_int64 * 7)(*shape)
    us = C.c_double(0.0)
    NL.check(N_lib().hm_k_gemm_replay(arr, reps, _stream(), C.byref(us)))
    return us.value

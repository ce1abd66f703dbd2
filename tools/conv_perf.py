"""Implicit-GEMM conv micro-benchmark at the resnet-bench stage shapes:
fwd / dgrad / wgrad per forced tile configuration (CUDA events, L2 flushed)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2202_01306_b200 import ops

flush_buf = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def timeit(fn, iters=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(iters):
        flush_buf.zero_()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn()
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    return ts[len(ts) // 2]


for n, h, c in ((16, 56, 128), (32, 56, 128), (16, 28, 256), (32, 28, 256)):
    x = torch.randn(n, h, h, c, device="cuda").to(torch.bfloat16)
    w = (torch.randn(c, 3, 3, c, device="cuda") * 0.05).to(torch.bfloat16)
    y = torch.empty_like(x)
    dw = torch.zeros(c, 3, 3, c, device="cuda")
    bias = torch.zeros(c, device="cuda")
    fl = 2.0 * n * h * h * 9 * c * c
    for cfg in ((0, 0), (128, 1), (256, 1), (128, 2), (256, 2)):
        ops.gemm_set_tile(cfg[0], cfg[1], 0)
        r = {"n": n, "h": h, "c": c, "bn": cfg[0], "cg": cfg[1]}
        for name, fn in (("fwd", lambda: ops.conv_fwd(x, w, y, epi="relu_bf16", bias=bias)),
                         ("dgrad", lambda: ops.conv_dgrad(x, w, y)),
                         ("wgrad", lambda: ops.conv_wgrad(x, x, dw))):
            ms = timeit(fn)
            r[name + "_tflops"] = round(fl / ms / 1e9, 1)
        print(json.dumps(r), flush=True)
    ops.gemm_set_tile(0, 0, 0)

"""Attention forward / backward timing (CUDA events, warm, inputs > L2 not
needed: one head-block's K/V is the working set).  One JSON line per shape.

    python tools/attn_perf.py B S H DH causal [iters]

Kernel selection follows the library's env switches (HM_ATTN=mma,
HM_ATTN_BWD=mma force the mma.sync kernels)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_2202_01306_b200 import ops  # noqa: E402


def main() -> None:
    B, S, H, DH, causal = (int(x) for x in sys.argv[1:6])
    iters = int(sys.argv[6]) if len(sys.argv) > 6 else 20
    d = H * DH
    torch.manual_seed(0)
    qkv = torch.randn(B * S, 3 * d, device="cuda").to(torch.bfloat16)
    out = torch.empty(B * S, d, device="cuda", dtype=torch.bfloat16)
    lse = torch.empty(B * S, H, device="cuda")
    dout = torch.randn(B * S, d, device="cuda").to(torch.bfloat16)
    dqkv = torch.empty_like(qkv)
    for _ in range(3):
        ops.attn_fwd(qkv, out, lse, batch=B, seq=S, heads=H, head_dim=DH, causal=bool(causal))
        ops.attn_bwd(qkv, out, dout, lse, dqkv, batch=B, seq=S, heads=H, head_dim=DH, causal=bool(causal))
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    ev[0].record()
    for _ in range(iters):
        ops.attn_fwd(qkv, out, lse, batch=B, seq=S, heads=H, head_dim=DH, causal=bool(causal))
    ev[1].record()
    for _ in range(iters):
        ops.attn_bwd(qkv, out, dout, lse, dqkv, batch=B, seq=S, heads=H, head_dim=DH, causal=bool(causal))
    ev[2].record()
    torch.cuda.synchronize()
    f_ms = ev[0].elapsed_time(ev[1]) / iters
    b_ms = ev[1].elapsed_time(ev[2]) / iters
    frac = 0.5 if causal else 1.0
    ffl = 4.0 * B * S * S * H * DH * frac
    bfl = 2.5 * ffl  # dV, dK, dQ, dP, S recompute: 5 GEMMs vs the forward's 2
    print(json.dumps({"B": B, "S": S, "H": H, "DH": DH, "causal": causal, "fwd_us": round(f_ms * 1e3, 2),
                      "bwd_us": round(b_ms * 1e3, 2), "fwd_tflops": round(ffl / f_ms / 1e9, 1),
                      "bwd_tflops": round(bfl / b_ms / 1e9, 1),
                      "env": {k: v for k, v in os.environ.items() if k.startswith("HM_ATTN")}}), flush=True)


if __name__ == "__main__":
    main()

"""Numerical A/B of GEMM tile configurations on MN-major-B shapes: each forced
(bn, CTA pair, split) against an fp64 reference, for the plain fp32 store and
the accumulating (TMA reduce-add) epilogue.

    python tools/gemm_tile_diff.py"""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_2202_01306_b200 import ops  # noqa: E402


def main() -> None:
    torch.manual_seed(0)
    for (M, N, K) in [(4096, 1600, 6400), (2048, 1600, 1600), (640, 1600, 320), (1000, 1600, 800)]:
        a = torch.randn(M, K, device="cuda").to(torch.bfloat16)
        bt = torch.randn(K, N, device="cuda").to(torch.bfloat16)  # MN-major B [K, N]
        ref = a.double() @ bt.double()
        c0 = torch.randn(M, N, device="cuda")
        for cfg in [(192, 1, 0), (192, 2, 0), (192, 1, 3), (192, 2, 3), (192, 2, -1), (256, 2, 0), (0, 0, 0)]:
            ops.gemm_set_tile(*cfg)
            d = torch.empty(M, N, device="cuda")
            ops.gemm(a, bt, d, b_mn=True, epi="f32")
            acc = c0.clone()
            ops.gemm(a, bt, acc, b_mn=True, epi="acc_f32")
            torch.cuda.synchronize()
            e1 = ((d.double() - ref).abs().max() / ref.abs().max()).item()
            e2 = ((acc.double() - c0.double() - ref).abs().max() / ref.abs().max()).item()
            print(json.dumps({"shape": [M, N, K], "tile": cfg, "f32_rel": e1, "acc_f32_rel": e2}), flush=True)
        ops.gemm_set_tile(0, 0, 0)


if __name__ == "__main__":
    main()

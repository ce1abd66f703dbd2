"""GEMM shapes of one GPT-2 XL Harmony iteration (bench.py's gemm_replay list),
timed by graph replay (ops.gemm_replay_us, L2-rotating operand sets).  One
JSON line per shape; the tile configuration follows the process's env
switches (HM_GEMM_STREAMK, HM_GEMM_BN, ...).

    python tools/gemm_shapes.py [tag] [shape index]"""
import json
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_2202_01306_b200 import ops  # noqa: E402

# (m, n, k, a_mn, b_mn, epilogue, has_bias) and launches per iteration
SHAPES = [((4096, 1600, 6400, 0, 0, 3, 1), 352), ((4096, 6400, 1600, 0, 0, 4, 1), 352),
          ((4096, 6400, 1600, 0, 1, 5, 0), 192), ((1600, 6400, 4096, 1, 1, 2, 0), 192),
          ((4096, 4800, 1600, 0, 0, 0, 1), 352), ((4096, 1600, 6400, 0, 1, 1, 0), 192),
          ((6400, 1600, 4096, 1, 1, 2, 0), 192), ((4096, 1600, 4800, 0, 1, 1, 0), 192),
          ((4800, 1600, 4096, 1, 1, 2, 0), 192), ((4096, 1600, 1600, 0, 0, 3, 1), 352),
          ((1600, 1600, 4096, 1, 1, 2, 0), 192), ((4096, 1600, 1600, 0, 1, 0, 0), 192)]


EPI_NAME = {v: k for k, v in ops.EPI.items()}


def main() -> None:
    import torch
    tag = sys.argv[1] if len(sys.argv) > 1 else ""
    only = int(sys.argv[2]) if len(sys.argv) > 2 else None
    torch.cuda.init()
    tot_f = tot_us = 0.0
    for idx, (shp, count) in enumerate(SHAPES):
        if only is not None and idx != only:
            continue
        us = ops.gemm_replay_us(shp, reps=32)
        fl = 2.0 * shp[0] * shp[1] * shp[2]
        tot_f += fl * count
        tot_us += us * count
        print(json.dumps({"tag": tag, "shape": shp, "count": count, "us": round(us, 2),
                          "tflops": round(fl / (us * 1e-6) / 1e12, 1),
                          "tile": ops.gemm_tile(shp[0], shp[1], shp[2], EPI_NAME[shp[5]], bool(shp[4]))}),
              flush=True)
    print(json.dumps({"tag": tag, "weighted_tflops": round(tot_f / (tot_us * 1e-6) / 1e12, 1),
                      "ms_per_iter": round(tot_us / 1e3, 2)}), flush=True)


if __name__ == "__main__":
    main()

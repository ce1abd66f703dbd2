"""One GEMM shape under each epilogue (graph replay): the epilogue's share of
a short-K GEMM.   python tools/gemm_epi_ab.py M N K"""
import json
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
from paper_2202_01306_b200 import ops  # noqa: E402


def main() -> None:
    import torch
    torch.cuda.init()
    m, n, k = (int(x) for x in sys.argv[1:4])
    for epi, name in ((0, "bf16"), (1, "f32"), (3, "resid_f32"), (4, "gelu_bf16"), (2, "acc_f32")):
        shp = (m, n, k, 0 if epi != 2 else 1, 0 if epi != 2 else 1, epi, 1 if epi in (0, 1, 3, 4) else 0)
        us = ops.gemm_replay_us(shp, reps=32)
        print(json.dumps({"shape": [m, n, k], "epi": name, "us": round(us, 2),
                          "tflops": round(2.0 * m * n * k / (us * 1e-6) / 1e12, 1),
                          "tile": ops.gemm_tile(m, n, k, name, epi == 2),
                          "env": {e: os.environ.get(e) for e in ("HM_GEMM_BN", "HM_GEMM_CG", "HM_GEMM_SPLITK")}}),
              flush=True)


if __name__ == "__main__":
    main()

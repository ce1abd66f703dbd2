"""cuBLAS (torch.matmul, bf16 in / bf16 out, fp32 accumulate) on the GPT-2 XL
iteration's GEMM shapes, CUDA-graph timed like tools/gemm_shapes.py (rotating
operand sets larger than L2): the library baseline for the tcgen05 GEMM."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
from gemm_shapes import SHAPES  # noqa: E402


def main() -> None:
    tot_f = tot_us = 0.0
    for (m, n, k, a_mn, b_mn, epi, _), count in SHAPES:
        nset = max(2, int((300 << 20) // ((m * k + n * k) * 2)) + 1)
        A = [torch.randn(m, k, device="cuda", dtype=torch.bfloat16) for _ in range(nset)]
        B = [torch.randn(k, n, device="cuda", dtype=torch.bfloat16) for _ in range(nset)]
        if b_mn == 0:  # K-major B: weights [n, k] used transposed
            B = [torch.randn(n, k, device="cuda", dtype=torch.bfloat16).t() for _ in range(nset)]
        if a_mn:
            A = [torch.randn(k, m, device="cuda", dtype=torch.bfloat16).t() for _ in range(nset)]
        out = torch.empty(m, n, device="cuda", dtype=torch.bfloat16)
        reps = 32
        for i in range(3):
            torch.matmul(A[i % nset], B[i % nset], out=out)
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        g = torch.cuda.CUDAGraph()
        with torch.cuda.stream(s):
            torch.matmul(A[0], B[0], out=out)
            with torch.cuda.graph(g, stream=s):
                for i in range(reps):
                    torch.matmul(A[i % nset], B[i % nset], out=out)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        g.replay()
        torch.cuda.synchronize()
        e0.record()
        for _ in range(3):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / (3 * reps)
        fl = 2.0 * m * n * k
        tot_f += fl * count
        tot_us += us * count
        print(json.dumps({"lib": "cublas", "shape": [m, n, k, a_mn, b_mn, epi], "us": round(us, 2),
                          "tflops": round(fl / (us * 1e-6) / 1e12, 1)}), flush=True)
    print(json.dumps({"lib": "cublas", "weighted_tflops": round(tot_f / (tot_us * 1e-6) / 1e12, 1),
                      "ms_per_iter": round(tot_us / 1e3, 2)}), flush=True)


if __name__ == "__main__":
    main()

"""Config c3 exactly as benched (bench.py gpt2-xl-dp: GPT-2 XL, 48 layers,
Harmony-DP on one GPU, D = 16 as u = 4 microbatches, packs of 8 layers), 2
steps in both arithmetic modes vs the torch-CPU fp32 oracle
(tests/test_parity_gpu.run_parity).  Evidence run, not in the suite (the
full-depth oracle takes minutes on the host)."""
import json
import os
import sys

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main() -> None:
    import paper_2202_01306_b200 as H
    from paper_2202_01306_b200.model import GPT_PRESETS
    from test_parity_gpu import BF16_TOL, FP32_TOL, run_parity
    spec = GPT_PRESETS["gpt2-xl"]
    packs = tuple((i, min(i + 8, 48) - 1) for i in range(0, 48, 8))
    cfg = H.Configuration(4, packs, 4, packs, 16, H.Mode.DP)
    for math in sys.argv[1:] or ("fp32", "bf16"):
        res = run_parity(spec, cfg, 2, math, alpha=(32 if math == "bf16" else 60) << 30)
        tol = FP32_TOL if math == "fp32" else BF16_TOL
        ok = res["loss"] < tol["loss"] and all(max(res[k]) < tol[k] for k in ("dw", "m", "v"))
        print(json.dumps({"config": "c3 gpt2-xl 48 layers, Harmony-DP, D=16, u=4, packs of 8, 2 steps", "math": math,
                          "loss_rel": res["loss"], "dw_max": max(res["dw"]), "m_max": max(res["m"]),
                          "v_max": max(res["v"]), "tolerance": tol, "within": ok}), flush=True)


if __name__ == "__main__":
    main()

"""Config c2 at full depth and the benched grouping (BERT-Large: 24 layers,
d=1024, 16 heads, seq 512, V=30522, full attention; D = 64 as u = 16
microbatches, packs of 6), 2 steps in both arithmetic modes vs the torch-CPU
fp32 oracle (tests/test_parity_gpu.run_parity).  Evidence run, not in the
suite (the 24-layer oracle takes minutes on the host)."""
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
    spec = GPT_PRESETS["bert-large"]
    packs = tuple((i, i + 5) for i in range(0, 24, 6))
    cfg = H.Configuration(16, packs, 16, packs, 64, H.Mode.PP)
    for math in ("fp32", "bf16"):
        res = run_parity(spec, cfg, 2, math, alpha=60 << 30)
        tol = FP32_TOL if math == "fp32" else BF16_TOL
        ok = res["loss"] < tol["loss"] and all(max(res[k]) < tol[k] for k in ("dw", "m", "v"))
        print(json.dumps({"config": "c2 bert-large 24 layers, D=64, u=16, packs of 6, 2 steps", "math": math,
                          "loss_rel": res["loss"], "dw_max": max(res["dw"]), "m_max": max(res["m"]),
                          "v_max": max(res["v"]), "tolerance": tol, "within": ok}), flush=True)


if __name__ == "__main__":
    main()

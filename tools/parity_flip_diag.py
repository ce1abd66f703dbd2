"""Where the fp32-mode per-layer update error of the c3-shape parity test comes
from: after Adam's first steps every update is ~lr * sign(m / sqrt(v)), so the
metric ||dw - dw_ref|| / ||dw_ref|| counts the elements whose gradient is so
close to zero that two fp32 summation orders disagree on its sign.  Prints,
per layer, the metric, the number of sign-disagreeing update elements and the
metric with those elements left out.

    python tools/parity_flip_diag.py [steps]"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), ".."))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests"))


def main() -> None:
    import paper_2202_01306_b200 as H
    from paper_2202_01306_b200.model import GPTSpec, gpt_profiles, synthetic_batch
    from paper_2202_01306_b200.runtime import HarmonyRuntime
    from oracle.gpt_cpu import GPTOracle
    steps = int(sys.argv[1]) if len(sys.argv) > 1 else 3
    spec = GPTSpec(4, 1600, 25, 1024, 50257, True, "gpt2-xl-4l")
    packs = ((0, 1), (2, 3))
    cfg = H.Configuration(2, packs, 2, packs, 4, H.Mode("dp"))
    alpha, lr = 40 << 30, 1e-4
    prof = gpt_profiles(spec, u_max=64)
    mach = H.MachineModel(gpu_count=1, gpu_mem_capacity=alpha, pcie_bandwidth=55_000_000_000)
    g = H.generate_task_graph(cfg, mach, prof)
    rt = HarmonyRuntime(spec, alpha_bytes=alpha, lr=lr, math="fp32")
    rt.init_weights(0)
    w0 = rt.w.copy()
    rt.load(g, mach, prof)
    tok, lab = synthetic_batch(spec, cfg.minibatch)
    for _ in range(steps):
        rt.step(tok, lab)
    w, off = rt.w.copy(), rt.w_off.copy()
    rt.close()
    o = GPTOracle(spec, w0, off, lr=lr)
    groups = list(H.microbatch_groups(cfg.minibatch, cfg.u_f))
    for _ in range(steps):
        o.step(tok, lab, groups)
    ref = o.w.numpy()
    for L in range(len(off) - 1):
        a, b = int(off[L]), int(off[L + 1])
        da, db = w[a:b] - w0[a:b], ref[a:b] - w0[a:b]
        flip = np.sign(da) != np.sign(db)
        keep = ~flip
        print(json.dumps({"layer": L, "params": b - a, "dw_rel": float(np.linalg.norm(da - db) / np.linalg.norm(db)),
                          "sign_disagreements": int(flip.sum()),
                          "dw_rel_without_them": float(np.linalg.norm((da - db)[keep]) / np.linalg.norm(db[keep])),
                          "env": {k: v for k, v in os.environ.items() if k.startswith("HM_GEMM")}}), flush=True)


if __name__ == "__main__":
    main()

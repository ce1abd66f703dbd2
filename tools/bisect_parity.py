"""Loss of the first iteration vs the fp32 oracle across model shapes (bisects
a parity failure by d_model / head_dim / u)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2202_01306_b200 as H
from paper_2202_01306_b200.model import GPTSpec, gpt_profiles, synthetic_batch
from paper_2202_01306_b200.runtime import HarmonyRuntime
from oracle.gpt_cpu import GPTOracle

cases = [
    (GPTSpec(2, 1024, 16, 256, 1024), 1), (GPTSpec(2, 1024, 8, 256, 1024), 1),
    (GPTSpec(2, 2048, 16, 256, 1024), 1), (GPTSpec(2, 4096, 32, 256, 1024), 1),
    (GPTSpec(2, 4096, 64, 256, 1024), 1), (GPTSpec(2, 8192, 64, 256, 1024), 2),
    (GPTSpec(2, 8192, 128, 256, 1024), 1),
]
for spec, u in cases:
    packs = ((0, 0), (1, 1))
    cfg = H.Configuration(u, packs, u, packs, 2, H.Mode.PP)
    prof = gpt_profiles(spec)
    mach = H.MachineModel(gpu_count=1, gpu_mem_capacity=48 << 30, pcie_bandwidth=55_000_000_000)
    g = H.generate_task_graph(cfg, mach, prof)
    rt = HarmonyRuntime(spec, alpha_bytes=48 << 30)
    rt.init_weights(0)
    orc = GPTOracle(spec, rt.w.copy(), rt.w_off)
    rt.load(g, mach, prof)
    tok, lab = synthetic_batch(spec, 2)
    loss = rt.step(tok, lab)
    ref = orc.step(tok, lab, list(g.tasks[0].group))
    w_ref = orc.w.numpy()
    print(json.dumps({"d": spec.d_model, "h": spec.n_head, "dh": spec.head_dim, "u": u, "loss": loss, "ref": ref,
                      "rel": abs(loss - ref) / ref,
                      "rel_w": float(np.linalg.norm(rt.w - w_ref) / np.linalg.norm(w_ref))}), flush=True)
    rt.close()
    del orc

"""First-iteration loss vs the fp32 oracle for one shape chosen by env vars
(DM, NH, NL, U, DD, PK, MODE) -- a bisection aid for parity failures."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2202_01306_b200 as H
from paper_2202_01306_b200.model import GPTSpec, gpt_profiles, synthetic_batch
from paper_2202_01306_b200.runtime import HarmonyRuntime
from oracle.gpt_cpu import GPTOracle
spec = GPTSpec(int(os.environ.get("NL", 2)), int(os.environ.get("DM", 2048)), int(os.environ.get("NH", 16)), 256, 1024)
u = int(os.environ.get("U", 1)); D = int(os.environ.get("DD", 2))
packs = tuple((i, i) for i in range(spec.n_layer)) if os.environ.get("PK", "1") == "1" else ((0, spec.n_layer - 1),)
cfg = H.Configuration(u, packs, u, packs, D, H.Mode(os.environ.get("MODE", "pp")))
prof = gpt_profiles(spec)
mach = H.MachineModel(gpu_count=1, gpu_mem_capacity=48 << 30, pcie_bandwidth=55_000_000_000)
g = H.generate_task_graph(cfg, mach, prof)
rt = HarmonyRuntime(spec, alpha_bytes=48 << 30)
rt.init_weights(0)
orc = GPTOracle(spec, rt.w.copy(), rt.w_off)
rt.load(g, mach, prof)
tok, lab = synthetic_batch(spec, D)
loss = rt.step(tok, lab)
ref = orc.step(tok, lab, list(g.tasks[0].group))
print(json.dumps({k: os.environ.get(k) for k in ("HM_GEMM_PDL", "CUDA_LAUNCH_BLOCKING", "U", "DD", "PK", "MODE", "DM", "NL")} |
                 {"loss": loss, "ref": ref, "rel": abs(loss - ref) / ref}), flush=True)

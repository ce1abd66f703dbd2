"""Loss trajectory of a bench workload, step-by-step vs pipelined (run_steps)
from the same initial state: equal up to atomics-order noise if the
cross-iteration dependencies of the pipelined schedule are complete."""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2202_01306_b200 as H
from paper_2202_01306_b200.model import GPT_PRESETS, gpt_machine, gpt_profiles, synthetic_batch
from paper_2202_01306_b200.runtime import HarmonyRuntime
import bench

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="gpt2-xl-dp")
ap.add_argument("--steps", type=int, default=8)
a = ap.parse_args()
preset, D, u, lpp, alpha_gib, mode, *_ = bench.WORKLOADS[a.workload]
spec = GPT_PRESETS[preset]
R = spec.n_layer
packs = tuple((i, min(i + lpp, R) - 1) for i in range(0, R, lpp))
mach = gpt_machine(1, alpha_bytes=alpha_gib << 30)
prof = gpt_profiles(spec)
g = H.generate_task_graph(H.Configuration(u, packs, u, packs, D, H.Mode(mode)), mach, prof)
tok, lab = synthetic_batch(spec, D)
td, ld = torch.from_numpy(tok).cuda(), torch.from_numpy(lab).cuda()
rt = HarmonyRuntime(spec, alpha_bytes=alpha_gib << 30)
big = spec.total_params() > 4_000_000_000
out = {}
for how in ("step", "pipelined"):
    rt.init_weights(0, device="cuda" if big else None)
    rt.k[:] = 0.0
    rt.lib.hm_runtime_set_step(rt.handle, 0)
    if rt.plan is None:
        rt.load(g, mach, prof)
    if how == "step":
        out[how] = [round(rt.step(td, ld), 5) for _ in range(a.steps)]
    else:
        out[how] = [round(x, 5) for x in rt.run_steps(a.steps, td, ld)[0]]
    print(json.dumps({how: out[how]}), flush=True)

"""Run the bench workload for a few iterations (eager or graph mode) and dump
the measured trace of the last iteration as JSON for timeline analysis."""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2202_01306_b200 as H
from paper_2202_01306_b200.model import GPT_PRESETS, gpt_machine, gpt_profiles, synthetic_batch
from paper_2202_01306_b200.runtime import HarmonyRuntime
from paper_2202_01306_b200 import _native as NL

ap = argparse.ArgumentParser()
ap.add_argument("--graph", type=int, default=1)
ap.add_argument("--iters", type=int, default=4)
ap.add_argument("--d", type=int, default=16)
ap.add_argument("--lpp", type=int, default=8)
ap.add_argument("--u", type=int, default=4)
ap.add_argument("--alpha", type=int, default=32)
ap.add_argument("--out", default="gpurun_out/trace.json")
a = ap.parse_args()
spec = GPT_PRESETS["gpt2-xl"]
packs = tuple((i, min(i + a.lpp, 48) - 1) for i in range(0, 48, a.lpp))
mach = gpt_machine(1, alpha_bytes=a.alpha << 30)
prof = gpt_profiles(spec)
g = H.generate_task_graph(H.Configuration(a.u, packs, a.u, packs, a.d, H.Mode.DP), mach, prof)
rt = HarmonyRuntime(spec, alpha_bytes=a.alpha << 30)
NL.check(rt.lib.hm_runtime_set_graph(rt.handle, a.graph))
rt.init_weights(0)
rt.load(g, mach, prof)
tok, lab = synthetic_batch(spec, a.d)
td, ld = torch.from_numpy(tok).cuda(), torch.from_numpy(lab).cuda()
its = []
for i in range(a.iters):
    rt.step(td, ld)
    its.append(rt.counters()["iteration_ns"] / 1e6)
rep = rt.report()
ev = [[e.resource, e.task, e.kind, e.label, e.start_ns, e.end_ns] for e in rep.trace]
items = rt.measured_items()
led = [[int(x["task"]), int(x["stage"]), int(x["member"]), int(x["tensor"]), int(x["nbytes"]), int(x["start_ns"]), int(x["end_ns"])] for x in items if not x["is_compute"]]
json.dump({"graph": a.graph, "iter_ms": its, "trace": ev, "ledger": led}, open(a.out, "w"))
print(json.dumps({"graph": a.graph, "iter_ms": its}))

import os, sys, json
sys.path.insert(0, os.getcwd())
import torch
import paper_2202_01306_b200 as H
from paper_2202_01306_b200 import _native as NL
from paper_2202_01306_b200.model import GPT_PRESETS, gpt_machine, gpt_profiles, synthetic_batch
from paper_2202_01306_b200.runtime import HarmonyRuntime
spec = GPT_PRESETS["gpt2-xl"]
packs = tuple((i, i + 7) for i in range(0, 48, 8))
mach = gpt_machine(1, alpha_bytes=32 << 30)
prof = gpt_profiles(spec)
g = H.generate_task_graph(H.Configuration(4, packs, 4, packs, 16, H.Mode.DP), mach, prof)
rt = HarmonyRuntime(spec, alpha_bytes=32 << 30)
rt.init_weights(0)
rt.load(g, mach, prof)
tok, lab = synthetic_batch(spec, 16)
td, ld = torch.from_numpy(tok).cuda(), torch.from_numpy(lab).cuda()
for _ in range(3): rt.step(td, ld)
for mode in (1, 0):
    NL.check(rt.lib.hm_runtime_set_graph(rt.handle, mode))
    rt.set_profiling(True); rt.step(td, ld); rt.set_profiling(True); rt.step(td, ld)
    ks = rt.kernel_stats()
    print(json.dumps({"graph": mode, "iter_ms": rt.counters()["iteration_ns"] / 1e6,
                      **{k: round(v["ms"], 2) for k, v in ks.items()},
                      "gemm_tflops": round(ks["gemm"]["flops"] / ks["gemm"]["ms"] / 1e9, 1)}))
    rt.set_profiling(False)

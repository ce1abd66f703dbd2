"""Estimator vs runtime on B200 (the paper reports its
estimator within 5% of real runs): profile the GPT-2 XL layers
on this GPU, fit the reference's affine models, then compare simulate()'s
makespan with the measured iteration for several configurations.

    python tools/estimator_check.py > gpurun_out/estimator.json
"""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2202_01306_b200 as H
from paper_2202_01306_b200.model import GPT_PRESETS, synthetic_batch
from paper_2202_01306_b200.profiling import profile_gpt
from paper_2202_01306_b200.runtime import HarmonyRuntime
from paper_2202_01306_b200.search import SearchSpec, search

spec = GPT_PRESETS[os.environ.get("HM_PRESET", "gpt2-xl")]
t0 = time.time()
prof, samples = profile_gpt(spec, u_values=(1, 2, 4), alpha_bytes=48 << 30)
t_prof = time.time() - t0
print(json.dumps({"profiled_s": round(t_prof, 1), "samples": len(samples),
                  "F_ns_u4_layer5": prof.time_ns("F", 5, 4), "B_ns_u4_layer5": prof.time_ns("B", 5, 4),
                  "U_ns_layer5": prof.time_ns("U", 5, 1)}), flush=True)
# measured link rates when both directions are busy (the estimator has one PCIe figure)
for pcie_gbs in (50e9, 55.5e9):
    mach = H.MachineModel(gpu_count=1, gpu_mem_capacity=48 << 30, pcie_bandwidth=int(pcie_gbs))
    rt = HarmonyRuntime(spec, alpha_bytes=48 << 30)
    rt.init_weights(0)
    for D, lpp, u in ((16, 8, 4), (16, 6, 4), (32, 8, 4), (8, 12, 2)):
        packs = tuple((i, min(i + lpp, spec.n_layer) - 1) for i in range(0, spec.n_layer, lpp))
        cfg = H.Configuration(u, packs, u, packs, D, H.Mode.DP)
        g = H.generate_task_graph(cfg, mach, prof)
        est = H.simulate(g, mach, prof).makespan_ns
        try:
            rt.load(g, mach, prof)
        except H.CapacityViolationError as exc:
            print(json.dumps({"D": D, "layers_per_pack": lpp, "u": u, "skipped": str(exc)}), flush=True)
            continue
        tok, lab = synthetic_batch(spec, D)
        td, ld = torch.from_numpy(tok).cuda(), torch.from_numpy(lab).cuda()
        ts = []
        for _ in range(4):
            rt.step(td, ld)
            ts.append(rt.counters()["iteration_ns"])
        meas = min(ts[1:])
        print(json.dumps({"pcie_model_gbs": pcie_gbs / 1e9, "D": D, "layers_per_pack": lpp, "u": u,
                          "estimate_ms": round(est / 1e6, 2), "measured_ms": round(meas / 1e6, 2),
                          "rel_err": round((est - meas) / meas, 4)}), flush=True)
    rt.close()
# the planner's choice on measured costs
mach = H.MachineModel(gpu_count=1, gpu_mem_capacity=32 << 30, pcie_bandwidth=int(50e9))
t0 = time.time()
res = search(SearchSpec(minibatch=16, mode=H.Mode.DP, u_fmax=4, u_bmax=4), mach, prof)
print(json.dumps({"search_s": round(time.time() - t0, 2), "explored": res.explored,
                  "best": [res.best.u_f, len(res.best.p_f), res.best.u_b, len(res.best.p_b)],
                  "best_estimate_ms": round(res.best_time_ns / 1e6, 2)}), flush=True)

"""Distinct-FB vs Equi-FB on the real runtime (paper §4.3, PAPER.md:1379-1394:
Distinct-FB wins most on CNNs -- 12.3% VGG416, 29.1% ResNet1K on 4x1080Ti).

Profile every layer of a chain on this B200 (the profiler loop), search the
best configuration under each strategy with the fitted costs and a capped
alpha, execute both on the GPU and report estimate vs measured iteration time.

    python tools/fb_experiment.py [--model resnet-fb] [--alpha-gib 2] [--d 32]
"""
import argparse, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2202_01306_b200 as H
from paper_2202_01306_b200.cnn import CNN_PRESETS, cnn_chain
from paper_2202_01306_b200.model import GPT_PRESETS
from paper_2202_01306_b200.profiling import profile_model, synthetic_inputs
from paper_2202_01306_b200.runtime import HarmonyRuntime
from paper_2202_01306_b200.search import SearchSpec, Strategy, search

ap = argparse.ArgumentParser()
ap.add_argument("--model", default="resnet-fb")
ap.add_argument("--alpha-gib", type=float, default=2.0)
ap.add_argument("--d", type=int, default=32)
ap.add_argument("--umax", type=int, default=16)
ap.add_argument("--iters", type=int, default=4)
ap.add_argument("--pack-layers", type=int, default=1, help="layers per profiling pack (apportioned by FLOPs)")
a = ap.parse_args()
presets = dict(CNN_PRESETS, **GPT_PRESETS)
# an irregular chain: wide, high-resolution stages early (big activations, few
# weights), narrow deep ones late (small activations, many weights)
presets["resnet-fb"] = cnn_chain("resnet-fb", 64, [64, 128, 256, 512], [6, 6, 6, 6], 1000, "res")
spec = presets[a.model]
alpha = int(a.alpha_gib * (1 << 30))
t0 = time.time()
prof, samples = profile_model(spec, u_values=(1, 2, 4, 8, 16), u_max=16, stride=4, alpha_bytes=48 << 30,
                              pack_layers=a.pack_layers)
print(json.dumps({"model": spec.name, "layers": spec.n_layer, "params_M": round(spec.total_params() / 1e6, 1),
                  "profiled_s": round(time.time() - t0, 1), "samples": len(samples)}), flush=True)
mach = H.MachineModel(gpu_count=1, gpu_mem_capacity=alpha, pcie_bandwidth=int(50e9))
results = {}
for strat in (Strategy.EQUI_FB, Strategy.DISTINCT_FB):
    t0 = time.time()
    res = search(SearchSpec(minibatch=a.d, mode=H.Mode.PP, strategy=strat, u_fmax=a.umax, u_bmax=a.umax), mach, prof)
    cfg = res.best
    row = {"strategy": strat.value, "search_s": round(time.time() - t0, 2), "explored": res.explored,
           "u_f": cfg.u_f, "packs_f": len(cfg.p_f), "u_b": cfg.u_b, "packs_b": len(cfg.p_b),
           "estimate_ms": round(res.best_time_ns / 1e6, 2)}
    g = H.generate_task_graph(cfg, mach, prof)
    rt = HarmonyRuntime(spec, alpha_bytes=48 << 30)
    try:
        rt.init_weights(0)
        rt.load(g, mach, prof)
        inp, lab = synthetic_inputs(spec, a.d)
        if isinstance(inp, torch.Tensor):
            inp, lab = inp.cuda(), lab.cuda()
        else:
            inp, lab = torch.from_numpy(inp).cuda(), torch.from_numpy(lab).cuda()
        ts = []
        for _ in range(a.iters):
            rt.step(inp, lab)
            ts.append(rt.counters()["iteration_ns"] / 1e6)
        row["measured_ms"] = round(min(ts[1:]), 2)
        row["device_bytes"] = rt.counters()["device_bytes"]
        row["ledger_equals_plan"] = rt.report().ledger == H.simulate(g, mach, prof).ledger
    finally:
        rt.close()
    row["est_rel_err"] = round((row["estimate_ms"] - row["measured_ms"]) / row["measured_ms"], 4)
    results[strat.value] = row
    print(json.dumps(row), flush=True)
e, d = results["equi_fb"], results["distinct_fb"]
print(json.dumps({"distinct_vs_equi_measured_speedup": round(e["measured_ms"] / d["measured_ms"], 4),
                  "distinct_vs_equi_estimated_speedup": round(e["estimate_ms"] / d["estimate_ms"], 4)}), flush=True)

"""Per-iteration time of one bench workload three ways (CUDA events around
whole iterations, device-resident tokens):
  graph      rt.step() with the iteration recorded once and replayed as a CUDA graph
  eager      rt.step() with graphs off (every launch from the host)
  pipelined  rt.run_steps(n) (eager enqueue of n iterations, cross-iteration overlap)

    python tools/graph_vs_eager.py [workload] [steps]"""
import json
import os
import sys
import time

ROOT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..")
sys.path.insert(0, ROOT)


def main() -> None:
    import torch
    import bench
    import paper_2202_01306_b200 as H
    from paper_2202_01306_b200.model import GPT_PRESETS, gpt_machine, gpt_profiles, synthetic_batch
    from paper_2202_01306_b200.runtime import HarmonyRuntime
    workload = sys.argv[1] if len(sys.argv) > 1 else "gpt2-xl-dp-d64"
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
    preset, per_gpu, u, lpp, alpha_gib, mode, *_ = bench.WORKLOADS[workload]
    spec = GPT_PRESETS[preset]
    R = spec.n_layer
    packs = tuple((i, min(i + lpp, R) - 1) for i in range(0, R, lpp))
    machine = gpt_machine(1, alpha_bytes=alpha_gib << 30)
    prof = gpt_profiles(spec)
    graph = H.generate_task_graph(H.Configuration(u, packs, u, packs, per_gpu, H.Mode(mode)), machine, prof)
    rt = HarmonyRuntime(spec, alpha_bytes=alpha_gib << 30, device=0)
    rt.init_weights(0, device="cuda")
    rt.load(graph, machine, prof)
    tok, lab = synthetic_batch(spec, per_gpu)
    tok_d, lab_d = torch.from_numpy(tok).cuda(), torch.from_numpy(lab).cuda()
    out = {"workload": workload, "steps": steps}
    for name, use_graph in (("graph", 1), ("eager", 0)):
        rt.lib.hm_runtime_set_graph(rt.handle, use_graph)
        for _ in range(2):
            rt.step(tok_d, lab_d)
        torch.cuda.synchronize()
        t = 0.0
        for _ in range(steps):
            rt.step(tok_d, lab_d)
            t += rt.counters()["iteration_ns"] / 1e6
        out[f"{name}_ms"] = round(t / steps, 2)
    rt.lib.hm_runtime_set_graph(rt.handle, 1)
    _, t_s = rt.run_steps(steps, tok_d, lab_d)
    out["pipelined_ms"] = round(t_s * 1e3 / steps, 2)
    print(json.dumps(out), flush=True)
    rt.close()


if __name__ == "__main__":
    main()

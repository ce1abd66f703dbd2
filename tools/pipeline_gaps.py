"""Timeline of one pipelined iteration of the bench workload: per-stream busy
fraction and the H2D queue in order with the idle gap before each transfer
(what the swap-in stream waited for).  Writes gpurun_out/pipeline.json."""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2202_01306_b200 as H
from paper_2202_01306_b200.model import GPT_PRESETS, gpt_machine, gpt_profiles, synthetic_batch
from paper_2202_01306_b200.runtime import HarmonyRuntime

import bench  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="gpt2-xl-dp")
ap.add_argument("--steps", type=int, default=4)
ap.add_argument("--out", default="gpurun_out/pipeline.json")
a = ap.parse_args()
preset, a.d, a.u, a.lpp, a.alpha, mode, *_ = bench.WORKLOADS[a.workload]
from paper_2202_01306_b200.cnn import CNN_PRESETS, cnn_profiles, synthetic_images  # noqa: E402
is_cnn = preset in CNN_PRESETS
spec = CNN_PRESETS[preset] if is_cnn else GPT_PRESETS[preset]
R = spec.n_layer
packs = tuple((i, min(i + a.lpp, R) - 1) for i in range(0, R, a.lpp))
mach = gpt_machine(1, alpha_bytes=a.alpha << 30)
prof = cnn_profiles(spec) if is_cnn else gpt_profiles(spec)
g = H.generate_task_graph(H.Configuration(a.u, packs, a.u, packs, a.d, H.Mode(mode)), mach, prof)
rt = HarmonyRuntime(spec, alpha_bytes=a.alpha << 30)
rt.init_weights(0, device="cuda" if spec.total_params() > 4_000_000_000 and not is_cnn else None)
rt.load(g, mach, prof)
if is_cnn:
    img, lab = synthetic_images(spec, a.d)
    td, ld = img.cuda(), lab.cuda()
else:
    tok, lab = synthetic_batch(spec, a.d)
    td, ld = torch.from_numpy(tok).cuda(), torch.from_numpy(lab).cuda()
rt.run_steps(2, td, ld)
_, secs = rt.run_steps(a.steps, td, ld)
c = rt.counters()
items = rt.measured_items()
types = {t.index: t.type.value for t in g.tasks}
rows = []
for x in items:
    kind = "compute" if x["is_compute"] else ("h2d" if int(x["stage"]) == 0 else "d2h")
    if kind == "compute" and types[int(x["task"])] == "U":
        kind = "update"
    rows.append({"kind": kind, "task": int(x["task"]), "ttype": types[int(x["task"])], "member": int(x["member"]),
                 "tensor": int(x["tensor"]), "bytes": int(x["nbytes"]), "t0": x["start_ns"] / 1e6,
                 "t1": x["end_ns"] / 1e6})
it = c["iteration_ns"] / 1e6
print(json.dumps({"ms_per_step_pipelined": secs * 1e3 / a.steps, "last_iter_ms": it}))
for k in ("h2d", "d2h", "compute", "update"):
    rs = sorted([r for r in rows if r["kind"] == k], key=lambda r: r["t0"])
    busy = sum(r["t1"] - r["t0"] for r in rs)
    print(k, "busy ms", round(busy, 1))
    if k in ("h2d", "d2h"):
        prev = rs[0]["t0"] if rs else 0
        for r in rs:
            gb = r["bytes"] / 1e9
            print(f"  {k} task {r['task']:3d}{r['ttype']} tensor {r['tensor']} {gb:6.3f} GB  start {r['t0']:8.1f} "
                  f"end {r['t1']:8.1f}  gap {r['t0'] - prev:7.1f}  GB/s {gb / max(1e-9, (r['t1'] - r['t0']) / 1e3):6.1f}")
            prev = r["t1"]
tasks = {}
for r in rows:
    if r["kind"] in ("compute", "update"):
        t = tasks.setdefault(r["task"], [1e18, -1e18, r["ttype"]])
        t[0] = min(t[0], r["t0"]); t[1] = max(t[1], r["t1"])
for k in sorted(tasks):
    print(f"  task {k:3d}{tasks[k][2]} compute {tasks[k][0]:8.1f} -> {tasks[k][1]:8.1f}")
json.dump(rows, open(a.out, "w"))

"""Documents written by the REFERENCE's fileio (wrapsched, /root/reference)
for tests/test_fileio.py.  Run here: python oracle/make_golden_fileio.py"""
import json, os, sys
sys.path.insert(0, "/root/reference/pkg/src")
import wrapsched as W
from wrapsched import fileio as F
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
prof = W.synth_profiles(W.SynthSpec(layer_count=6, preset="irregular", seed=3, u_max=8, w_bytes=1 << 20,
                                    act_bytes_per_u=1 << 12, time_intercept_ns=1000))
m = W.MachineModel(gpu_count=2, gpu_mem_capacity=1 << 40, pcie_bandwidth=16 << 30, root_link_bandwidth=8 << 30)
cfg = W.Configuration(2, ((0, 1), (2, 3), (4, 5)), 2, ((0, 2), (3, 3), (4, 5)), 6, W.Mode.PP)
g = W.generate_task_graph(cfg, m, prof)
rep = W.simulate(g, m, prof)
samples = W.synth_samples(W.SynthSpec(layer_count=2, u_max=4), stride=2)
docs = {"machine": F.machine_to_doc(m), "profile_set": F.profileset_to_doc(prof),
        "configuration": F.config_to_doc(cfg), "task_graph": F.taskgraph_to_doc(g),
        "sim_report": F.report_to_doc(rep), "trace_csv": F.trace_to_csv(rep),
        "profile_samples": F.samples_to_doc(samples, seed=7)}
out = os.path.join(ROOT, "tests", "golden", "fileio.json")
json.dump(docs, open(out, "w"), separators=(",", ":"))
print("wrote", out, os.path.getsize(out))

"""Golden vectors for the configuration search (caller of the hot path),
produced by running the REFERENCE's `search` (wrapsched, /root/reference) on
the reference tests' profile presets.  Run here: python oracle/make_golden_search.py"""
import json, os, sys
sys.path.insert(0, "/root/reference/pkg/src")
import wrapsched as W
from wrapsched.search import SearchSpec, Strategy, search, greedy_baseline
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
MiB = 1 << 20

def irregular(seed=5, **kw):
    d = dict(layer_count=12, preset="irregular", seed=seed, u_max=16, base_time_ns=500_000,
             time_intercept_ns=20_000_000, ratio_b=1.5, mem_ratio_b=4.0, w_bytes=64 * MiB,
             act_bytes_per_u=24 * MiB, k_ratio=2.0)
    d.update(kw)
    return d

cases = []
for name, synth, n, alpha, beta, spec in [
    ("irregular_pp_distinct", irregular(), 4, 1200 * MiB, 8 << 30, dict(minibatch=16)),
    ("irregular_pp_equi", irregular(), 4, 1200 * MiB, 8 << 30, dict(minibatch=16, strategy="equi_fb")),
    ("irregular_seed2_bounds", irregular(seed=2), 4, 1200 * MiB, 8 << 30, dict(minibatch=16, u_fmax=6, u_bmax=4)),
    ("irregular_stride2", irregular(), 4, 1200 * MiB, 8 << 30, dict(minibatch=16, stride=2)),
    ("uniform_dp", dict(layer_count=4, preset="uniform", u_max=16, base_time_ns=1_000_000,
                        w_bytes=4 * MiB, act_bytes_per_u=64 << 10), 4, 1 << 40, 16 << 30,
     dict(minibatch=10, mode="dp")),
    ("r96_pp", dict(layer_count=24, preset="irregular", seed=3, u_max=8, base_time_ns=1_000_000,
                    time_intercept_ns=5_000_000, w_bytes=32 * MiB, act_bytes_per_u=8 * MiB), 4, 600 * MiB,
     16 << 30, dict(minibatch=16)),
]:
    prof = W.synth_profiles(W.SynthSpec(**synth))
    m = W.MachineModel(gpu_count=n, gpu_mem_capacity=alpha, pcie_bandwidth=beta)
    sp = dict(spec)
    if "mode" in sp: sp["mode"] = W.Mode(sp["mode"])
    if "strategy" in sp: sp["strategy"] = Strategy(sp["strategy"])
    s = SearchSpec(**sp)
    res = search(s, m, prof)
    gcfg, gt = greedy_baseline(s, m, prof)
    cfg = res.best
    cases.append({"name": name, "synth": synth, "machine": [n, alpha, beta], "spec": spec,
                  "best": [cfg.u_f, [list(p) for p in cfg.p_f], cfg.u_b, [list(p) for p in cfg.p_b]],
                  "best_time_ns": res.best_time_ns, "explored": res.explored,
                  "log": [[c.u_f, c.u_b, c.pf_count, c.pb_count, c.time_ns, c.note] for c in res.log],
                  "greedy": [gcfg.u_f, [list(p) for p in gcfg.p_f], gcfg.u_b, [list(p) for p in gcfg.p_b], gt]})
out = os.path.join(ROOT, "tests", "golden", "search.json")
json.dump({"generator": "oracle/make_golden_search.py", "cases": cases}, open(out, "w"), separators=(",", ":"))
print("wrote", len(cases), "cases", os.path.getsize(out))

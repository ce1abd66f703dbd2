"""Generate tests/golden/*.json by running the REFERENCE planner (wrapsched,
imported read-only from /root/reference/pkg/src).  Run here, in the build
container; the GPU box never reads /root/reference.

    python oracle/make_golden.py

Each case stores its inputs (configuration, machine, affine profile
parameters) and the reference's outputs: per-task structure, unroll order,
the ledger rows in the SURVEY §8c comparison form, makespan, volumes and
the trace.  tests/test_oracle.py pins oracle/schedule.py against these;
tests/test_planner.py pins the product (Python API + native plan).
"""

from __future__ import annotations

import json
import os
import random
import sys

REF = "/root/reference/pkg/src"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REF)
sys.path.insert(0, ROOT)

import wrapsched as W  # noqa: E402
import wrapsched.simulator as WS  # noqa: E402

from paper_2202_01306_b200.model import GPT_PRESETS, gpt_profiles  # noqa: E402  (shapes only)


def prof_doc(p) -> dict:
    aff = lambda m: [m.slope, m.intercept]
    return {"layer_count": p.layer_count, "u_max_f": p.u_max_f, "u_max_b": p.u_max_b,
            "time": {f"{l},{ps}": aff(m) for (l, ps), m in sorted(p._time.items())},
            "mem": {f"{l},{ps}": aff(m) for (l, ps), m in sorted(p._mem.items())},
            "x": {str(l): aff(m) for l, m in sorted(p._x.items())},
            "y": {str(l): aff(m) for l, m in sorted(p._y.items())},
            "w": {str(l): v for l, v in sorted(p._w.items())},
            "dw": {str(l): v for l, v in sorted(p._dw.items())},
            "k": {str(l): v for l, v in sorted(p._k.items())}}


def ch_doc(ch) -> list:
    return [ch.kind.value, ch.src_task, ch.dst_task, ch.src_layer]


def case(name, cfg, machine, prof, check_memory=False) -> dict:
    g = W.generate_task_graph(cfg, machine, prof)
    items = WS._build_items(g, machine, prof)
    ledger = sorted([it.task, it.key[1], it.key[2], it.tensor.value, it.channel.value,
                     list(it.resources), it.nbytes, it.gpu] for it in items if it.kind != "compute")
    rep = W.simulate(g, machine, prof)
    return {
        "name": name,
        "config": {"u_f": cfg.u_f, "p_f": [list(p) for p in cfg.p_f], "u_b": cfg.u_b,
                   "p_b": [list(p) for p in cfg.p_b], "minibatch": cfg.minibatch,
                   "mode": cfg.mode.value},
        "machine": {"gpu_count": machine.gpu_count, "gpu_mem_capacity": machine.gpu_mem_capacity,
                    "pcie_bandwidth": machine.pcie_bandwidth,
                    "root_link_bandwidth": machine.root_link_bandwidth,
                    "p2p_groups": [list(x) for x in machine.p2p_groups],
                    "cpu_offload_update": machine.cpu_offload_update,
                    "update_cpu_rate": machine.update_cpu_rate},
        "profiles": prof_doc(prof),
        "expect": {
            "tasks": [{"index": t.index, "pack": list(t.pack), "type": t.type.value,
                       "group": list(t.group), "device": list(t.device), "recompute": t.recompute,
                       "inputs": [[k.value, [[l, *ch_doc(c)] for l, c in e.items()]]
                                  for k, e in t.inputs.items()],
                       "outputs": [[k.value, [[l, *ch_doc(c)] for l, c in e.items()]]
                                   for k, e in t.outputs.items()]} for t in g.tasks],
            "unroll": W.unroll_schedule(g),
            "ledger": ledger,
            "makespan_ns": rep.makespan_ns,
            "channel_volumes": rep.channel_volumes,
            "tensor_volumes": rep.tensor_volumes,
            "per_gpu_volumes": {str(k): v for k, v in rep.per_gpu_volumes.items()},
            "gpu_busy_ns": {str(k): v for k, v in rep.gpu_busy_ns.items()},
            "trace": [[e.resource, e.task, e.kind, e.label, e.start_ns, e.end_ns] for e in rep.trace],
            "caveats": list(rep.caveats),
        },
    }


def table(r, x=0, y=0, w=0, k=0, tf=1_000_000, tb=2_000_000, tu=100_000, u_max=16, dw=None):
    """Constant-in-u ProfileSet (the reference's conftest.table_profiles)."""
    A = W.profiler.AffineModel
    tm, mm = {}, {}
    for i in range(r):
        tm[(i, "F")], tm[(i, "B")], tm[(i, "U")] = A(0.0, tf), A(0.0, tb), A(0.0, tu)
        for p in ("F", "B", "U"):
            mm[(i, p)] = A(0.0, 0)
    return W.ProfileSet(r, tm, mm, {i: A(float(x), 0.0) for i in range(r)},
                        {i: A(float(y), 0.0) for i in range(r)}, {i: w for i in range(r)},
                        {i: (w if dw is None else dw) for i in range(r)}, {i: k for i in range(r)},
                        u_max, u_max)


def mach(n, **kw):
    return W.MachineModel(gpu_count=n, gpu_mem_capacity=kw.pop("cap", 1 << 40),
                          pcie_bandwidth=kw.pop("pcie", 16 << 30), **kw)


def cfg(pf, pb, uf, ub, d, mode="pp"):
    return W.Configuration(uf, tuple(map(tuple, pf)), ub, tuple(map(tuple, pb)), d, W.Mode(mode))


def rand_packs(rng, r):
    cuts = sorted(rng.sample(range(1, r), rng.randint(0, r - 1))) if r > 1 else []
    b = [0] + cuts + [r]
    return [(b[i], b[i + 1] - 1) for i in range(len(b) - 1)]


def main() -> None:
    cases = []
    # c1 probe (SURVEY §8c "Tiny-config ledger"): uniform block W, x = y = 131,072 B/sample
    tiny_w = 3_159_040
    tiny = table(4, x=131_072, y=131_072, w=tiny_w, k=2 * tiny_w)
    cases.append(case("c1_tiny_probe_pp_n1", cfg([(0, 1), (2, 3)], [(0, 1), (2, 3)], 4, 4, 16),
                      mach(1), tiny))
    cases.append(case("c1_tiny_probe_pp_n2", cfg([(0, 1), (2, 3)], [(0, 1), (2, 3)], 4, 4, 16),
                      mach(2), tiny))
    # reference taskgraph tests (test_taskgraph.py:31-156) on synth profiles
    sp = W.synth_profiles(W.SynthSpec(layer_count=6, u_max=8, w_bytes=1 << 20, act_bytes_per_u=1 << 10))
    three = [(0, 1), (2, 3), (4, 5)]
    cases.append(case("ref_wraparound_3packs_2gpus", cfg(three, three, 1, 1, 2), mach(2), sp))
    six = [(i, i) for i in range(6)]
    cases.append(case("ref_six_singletons_2gpus", cfg(six, six, 1, 1, 2), mach(2), sp))
    sp4 = W.synth_profiles(W.SynthSpec(layer_count=4, u_max=8, w_bytes=1 << 20, act_bytes_per_u=1 << 10))
    cases.append(case("ref_degenerate_single_pack", cfg([(0, 3)], [(0, 3)], 1, 1, 2), mach(1), sp4))
    cases.append(case("ref_dp_4gpus", cfg([(0, 1), (2, 3)], [(0, 1), (2, 3)], 1, 1, 8, "dp"),
                      mach(4), sp4))
    cases.append(case("ref_weight_once", cfg([(0, 2), (3, 5)], [(0, 2), (3, 5)], 2, 2, 8), mach(2), sp))
    cases.append(case("ref_stash_edges", cfg([(0, 3), (4, 5)], [(0, 1), (2, 3), (4, 5)], 1, 1, 2),
                      mach(2), sp))
    # SURVEY §8(a') edge cases: R=4, x=y=1000 B/sample, W=10,000, K=20,000
    e = table(4, x=1000, y=1000, w=10_000, k=20_000)
    cases.append(case("edge_uf_ne_ub", cfg([(0, 1), (2, 3)], [(0, 1), (2, 3)], 4, 2, 8), mach(2), e))
    cases.append(case("edge_remainder_group", cfg([(0, 1), (2, 3)], [(0, 1), (2, 3)], 4, 4, 10),
                      mach(1), e))
    cases.append(case("edge_dp_uneven", cfg([(0, 1), (2, 3)], [(0, 1), (2, 3)], 2, 2, 10, "dp"),
                      mach(4), e))
    cases.append(case("edge_f_pack_two_heads", cfg([(0, 2), (3, 3)], [(0, 0), (1, 2), (3, 3)], 2, 2, 4),
                      mach(3), e))
    cases.append(case("edge_zero_stash", cfg([(0, 1), (2, 3)], [(0, 1), (2, 3)], 2, 2, 4),
                      mach(2), table(4, x=0, y=1000, w=10_000, k=20_000)))
    cases.append(case("edge_root_groups", cfg(three, three, 2, 2, 4),
                      mach(4, p2p_groups=((0, 1), (2, 3)), root_link_bandwidth=8 << 30), sp))
    cases.append(case("edge_cpu_offload", cfg(three, three, 2, 1, 4),
                      mach(2, cpu_offload_update=True), sp))
    # GPT shapes of the BASELINE configs (real W/K/x from the runtime's byte model)
    for name, preset, packs, u, d, n, mode in (
            ("c1_tiny_gpt_pp_n1", "tiny", [(0, 1), (2, 3)], 4, 16, 1, "pp"),
            ("c2_bert_large_pp_n1", "bert-large", [(0, 7), (8, 15), (16, 23)], 8, 64, 1, "pp"),
            ("c3_gpt2xl_dp_n8", "gpt2-xl", [(0, 15), (16, 31), (32, 47)], 4, 128, 8, "dp"),
            ("c3_gpt2xl_pp_n4", "gpt2-xl", [(0, 11), (12, 23), (24, 35), (36, 47)], 4, 64, 4, "pp"),
            ("c4_gpt40b_pp_n8", "gpt-40b", [(i * 6, i * 6 + 5) for i in range(8)], 4, 64, 8, "pp")):
        prof = W.ProfileSet(**_to_ref_kwargs(gpt_profiles(GPT_PRESETS[preset], u_max=64)))
        cases.append(case(name, cfg(packs, packs, u, u, d, mode),
                          mach(n, pcie=55_000_000_000), prof))
    # randomized (test_taskgraph.py:169-192 style, plus irregular profiles)
    rng = random.Random(20261017)
    for i in range(60):
        r = rng.randint(1, 9)
        n = rng.randint(1, 4)
        d = rng.randint(1, 12)
        mode = rng.choice(["pp", "dp"])
        pb = rand_packs(rng, r)
        pf = (rand_packs(rng, pb[-1][0]) if pb[-1][0] > 0 else []) + [pb[-1]]
        uf, ub = rng.randint(1, d), rng.randint(1, d)
        prof = W.synth_profiles(W.SynthSpec(
            layer_count=r, u_max=16, preset=rng.choice(["uniform", "irregular"]), seed=i,
            w_bytes=rng.randint(1, 1 << 22), act_bytes_per_u=rng.randint(0, 1 << 14),
            time_intercept_ns=rng.randint(0, 5000)))
        groups = ()
        if n == 4 and rng.random() < 0.5:
            groups = ((0, 1), (2, 3))
        m = mach(n, pcie=rng.choice([16 << 30, 12_345_678_901, 55_000_000_000]),
                 root_link_bandwidth=rng.choice([0, 20 << 30, 5 << 30]), p2p_groups=groups,
                 cpu_offload_update=rng.random() < 0.25)
        cases.append(case(f"random_{i:02d}", cfg(pf, pb, uf, ub, d, mode), m, prof))
    out = os.path.join(ROOT, "tests", "golden", "schedule_ledger.json")
    with open(out, "w") as f:
        json.dump({"generator": "oracle/make_golden.py", "reference": "wrapsched 0.1.0 @ /root/reference",
                   "cases": cases}, f, separators=(",", ":"))
    print(f"wrote {len(cases)} cases to {out} ({os.path.getsize(out)} bytes)")


def _to_ref_kwargs(p) -> dict:
    A = W.profiler.AffineModel
    conv = lambda d: {k: A(m.slope, m.intercept) for k, m in d.items()}
    return dict(layer_count=p.layer_count, time_models=conv(p._time), mem_models=conv(p._mem),
                x_models=conv(p._x), y_models=conv(p._y), w_bytes=dict(p._w), dw_bytes=dict(p._dw),
                k_bytes=dict(p._k), u_max_f=p.u_max_f, u_max_b=p.u_max_b)


if __name__ == "__main__":
    main()

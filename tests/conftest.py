import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (run with -m gpu on the GPU box)")
    config.addinivalue_line("markers", "slow: long-running test")


_cache = {}


def golden(name):
    if name not in _cache:
        with open(os.path.join(GOLDEN, name)) as f:
            _cache[name] = json.load(f)
    return _cache[name]


def golden_cases():
    return golden("schedule_ledger.json")["cases"]


def product_inputs(case):
    """(Configuration, MachineModel, ProfileSet) of the product from a golden case."""
    import paper_2202_01306_b200 as H
    c, m, p = case["config"], case["machine"], case["profiles"]
    A = H.AffineModel
    split = lambda k: (int(k.split(",")[0]), k.split(",")[1])
    prof = H.ProfileSet(
        p["layer_count"],
        {split(k): A(*v) for k, v in p["time"].items()},
        {split(k): A(*v) for k, v in p["mem"].items()},
        {int(k): A(*v) for k, v in p["x"].items()},
        {int(k): A(*v) for k, v in p["y"].items()},
        {int(k): v for k, v in p["w"].items()}, {int(k): v for k, v in p["dw"].items()},
        {int(k): v for k, v in p["k"].items()}, p["u_max_f"], p["u_max_b"])
    mach = H.MachineModel(gpu_count=m["gpu_count"], gpu_mem_capacity=m["gpu_mem_capacity"],
                          pcie_bandwidth=m["pcie_bandwidth"],
                          root_link_bandwidth=m["root_link_bandwidth"],
                          p2p_groups=tuple(tuple(g) for g in m["p2p_groups"]),
                          cpu_offload_update=m["cpu_offload_update"],
                          update_cpu_rate=m["update_cpu_rate"])
    cfg = H.Configuration(c["u_f"], tuple(map(tuple, c["p_f"])), c["u_b"],
                          tuple(map(tuple, c["p_b"])), c["minibatch"], H.Mode(c["mode"]))
    return cfg, mach, prof


def oracle_inputs(case):
    """Plain-dict inputs of oracle/schedule.py from a golden case."""
    m, p = case["machine"], case["profiles"]
    R = p["layer_count"]
    u_top = max(case["config"]["minibatch"], 1)

    def aff(v, u):
        return max(0, round(v[0] * u + v[1]))

    def tab(models):
        return [[aff(models[str(L)], u) if str(L) in models else -1 for u in range(u_top + 1)]
                for L in range(R)]

    def ttab(ps):
        return [[aff(p["time"][f"{L},{ps}"], 1 if ps == "U" else u) for u in range(u_top + 1)]
                for L in range(R)]

    prof = {"x": tab(p["x"]), "y": tab(p["y"]),
            "w": [p["w"][str(L)] for L in range(R)], "dw": [p["dw"][str(L)] for L in range(R)],
            "k": [p["k"][str(L)] for L in range(R)], "tF": ttab("F"), "tB": ttab("B"),
            "tU": ttab("U")}
    group_of = {}
    for i, g in enumerate(m["p2p_groups"]):
        for x in g:
            group_of[x] = i
    mach = {"gpu_count": m["gpu_count"], "pcie": m["pcie_bandwidth"],
            "root": m["root_link_bandwidth"],
            "p2p_group_of": [group_of[i] for i in range(m["gpu_count"])],
            "cpu_offload_update": m["cpu_offload_update"], "update_cpu_rate": m["update_cpu_rate"]}
    return case["config"], mach, prof


@pytest.fixture(scope="session")
def native_lib():
    from paper_2202_01306_b200 import _native
    return _native.lib()


def collect_or_fail(q, procs, timeout: float):
    """Wait for the rank processes' result on ``q``; fail at once (with the
    exit codes) if a rank dies first instead of waiting out the timeout."""
    import queue as _queue
    import time as _time
    t_end = _time.monotonic() + timeout
    while True:
        try:
            return q.get(timeout=2.0)
        except _queue.Empty:
            dead = [(i, p.exitcode) for i, p in enumerate(procs) if p.exitcode is not None and p.exitcode != 0]
            if dead:
                for p in procs:
                    if p.is_alive():
                        p.kill()
                raise AssertionError(f"rank process(es) died before reporting: {dead}")
            if _time.monotonic() > t_end:
                for p in procs:
                    if p.is_alive():
                        p.kill()
                raise AssertionError(f"no result from the ranks within {timeout} s")

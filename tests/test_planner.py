"""Product planner parity: the Python API (generate_task_graph, unroll) and the
native swap plan (ledger, estimator) against the reference's golden outputs,
and against the oracle on fresh random configurations."""

import random

import pytest

import paper_2202_01306_b200 as H
from conftest import golden_cases, oracle_inputs, product_inputs
from oracle import schedule as O
from paper_2202_01306_b200.lowering import NativePlan, ledger_rows


def _task_doc(t):
    def ents(d):
        return [[k.value, [[l, c.kind.value, c.src_task, c.dst_task, c.src_layer]
                           for l, c in e.items()]] for k, e in d.items()]
    return {"index": t.index, "pack": list(t.pack), "type": t.type.value, "group": list(t.group),
            "device": list(t.device), "recompute": t.recompute, "inputs": ents(t.inputs),
            "outputs": ents(t.outputs)}


@pytest.mark.parametrize("case", golden_cases(), ids=lambda c: c["name"])
def test_schedule_and_ledger_bit_exact(case):
    cfg, mach, prof = product_inputs(case)
    g = H.generate_task_graph(cfg, mach, prof)
    exp = case["expect"]
    assert [_task_doc(t) for t in g.tasks] == exp["tasks"]
    assert H.unroll_schedule(g) == exp["unroll"]
    rep = H.simulate(g, mach, prof)
    assert [list(r[:5]) + [list(r[5])] + list(r[6:]) for r in rep.ledger] == exp["ledger"]
    assert rep.makespan_ns == exp["makespan_ns"]
    assert rep.channel_volumes == exp["channel_volumes"]
    assert rep.tensor_volumes == exp["tensor_volumes"]
    assert {str(k): v for k, v in rep.per_gpu_volumes.items()} == exp["per_gpu_volumes"]
    assert {str(k): v for k, v in rep.gpu_busy_ns.items()} == exp["gpu_busy_ns"]
    assert [[e.resource, e.task, e.kind, e.label, e.start_ns, e.end_ns] for e in rep.trace] == exp["trace"]
    assert list(rep.caveats) == exp["caveats"]


def _rand_cfg(rng):
    r = rng.randint(1, 12)
    pb_cuts = sorted(rng.sample(range(1, r), rng.randint(0, r - 1))) if r > 1 else []
    b = [0] + pb_cuts + [r]
    pb = [(b[i], b[i + 1] - 1) for i in range(len(b) - 1)]
    head = pb[-1][0]
    pf = []
    if head:
        c2 = sorted(rng.sample(range(1, head), rng.randint(0, head - 1))) if head > 1 else []
        b2 = [0] + c2 + [head]
        pf = [(b2[i], b2[i + 1] - 1) for i in range(len(b2) - 1)]
    pf.append(pb[-1])
    d = rng.randint(1, 16)
    return r, {"u_f": rng.randint(1, d), "p_f": pf, "u_b": rng.randint(1, d), "p_b": pb,
               "minibatch": d, "mode": rng.choice(["pp", "dp"])}


def test_native_plan_matches_oracle_random():
    """Product (native) vs oracle on 150 fresh random graphs; the oracle is
    itself pinned to the reference by test_oracle.py."""
    rng = random.Random(7)
    for trial in range(150):
        r, c = _rand_cfg(rng)
        n = rng.randint(1, 5)
        spec = H.SynthSpec(layer_count=r, u_max=16, preset=rng.choice(["uniform", "irregular"]),
                           seed=trial, w_bytes=rng.randint(1, 1 << 24),
                           act_bytes_per_u=rng.randint(0, 1 << 16),
                           time_intercept_ns=rng.randint(0, 10_000))
        prof = H.synth_profiles(spec)
        mach = H.MachineModel(gpu_count=n, gpu_mem_capacity=1 << 40,
                              pcie_bandwidth=rng.choice([16 << 30, 55_000_000_000, 999_999_937]),
                              root_link_bandwidth=rng.choice([0, 7 << 30]),
                              cpu_offload_update=rng.random() < 0.2)
        cfg = H.Configuration(c["u_f"], tuple(c["p_f"]), c["u_b"], tuple(c["p_b"]),
                              c["minibatch"], H.Mode(c["mode"]))
        g = H.generate_task_graph(cfg, mach, prof)
        plan = NativePlan(g, mach, prof)
        ms = plan.simulate()
        rows = ledger_rows(plan.items(), n)
        plan.close()
        # oracle on the same inputs
        case = {"config": c, "machine": {
            "gpu_count": n, "pcie_bandwidth": mach.pcie_bandwidth,
            "root_link_bandwidth": mach.root_link_bandwidth, "p2p_groups": [list(range(n))],
            "cpu_offload_update": mach.cpu_offload_update, "update_cpu_rate": mach.update_cpu_rate},
            "profiles": {"layer_count": r,
                         "time": {f"{l},{p}": [m.slope, m.intercept] for (l, p), m in prof._time.items()},
                         "x": {str(l): [m.slope, m.intercept] for l, m in prof._x.items()},
                         "y": {str(l): [m.slope, m.intercept] for l, m in prof._y.items()},
                         "w": {str(l): v for l, v in prof._w.items()},
                         "dw": {str(l): v for l, v in prof._dw.items()},
                         "k": {str(l): v for l, v in prof._k.items()}}}
        oc, om, op = oracle_inputs(case)
        items = O.ledger_items(O.task_graph(oc, n), om, op)
        assert rows == O.ledger_rows(items), trial
        assert ms == O.run(items), trial


def test_reference_examples():
    """Hand-traced values of the reference tests."""
    sp = H.synth_profiles(H.SynthSpec(layer_count=6, u_max=8, w_bytes=1 << 20, act_bytes_per_u=1 << 10))
    m2 = H.MachineModel(gpu_count=2, gpu_mem_capacity=1 << 40, pcie_bandwidth=16 << 30)
    packs = ((0, 1), (2, 3), (4, 5))
    g = H.generate_task_graph(H.Configuration(1, packs, 1, packs, 2, H.Mode.PP), m2, sp)
    # test_taskgraph.py:31-46
    assert [t.device[1] for t in g.tasks if t.type is H.TaskType.F] == [0, 1, 0]
    assert [t.device[1] for t in g.tasks if t.type is H.TaskType.B] == [1, 0, 1]
    # test_taskgraph.py:49-57
    u = H.unroll_schedule(g)
    assert (u["gpu0"], u["gpu1"], u["cpu1"], u["cpu0"]) == ([0, 2, 5], [1, 3, 7], [4, 8], [6])


def _table(times, mems, x=0):
    A = H.AffineModel
    r = len(times)
    tm = {(i, p): A(0.0, times[i]) for i in range(r) for p in "FB"}
    mm = {(i, p): A(0.0, mems[i]) for i in range(r) for p in "FB"}
    cx = {i: A(0.0, x) for i in range(r)}
    z = {i: 0 for i in range(r)}
    return H.ProfileSet(r, tm, mm, cx, cx, z, z, z, 8, 8)


def test_packing_reference_examples():
    """Hand-traced packs of test_packing.py:31-86."""
    p = H.balanced_time_pack("B", 1, 4, _table([1, 1, 1, 1], [1, 1, 1, 1]), 2)
    assert p.packs == ((0, 1), (2, 3)) and p.times_ns == (2, 2)
    p = H.balanced_time_pack("B", 1, 5, _table([3, 1, 1, 1, 2], [1] * 5), 3)
    assert p.packs == ((0, 1), (2, 4)) and p.times_ns == (4, 4) and p.mem_bytes == (2, 3)
    p = H.balanced_time_pack("B", 1, 4, _table([1, 1, 1, 1], [3, 3, 3, 3]), 3)
    assert p.packs == ((0, 0), (1, 1), (2, 2), (3, 3))
    with pytest.raises(H.LayerTooLargeError):
        H.balanced_time_pack("B", 1, 3, _table([1, 1, 1], [1, 9, 1]), 3)
    prof = _table([1] * 6, [1] * 6)
    p_b = H.balanced_time_pack("B", 1, 6, prof, 2)
    assert p_b.packs == ((0, 1), (2, 3), (4, 5))
    assert H.balanced_time_pack("F", 1, p_b, prof, 4).packs == ((0, 3), (4, 5))
    prof = _table([1, 1], [2, 2], x=1)
    assert H.balanced_time_pack("B", 1, 2, prof, 4).packs == ((0, 1),)
    assert H.balanced_time_pack("F", 1, 2, prof, 4).packs == ((0, 0), (1, 1))
    assert H.balanced_time_pack("B", 1, 4, _table([0] * 4, [1] * 4), 2).packs == ((0, 1), (2, 3))


def test_errors_are_reference_classes():
    with pytest.raises(H.InvalidConfigurationError):
        H.Configuration(1, ((0, 1),), 1, ((0, 0), (1, 1)), 2, H.Mode.PP).validate()
    with pytest.raises(H.ValidationError):
        H.MachineModel(gpu_count=0, gpu_mem_capacity=1, pcie_bandwidth=1)


# ---- sharded Harmony-DP update (SURVEY 8f row 4 fast mode) -------------------
def _dp_graph(n, D=16, u=2):
    import paper_2202_01306_b200 as H
    from paper_2202_01306_b200.model import GPT_PRESETS, gpt_profiles
    spec = GPT_PRESETS["tiny"]
    prof = gpt_profiles(spec)
    m = H.MachineModel(gpu_count=n, gpu_mem_capacity=4 << 30, pcie_bandwidth=55_000_000_000)
    packs = ((0, 1), (2, 3))
    g = H.generate_task_graph(H.Configuration(u, packs, u, packs, D, H.Mode.DP), m, prof)
    return H, spec, prof, m, g


def _vol(ledger, tensor, stage, gpu=None):
    return sum(r[6] for r in ledger if r[3] == tensor and r[1] == stage and (gpu is None or r[7] == gpu))


def test_sharded_update_is_the_reference_at_one_gpu():
    H, spec, prof, m, g = _dp_graph(1)
    a = H.simulate(g, m, prof)
    b = H.simulate(g, m, prof, dp_update="sharded")
    assert a.ledger == b.ledger and a.makespan_ns == b.makespan_ns


@pytest.mark.parametrize("n", [2, 3, 4, 8])
def test_sharded_update_moves_each_shard_once(n):
    H, spec, prof, m, g = _dp_graph(n, D=2 * n)
    ref = H.simulate(g, m, prof)
    sh = H.simulate(g, m, prof, dp_update="sharded")
    # K in / out and W out: |K| and |W| once per pack over all ranks (N copies in the reference)
    for tensor, stage in (("K", 0), ("K", 2), ("W", 2)):
        assert n * _vol(sh.ledger, tensor, stage) == _vol(ref.ledger, tensor, stage)
    # the forward / backward W swap-ins are unchanged
    assert _vol(sh.ledger, "W", 0) == _vol(ref.ledger, "W", 0)
    # every other row is identical
    keep = lambda led: sorted(r for r in led if not (r[3] in ("K", "W") and (r[3] == "K" or r[1] == 2)))  # noqa: E731
    assert keep(sh.ledger) == keep(ref.ledger)
    # rank g's rows are its 64-parameter-aligned shard of each pack
    P = [sum(spec.layer_params(L) for L in range(lo, hi + 1)) for lo, hi in ((0, 1), (2, 3))]
    c = [-(-p // (64 * n)) * 64 for p in P]
    for gpu in range(n):
        want = sum(max(0, min(ci, p - gpu * ci)) for p, ci in zip(P, c))
        assert _vol(sh.ledger, "W", 2, gpu) == 4 * want
        assert _vol(sh.ledger, "K", 0, gpu) == 8 * want
    assert sh.makespan_ns < ref.makespan_ns


def test_sharded_update_rejects_pp():
    import paper_2202_01306_b200 as H
    from paper_2202_01306_b200.errors import ValidationError
    from paper_2202_01306_b200.model import GPT_PRESETS, gpt_profiles
    prof = gpt_profiles(GPT_PRESETS["tiny"])
    m = H.MachineModel(gpu_count=2, gpu_mem_capacity=4 << 30, pcie_bandwidth=55_000_000_000)
    packs = ((0, 1), (2, 3))
    g = H.generate_task_graph(H.Configuration(4, packs, 4, packs, 16, H.Mode.PP), m, prof)
    with pytest.raises(ValidationError):
        H.simulate(g, m, prof, dp_update="sharded")
    with pytest.raises(ValidationError):
        H.simulate(g, m, prof, dp_update="zero")


@pytest.mark.parametrize("case", golden_cases()[:6], ids=lambda c: c["name"])
def test_python_duration_mirror_matches_native_plan(case):
    """simulator._compute_duration (the reference's private helper, restated)
    prices every compute member exactly as the native plan schedules it."""
    from paper_2202_01306_b200.simulator import _compute_duration
    cfg, mach, prof = product_inputs(case)
    g = H.generate_task_graph(cfg, mach, prof)
    rep = H.simulate(g, mach, prof)
    seen = 0
    for e in rep.trace:
        if e.kind != "compute":
            continue
        t = g.tasks[e.task]
        if t.type is H.TaskType.U and mach.gpu_count > 1 and cfg.mode is H.Mode.DP:
            continue  # the native plan may shard the update across ranks
        member = int(e.label.rsplit("mb", 1)[1])
        u = 1 if t.type is H.TaskType.U else t.group[member]
        assert e.end_ns - e.start_ns == _compute_duration(t, u, prof, mach), e
        seen += 1
    assert seen


def test_python_scheduler_mirror_deadlock_and_order():
    from paper_2202_01306_b200.errors import DeadlockError
    from paper_2202_01306_b200.simulator import _Item, _link, _run
    a = _Item((0,), ("gpu0",), 5, 0, "compute", "a")
    b = _Item((1,), ("gpu0",), 3, 1, "compute", "b")
    c = _Item((2,), ("swap0",), 4, 2, "X", "c")
    for n, it in enumerate((a, b, c)):
        it.idx = n
    _link(a, b)
    _link(a, c, at_start=True)
    _run([a, b, c])
    assert (a.start, a.end, b.start, b.end, c.start, c.end) == (0, 5, 5, 8, 0, 4)
    x = _Item((0,), ("r",), 1, 0, "compute", "x")
    y = _Item((1,), ("r",), 1, 1, "compute", "y")
    x.idx, y.idx = 0, 1
    _link(x, y)
    _link(y, x)
    with pytest.raises(DeadlockError):
        _run([x, y])

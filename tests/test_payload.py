"""bf16 swap payloads (SURVEY 8f4b fast mode), host side: the fp32 <-> (hi, lo)
plane split is exact, hi is the documented rounding, and the plan built with
forward W bytes differs from the reference ledger only in the forward tasks'
W rows."""

import numpy as np

import paper_2202_01306_b200 as H
from paper_2202_01306_b200.model import GPT_PRESETS, gpt_profiles, join_planes, split_planes


def _edge_floats():
    rng = np.random.default_rng(0)
    u = rng.integers(0, 2 ** 32, size=200_000, dtype=np.uint64).astype(np.uint32)
    # low halves at and around the rounding boundary, signs, zeros, denormals, max
    lows = np.array([0, 1, 0x7FFE, 0x7FFF, 0x8000, 0x8001, 0xFFFE, 0xFFFF], dtype=np.uint32)
    highs = np.array([0x0000, 0x0001, 0x3F80, 0x3F81, 0x7F7F, 0x8000, 0x8001, 0xBF80, 0xFF7F], dtype=np.uint32)
    u = np.concatenate([u, (highs[:, None] << 16 | lows[None, :]).reshape(-1)])
    f = u.view(np.float32)
    return f[np.isfinite(f)]


def test_planes_roundtrip_exactly():
    f = _edge_floats()
    hi, lo = split_planes(f)
    assert np.array_equal(join_planes(hi, lo).view(np.uint32), f.view(np.uint32))


def test_hi_plane_is_nearest_with_ties_toward_zero():
    f = _edge_floats()
    f = f[np.abs(f) < 3e38]  # (rounding the largest floats up overflows bf16, as RNE would)
    hi, _ = split_planes(f)
    h = (hi.astype(np.uint32) << 16).view(np.float32).astype(np.float64)
    x = f.astype(np.float64)
    u = f.view(np.uint32).astype(np.uint64)
    down = ((u >> 16) << 16).astype(np.uint32).view(np.float32).astype(np.float64)   # truncation
    up = (((u >> 16) + 1) << 16).astype(np.uint32).view(np.float32).astype(np.float64)
    err_h = np.abs(h - x)
    assert np.all(err_h <= np.minimum(np.abs(down - x), np.abs(up - x)) + 0.0)  # nearest
    tie = (u & 0xFFFF) == 0x8000
    assert np.array_equal(h[tie], down[tie])  # ties go toward zero magnitude


def test_forward_w_rows_are_the_only_ledger_change():
    spec = GPT_PRESETS["tiny"]
    prof = gpt_profiles(spec)
    mach = H.MachineModel(gpu_count=1, gpu_mem_capacity=4 << 30, pcie_bandwidth=55_000_000_000)
    pf, pb = ((0, 0), (1, 1), (2, 3)), ((0, 1), (2, 3))
    for mode in (H.Mode.PP, H.Mode.DP):
        g = H.generate_task_graph(H.Configuration(4, pf, 4, pb, 8, mode), mach, prof)
        w_f = [2 * spec.layer_params(L) + 2 * spec.f32_prefix(L) for L in range(spec.n_layer)]
        ref = H.simulate(g, mach, prof).ledger
        fast = H.simulate(g, mach, prof, w_fwd_bytes=w_f).ledger
        assert len(ref) == len(fast)
        ftasks = {t.index for t in g.tasks if t.type is H.TaskType.F}
        changed = 0
        for a, b in zip(ref, fast):
            da, db = dict(zip(("task", "stage", "member", "tensor"), a[:4])), b
            if a[0] in ftasks and a[3] == "W":
                lo, hi = g.tasks[a[0]].pack
                assert b[6] == sum(w_f[L] for L in range(lo, hi + 1)) < a[6]
                changed += 1
            else:
                assert a == b, (da, db)
        assert changed == len(ftasks)


def test_f32_prefix_is_the_fp32_read_segments():
    spec = GPT_PRESETS["tiny"]
    for L in range(spec.n_layer):
        names = [n for n, _ in spec.layer_segments(L)]
        k = sum(1 for n in names if not n.startswith("w_"))
        assert all(not n.startswith("w_") for n in names[:k]) and all(n.startswith("w_") for n in names[k:])
        assert spec.f32_prefix(L) == sum(c for n, c in spec.layer_segments(L)[:k])

"""Host logic of the profiler loop: per-layer samples from a measured trace
of single-layer packs (recompute subtracted), fitted with the reference's
affine models."""
import paper_2202_01306_b200 as H
from paper_2202_01306_b200.model import GPTSpec, gpt_profiles
from paper_2202_01306_b200.profiling import samples_from_trace
from paper_2202_01306_b200.simulator import TraceEvent


def test_samples_from_synthetic_trace_and_fit():
    spec = GPTSpec(3, 64, 1, 64, 96, True, "micro")
    packs = tuple((L, L) for L in range(3))
    mach = H.MachineModel(gpu_count=1, gpu_mem_capacity=1 << 34, pcie_bandwidth=1 << 34)
    samples = []
    for u in (1, 2, 4):
        g = H.generate_task_graph(H.Configuration(u, packs, u, packs, u, H.Mode.DP), mach, gpt_profiles(spec))
        trace = []
        for t in g.tasks:
            L = t.pack[0]
            f = 1000 * (L + 1) * u + 50
            b = 2000 * (L + 1) * u + 70
            d = {"F": f, "B": b + (f if t.recompute else 0), "U": 500 + L}[t.type.value]
            trace.append(TraceEvent("gpu0.compute", t.index, "compute", "x", 10, 10 + d))
        samples += samples_from_trace(spec, g, trace, u)
    prof = H.fit_profiles(samples)
    for L in range(3):
        for u in (1, 2, 3, 4):
            assert prof.time_ns("F", L, u) == 1000 * (L + 1) * u + 50
            assert prof.time_ns("B", L, u) == 2000 * (L + 1) * u + 70
        assert prof.time_ns("U", L, 1) == 500 + L
        assert prof.w_bytes(L) == 4 * spec.layer_params(L)
        assert prof.x_bytes(L, 2) == gpt_profiles(spec).x_bytes(L, 2)


def test_slow_start_with_a_monotone_oracle_matches_scan():
    """The probe the runtime oracle plugs into (reference `profiler.py:196-223`)."""
    from paper_2202_01306_b200.profiler import slow_start_max_u
    for limit in (1, 2, 3, 7, 8, 9, 31, 64, 100):
        calls = []

        def fits(u, limit=limit):
            calls.append(u)
            return u <= limit
        assert slow_start_max_u(fits, 64) == min(limit, 64)


def test_runtime_oom_probe_gpu():
    """The OOM oracle is the runtime itself: every u the slow-start search
    accepts loads under alpha, u + 1 does not, and the answer equals a brute
    scan; the measured pool bytes grow with u (the measured memory model)."""
    import pytest
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    from paper_2202_01306_b200.model import GPT_PRESETS
    from paper_2202_01306_b200.profiling import probe_max_microbatch, runtime_mem_oracle
    spec = GPT_PRESETS["tiny"]
    packs = ((0, 1), (2, 3))
    big = runtime_mem_oracle(spec, packs, 64 << 30)
    assert big(4) and big(16) and big(17)
    by = big.device_bytes
    big.close()
    assert by[17] > by[16] > by[4]
    alpha = (by[4] + by[16]) // 2  # the answer lies strictly between 4 and 16
    u, seen = probe_max_microbatch(spec, packs, alpha, u_cap=64)
    assert 4 <= u < 16
    scan = runtime_mem_oracle(spec, packs, alpha)
    assert [scan(v) for v in range(1, 20)] == [v <= u for v in range(1, 20)]
    scan.close()
    assert all(b <= alpha for b in seen.values())


test_runtime_oom_probe_gpu = __import__("pytest").mark.gpu(test_runtime_oom_probe_gpu)

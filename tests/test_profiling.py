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

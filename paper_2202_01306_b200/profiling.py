"""The profiler loop (paper §4.2, SURVEY §8f "next #1"): measure per-layer
F / B / U costs of the real B200 kernels, fit the reference's affine cost
models and hand them to the planner.

Samples come from the runtime's own measured trace: a task graph of
single-layer packs is executed with ``D = u`` samples (one microbatch member
per task), so each compute item's CUDA-event duration is one layer's cost:

* F task member           -> time_F(L, u)
* B task with recompute   -> time_B(L, u) + time_F(L, u)   (time_F subtracted)
* B task of the last pack -> time_B(L, u)                  (no recompute)
* U task                  -> time_U(L)                     (fused Adam)

Memory, activation and state sizes are the runtime's real byte layout
(`model.py`), so ``fit_profiles`` sees integer-exact W / dW / K / x / y
(`profiler.py:234-314` of the reference requires them to be u-independent).
"""

from __future__ import annotations

from .cnn import CNNSpec, cnn_profiles, synthetic_images
from .core import Configuration, MachineModel, Mode
from .model import GPTSpec, gpt_profiles, synthetic_batch
from .profiler import ProfileSample, ProfileSet, fit_profiles, sample_points
from .taskgraph import TaskType, generate_task_graph


def shape_profiles(spec: GPTSpec | CNNSpec, u_max: int = 64) -> ProfileSet:
    """Byte-exact ProfileSet of either model family (times FLOP-derived)."""
    return cnn_profiles(spec, u_max=u_max) if isinstance(spec, CNNSpec) else gpt_profiles(spec, u_max=u_max)


def synthetic_inputs(spec: GPTSpec | CNNSpec, samples: int):
    """Synthetic minibatch of either family (tokens / images, labels)."""
    return synthetic_images(spec, samples) if isinstance(spec, CNNSpec) else synthetic_batch(spec, samples)


def samples_from_trace(spec: GPTSpec | CNNSpec, graph, trace, u: int) -> list[ProfileSample]:
    """ProfileSamples of one profiling run (trace = measured compute
    TraceEvents of the report).  Packs of several layers are apportioned to
    their layers by FLOPs (F, B) and parameters (U): the layers then carry the
    kernel efficiency they have inside real packs, where consecutive kernels
    overlap their launches, instead of the isolated single-layer cost."""
    shapes = shape_profiles(spec)
    dur: dict[int, list[int]] = {}
    for e in trace:
        if e.kind == "compute":
            dur.setdefault(e.task, []).append(e.end_ns - e.start_ns)
    f_time, b_time, u_time = {}, {}, {}
    for t in graph.tasks:
        lo, hi = t.pack
        d = sum(dur.get(t.index, [0]))
        layers = range(lo, hi + 1)
        wts = [spec.layer_params(L) if t.type is TaskType.U else max(1, spec.layer_fwd_flops(L, 1)) for L in layers]
        tot = float(sum(wts))
        for L, w in zip(layers, wts):
            share = int(round(d * w / tot))
            if t.type is TaskType.F:
                f_time[L] = share
            elif t.type is TaskType.B:
                b_time[L] = (share, t.recompute)
            else:
                u_time[L] = share
    out = []
    for L in range(spec.n_layer):
        b, rec = b_time[L]
        tb = max(0, b - f_time[L]) if rec else b
        common = dict(layer_id=L, microbatch=u, x_bytes=shapes.x_bytes(L, u), y_bytes=shapes.y_bytes(L, u),
                      w_bytes=shapes.w_bytes(L), dw_bytes=shapes.dw_bytes(L), k_bytes=shapes.k_bytes(L))
        out.append(ProfileSample(pass_="F", compute_time_ns=f_time[L], mem_bytes=shapes.mem_bytes("F", L, u),
                                 **common))
        out.append(ProfileSample(pass_="B", compute_time_ns=tb, mem_bytes=shapes.mem_bytes("B", L, u), **common))
        out.append(ProfileSample(pass_="U", compute_time_ns=u_time[L], mem_bytes=shapes.mem_bytes("U", L, 1),
                                 **common))
    return out


def profile_gpt(spec: GPTSpec | CNNSpec, u_values=None, u_max: int = 8, stride: int = 4, alpha_bytes: int = 64 << 30,
                device: int = 0, warmup: int = 1, pack_layers: int = 1) -> tuple[ProfileSet, list[ProfileSample]]:
    """Measure and fit a ProfileSet on this GPU (sample points 1, stride
    multiples and u_max, as the reference's profiler, `profiler.py:421-427`)."""
    from .runtime import HarmonyRuntime
    us = tuple(u_values) if u_values else sample_points(u_max, stride)
    R = spec.n_layer
    packs = tuple((L, min(L + pack_layers, R) - 1) for L in range(0, R, pack_layers))
    samples: list[ProfileSample] = []
    rt = HarmonyRuntime(spec, alpha_bytes=alpha_bytes, device=device)
    try:
        rt.init_weights(0)
        mach = MachineModel(gpu_count=1, gpu_mem_capacity=alpha_bytes, pcie_bandwidth=55_000_000_000)
        prof0 = shape_profiles(spec, u_max=max(us))
        for u in us:
            g = generate_task_graph(Configuration(u, packs, u, packs, u, Mode.DP), mach, prof0)
            rt.load(g, mach, prof0)
            tok, lab = synthetic_inputs(spec, u)
            for _ in range(warmup + 1):
                rt.step(tok, lab)
            samples += samples_from_trace(spec, g, rt.report().trace, u)
    finally:
        rt.close()
    return fit_profiles(samples, stride=stride), samples


profile_model = profile_gpt  # either family (GPTSpec or CNNSpec)


def runtime_mem_oracle(spec: GPTSpec | CNNSpec, packs, alpha_bytes: int, *, minibatch_per_u: int = 1,
                       device: int = 0, mode: Mode = Mode.DP):
    """The paper's OOM probe (`PAPER.md:385-394`) on the real runtime: a
    callable u -> bool that loads the plan of ``packs`` at microbatch u
    (minibatch = u * ``minibatch_per_u``) into a runtime capped at
    ``alpha_bytes`` and reports whether it fits.  The runtime sizes every
    device buffer of the plan (W / dW / K slots, activation stores, scratch,
    receive buffers) and cudaMallocs them as ONE pool: a plan that does not fit
    raises CapacityViolationError (or the allocation fails) -- exactly the
    failure the reference's ``slow_start_max_u`` expects from its oracle
    (`profiler.py:196-223`).  The returned callable records the pool bytes of
    every fitting u in ``.device_bytes`` (the measured memory model) and is
    closed with ``.close()``."""
    from .errors import CapacityViolationError, DeviceError
    from .runtime import HarmonyRuntime
    rt = HarmonyRuntime(spec, alpha_bytes=alpha_bytes, device=device)
    mach = MachineModel(gpu_count=1, gpu_mem_capacity=alpha_bytes, pcie_bandwidth=55_000_000_000)

    def fits(u: int) -> bool:
        D = u * minibatch_per_u
        prof = shape_profiles(spec, u_max=max(64, u))
        g = generate_task_graph(Configuration(u, packs, u, packs, D, mode), mach, prof)
        try:
            rt.load(g, mach, prof)
        except (CapacityViolationError, DeviceError):
            return False
        fits.device_bytes[u] = rt.counters()["device_bytes"]
        return True

    fits.device_bytes = {}
    fits.close = rt.close
    return fits


def probe_max_microbatch(spec: GPTSpec | CNNSpec, packs, alpha_bytes: int, u_cap: int = 256, **kw) -> tuple[int, dict]:
    """Largest microbatch the runtime can execute ``packs`` with under
    ``alpha_bytes``: the reference's slow-start search driven by the runtime's
    own admission (``runtime_mem_oracle``).  Returns (u, {u: device bytes})."""
    from .profiler import slow_start_max_u
    oracle = runtime_mem_oracle(spec, packs, alpha_bytes, **kw)
    try:
        return slow_start_max_u(oracle, u_cap), dict(oracle.device_bytes)
    finally:
        oracle.close()

#!/usr/bin/env python
"""bench.py -- Harmony layer-pack training throughput on B200.

Workload (BASELINE.json configs[2], the config the metric is quoted on at
1/2/4/8 GPUs): GPT-2 XL (48 blocks, d=1600, 25 heads, seq 1024, V=50257,
1.64 B params incl. untied head; W+dW+K = 26 GB) trained with Harmony-DP
under a capped per-GPU memory budget alpha (default 32 GiB) so every pack's
weights and Adam state are swapped through PCIe each iteration.  Weak
scaling: 16 samples per GPU per iteration.  Synthetic data (tokens uniform
in [0, V), seed 1234; weights N(0, 0.02), seed 0).

One "step" = one full training iteration (all F/B/U tasks of the Harmony
schedule: swap-in of every pack's W and K, F/B compute with recompute,
fused Adam, swap-out of W and K).  Timing: the runtime's own CUDA events on
its compute stream (all streams joined), max over ranks, after W warm-up
steps.  Inputs are larger than L2 (model state streams from host memory every
step).  ``value`` runs on device-resident tokens; ``e2e`` feeds tokens from
pinned host memory and reads the loss back each step.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl native|reference]
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

WORKLOADS = {
    # name: (preset, samples_per_gpu, u, layers_per_pack, alpha_gib, mode)
    "gpt2-xl-dp": ("gpt2-xl", 16, 4, 8, 32, "dp"),
    # SURVEY 8f4b fast mode (NOT the reference's ledger): the headline workload with W
    # swapped as exact [bf16 hi | lo] planes; forward tasks move hi + the fp32 prefix
    "gpt2-xl-dp-bf16w": ("gpt2-xl", 16, 4, 8, 32, "dp", "bf16"),
    "tiny": ("tiny", 16, 4, 2, 4, "pp"),
    "tiny-dp": ("tiny", 16, 4, 2, 4, "dp"),
    "tiny-dp-shard": ("tiny", 16, 4, 2, 4, "dp", "fp32", "sharded"),
    # the same model at a 4x larger minibatch: Harmony's grouping amortises the fixed
    # per-iteration swap bytes (W, K) over more samples ("no grouping")
    "gpt2-xl-dp-d64": ("gpt2-xl", 64, 8, 4, 64, "dp"),
    # config c2: BERT-Large (24 x d1024, seq 512, full attention), D = 64, every pack swapped
    "bert-large-pp": ("bert-large", 64, 16, 6, 32, "pp"),
    # north-star target shape: W + Adam state (184 GB) > one GPU's HBM
    "gpt-15b-dp": ("gpt-15b", 24, 4, 3, 170, "dp"),
    "gpt-15b-dp-bf16w": ("gpt-15b", 24, 4, 3, 170, "dp", "bf16"),  # 8f4b fast mode (not the reference ledger)
    # SURVEY 8f row-4 fast mode (NOT the reference ledger at N > 1): one shared host arena,
    # gradients reduce-scattered, rank g updates / swaps shard g of each pack's K and W --
    # per GPU 2|W| + 5|W|/N of PCIe instead of 7|W|, one host copy instead of N (so the
    # >HBM model runs Harmony-DP past N = 1); identical to the replicated run at N = 1
    "gpt2-xl-dp-shard": ("gpt2-xl", 16, 4, 8, 32, "dp", "fp32", "sharded"),
    "gpt-15b-dp-shard": ("gpt-15b", 24, 4, 3, 170, "dp", "fp32", "sharded"),
    # config c4: GPT-style 40B (48 x d8192, 64 heads of 128; W + Adam = 474 GB of pinned host
    # state, one shared copy) as Harmony-PP: D = 8 per GPU (64 on 8 B200), packs of 2 layers;
    # skipped with a clear reason when the host cannot pin its state (the precheck)
    "gpt-40b-pp": ("gpt-40b", 8, 4, 2, 160, "pp"),
    # config c5: deep-CNN packs (128 residual blocks at 56x56 / 28x28, implicit-GEMM convs)
    "resnet-dp": ("resnet-bench", 64, 32, 16, 12, "dp"),
    # config c5 at its named depth: ResNet-1026 (517 chain layers: 511
    # residual blocks, 0.80 B parameters) and VGG-416 at 224x224 (stem to 56x56), 1000
    # classes, packs of 32 layers -- the deep-chain swap stress
    "resnet-1026-dp": ("resnet-1026", 32, 16, 32, 40, "dp"),
    "vgg-416-dp": ("vgg-416", 32, 16, 32, 40, "dp"),
}


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return {"bf16": d.get("bf16_tflops_sustained", d["bf16_tflops"]), "bf16_burst": d["bf16_tflops"],
                "hbm": d["hbm_gbs"], "kind": "measured"}
    return {"bf16": 1400.0, "bf16_burst": 1590.0, "hbm": 6650.0, "kind": "fallback"}


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.proc = None
        self.lines: list[str] = []

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self._t = threading.Thread(target=self._read, daemon=True)
            self._t.start()
        except (OSError, FileNotFoundError):
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def __exit__(self, *exc):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self) -> dict:
        sm, mx, reasons = [], 0, set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in self.lines:
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 6:
                continue
            try:
                sm.append(float(parts[0]))
                mx = max(mx, float(parts[1]))
            except ValueError:
                continue
            for n, v in zip(names, parts[2:6]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx or None,
                "reasons": sorted(reasons), "samples": len(sm)}


def _dist():
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if SHARE_GPU:  # test mode: every rank on cuda:0
        local = 0
    return world, rank, local


# HM_BENCH_SHARE_GPU=1 (test mode, never a bench number): N ranks share ONE GPU,
# the control plane runs on gloo and the per-pack gradient sum on the runtime's
# CUDA-IPC backend (NCCL cannot place two ranks on one device).  It exercises
# the multi-rank bench path -- launch, barriers, max over ranks, the ledger
# union, shared arenas, device-counter ordering -- on a one-GPU box.
SHARE_GPU = os.environ.get("HM_BENCH_SHARE_GPU") == "1"


def _coll_device() -> str:
    return "cpu" if SHARE_GPU else "cuda"


def _max_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device=_coll_device())
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def _barrier(world: int) -> None:
    if world > 1:
        import torch.distributed as dist
        dist.barrier()


def _pcie_rates(world: int, rank: int) -> tuple[dict, dict]:
    """(isolated, concurrent) link rates of this rank's GPU.  Isolated: the
    ranks probe one after another (the per-GPU PCIe bound).  Concurrent: all
    ranks probe at once; the sum over ranks is the host root complex's
    aggregate rate (the host-root bound)."""
    iso = {}
    for r in range(world):
        _barrier(world)
        if r == rank:
            iso = _pcie_gbs()
    _barrier(world)
    conc = _pcie_gbs(reps=1) if world > 1 else dict(iso)
    _barrier(world)
    return iso, conc


def _sum_over_ranks(x: float, world: int) -> float:
    if world == 1:
        return x
    import torch
    import torch.distributed as dist
    t = torch.tensor([x], dtype=torch.float64, device=_coll_device())
    dist.all_reduce(t)
    return float(t.item())


def _nccl_busbw(world: int, nbytes: int = 256 << 20) -> float:
    """Measured all-reduce bus bandwidth (GB/s): 2(N-1)/N x bytes / time."""
    if world == 1 or SHARE_GPU:
        return 0.0
    import torch
    import torch.distributed as dist
    x = torch.ones(nbytes // 4, dtype=torch.float32, device="cuda")
    for _ in range(3):
        dist.all_reduce(x)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        dist.all_reduce(x)
    e1.record()
    torch.cuda.synchronize()
    t = _max_over_ranks(e0.elapsed_time(e1) / 1e3 / 10, world)
    return 2 * (world - 1) / world * nbytes / t / 1e9


def _dp_update(workload: str) -> str:
    w = WORKLOADS[workload]
    return w[7] if len(w) > 7 else "replicated"


def _host_precheck(spec, world: int, mode: str, stash_bytes: int, dp_update: str = "replicated") -> str | None:
    """Pinned host memory the job needs (per-rank W + K replicas under
    Harmony-DP, one shared copy under PP and the sharded DP update) vs what
    the host has available."""
    replicas = world if mode == "dp" and dp_update == "replicated" else 1
    need = spec.total_params() * 12 * replicas + stash_bytes * (world if mode == "dp" else 1)
    avail = 0
    try:
        for ln in open("/proc/meminfo"):
            if ln.startswith("MemAvailable:"):
                avail = int(ln.split()[1]) * 1024
    except OSError:
        return None
    if avail and need > 0.92 * avail:
        return (f"needs {need / 2**30:.1f} GiB of pinned host memory (W + Adam state{' per DP rank' if mode == 'dp' else ''}"
                f" + stash), the host has {avail / 2**30:.1f} GiB available")
    return None


def phase_bound_s(graph, ledger, pcie: dict, rank: int = 0) -> float:
    """Phase-serialised link bound (seconds) of one iteration on `rank`: the
    forward packs' transfers (W in, stash out) and the backward + update packs'
    (W / stash / K in, W / K out) run in two windows -- the next iteration's
    forward waits on this one's updates -- so each window is bounded by its own
    direction mix: max(H2D / h2d, D2H / d2h, (H2D + D2H) / bidir), summed."""
    from paper_2202_01306_b200 import TaskType
    total = 0.0
    for is_f in (True, False):
        ph_in = ph_out = 0
        for r in ledger:
            if r[4] in ("cpu_gpu_swap", "message_passing") and r[7] == rank and \
                    (graph.tasks[r[0]].type is TaskType.F) == is_f:
                if r[1] == 0:
                    ph_in += r[6]
                elif r[1] == 2:
                    ph_out += r[6]
        total += max(ph_in / (pcie["h2d"] * 1e9), ph_out / (pcie["d2h"] * 1e9),
                     (ph_in + ph_out) / (pcie["bidir"] * 1e9))
    return total


def _pcie_gbs(reps: int = 3):
    """Measured pinned GB/s of this GPU's link (1 GiB copies): H2D alone, D2H
    alone, and both directions at once on two streams ("bidir", the sum;
    46 + 46 = 92 GB/s on the B200 boxes vs 55.6 alone -- the swap engine runs
    both directions concurrently for most of an iteration).  The best of
    ``reps`` probes: a roofline denominator is the link's attainable rate, and
    one probe has been seen reading half of it (a transient on the host)."""
    best = {}
    for _ in range(reps):
        for k, v in _pcie_probe().items():
            best[k] = max(best.get(k, 0.0), v)
    return best


def _pcie_probe():
    import torch
    n = 1 << 30
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
    out = {}
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    s1.wait_event(e0)
    s2.wait_event(e0)
    eh, ed = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s1):
        for _ in range(4):
            d.copy_(h, non_blocking=True)
        eh.record(s1)
    with torch.cuda.stream(s2):
        for _ in range(4):
            h2.copy_(d2, non_blocking=True)
        ed.record(s2)
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)
    e1.record()
    torch.cuda.synchronize()
    # each direction's rate over its own span (both start together): the sum is
    # the two-direction capacity even when one direction finishes first (the
    # total over the longer span would count the other's idle tail against it)
    out["bidir"] = 4 * n / (e0.elapsed_time(eh) / 1e3) / 1e9 + 4 * n / (e0.elapsed_time(ed) / 1e3) / 1e9
    del h2, d2
    for name, fn in (("h2d", lambda: d.copy_(h, non_blocking=True)), ("d2h", lambda: h.copy_(d, non_blocking=True))):
        fn()
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        for _ in range(3):
            fn()
        e.record()
        torch.cuda.synchronize()
        out[name] = 3 * n / (s.elapsed_time(e) / 1e3) / 1e9
    del h, d
    return out


def _gemm_groups(launches, top=8):
    """GEMM launches of the profiled iteration grouped by FLOPs per launch
    (one group per (M, N, K) product): where the GEMM time goes."""
    groups = {}
    for cls, fl, _by, ms, _span in launches:
        if int(cls) != 0:
            continue
        g = groups.setdefault(round(fl / 1e9, 3), [0, 0.0])
        g[0] += 1
        g[1] += ms
    rows = [{"gflop": k, "launches": n, "ms_total": round(t, 3), "us_avg": round(1e3 * t / n, 2),
             "tflops": round(k * n / t, 1) if t else 0.0} for k, (n, t) in groups.items()]
    rows.sort(key=lambda r: -r["ms_total"])
    return rows[:top]


def _ncu_traffic() -> dict:
    """DRAM traffic of the dominant kernel from the newest committed `ncu --set
    full` capture of in-step GEMM launches (profiles/r0N_gemm_ncu_summary.json,
    made by tools/ncu_summary.py)."""
    cands = [os.path.join(ROOT, "profiles", f"r0{n}_gemm_ncu_summary.json") for n in (2, 1)]
    p = next((c for c in cands if os.path.exists(c)), None)
    if p is None:
        return {}
    d = json.load(open(p))
    return {"traffic": d["dram_bytes_per_launch_mean"],
            "traffic_how": f"dram__bytes_read.sum + dram__bytes_write.sum per launch, mean of {d['launches']} "
                           f"in-step GEMM launches of one ncu --set full capture ({d['source']})"}


def step_flops(graph, spec) -> int:
    """Algorithmic FLOPs of one iteration: F member
    u*s*(24d^2+4sd) per block + 2*u*s*d*V for the head; B = 2F (+F recompute)."""
    total = 0
    for t in graph.tasks:
        if t.type.value == "U":
            continue
        f = sum(spec.layer_fwd_flops(L, u) for L in range(t.pack[0], t.pack[1] + 1) for u in t.group)
        total += f if t.type.value == "F" else (2 * f + (f if t.recompute else 0))
    return total


def cnn_port_sample(spec, threads: int, seconds_cap: float = 30.0) -> dict:
    """Time the torch-CPU fp32 port (oracle/cnn_cpu.py) on one sample through
    the whole chain (fwd + bwd + Adam): the per-sample cost of the workload."""
    import numpy as np
    import torch
    from oracle.cnn_cpu import CNNOracle
    from paper_2202_01306_b200.cnn import synthetic_images
    torch.set_num_threads(threads)
    n = spec.total_params()
    g = torch.Generator().manual_seed(0)
    w = (torch.randn(n, generator=g) * 0.02).numpy()
    off = np.cumsum([0] + [spec.layer_params(L) for L in range(spec.n_layer)])
    o = CNNOracle(spec, w, off)
    img, lab = synthetic_images(spec, 1)
    o.step(img, lab, [1])  # warm
    t0 = time.perf_counter()
    reps = 0
    while True:
        o.step(img, lab, [1])
        reps += 1
        if time.perf_counter() - t0 > min(seconds_cap, 10.0) or reps >= 5:
            break
    dt = (time.perf_counter() - t0) / reps
    return {"value": 1.0 / dt, "unit": "samples/s", "cores": threads, "kind": "port",
            "sample": f"torch-CPU fp32 port (oracle/cnn_cpu.py), 1 sample through the full {spec.name} chain "
                      f"(fwd + bwd + Adam), {reps} reps of {dt:.2f} s"}


def cpu_port_iteration(spec, samples: int, threads: int, groups=None) -> dict:
    """One REAL training iteration of the torch-CPU fp32 port (oracle/gpt_cpu.py)
    on the full-depth model: ``samples`` sequences forward + backward through
    every layer, then Adam over every parameter -- the same work the Harmony
    schedule does in one iteration at D = ``samples`` (its F/B/U tasks
    compute exactly full-batch backprop followed by a per-pack Adam).  Nothing
    is extrapolated: the returned rate is samples / measured seconds."""
    import numpy as np
    import torch
    from oracle.gpt_cpu import GPTOracle
    from paper_2202_01306_b200.model import synthetic_batch
    torch.set_num_threads(threads)
    n = spec.total_params()
    g = torch.Generator().manual_seed(0)
    w = torch.empty(n, dtype=torch.float32).normal_(0.0, 0.02, generator=g).numpy()
    off = np.cumsum([0] + [spec.layer_params(L) for L in range(spec.n_layer)])
    o = GPTOracle(spec, w, off)
    del w
    tok, lab = synthetic_batch(spec, samples)
    groups = groups or [1] * samples
    t0 = time.perf_counter()
    loss = o.step(tok, lab, groups)
    dt = time.perf_counter() - t0
    del o
    return {"value": samples / dt, "unit": "samples/s", "cores": threads, "kind": "port", "seconds": dt,
            "loss": loss,
            "sample": f"one measured iteration of the torch-CPU fp32 port (oracle/gpt_cpu.py) of the full "
                      f"{spec.n_layer}-layer {spec.name}: {samples} sample(s) x {spec.seq_len} tokens forward + "
                      f"backward (member loop {groups}) + Adam over all {n / 1e9:.2f} B parameters, "
                      f"{dt:.1f} s on {threads} threads"}


def planner_port_seconds(graph, machine, prof) -> dict:
    """Single-core wall time of the reference's planner path restated in pure
    Python (oracle/schedule.py: generate_task_graph -> _build_items -> _run,
    taskgraph.py:211-400, simulator.py:150-375) for the workload's config."""
    from oracle import schedule as S
    cfg = graph.config
    ocfg = {"u_f": cfg.u_f, "p_f": [list(p) for p in cfg.p_f], "u_b": cfg.u_b, "p_b": [list(p) for p in cfg.p_b],
            "minibatch": cfg.minibatch, "mode": cfg.mode.value}
    tab = prof.tables(prof.layer_count, max(cfg.minibatch, 1))
    oprof = {k: tab[k] for k in ("x", "y", "w", "dw", "k", "tF", "tB", "tU")}
    groups = {}
    for i, grp in enumerate(machine.p2p_groups):
        for x in grp:
            groups[x] = i
    omach = {"gpu_count": machine.gpu_count, "pcie": machine.pcie_bandwidth,
             "root": machine.root_link_bandwidth, "p2p_group_of": [groups[i] for i in range(machine.gpu_count)],
             "cpu_offload_update": machine.cpu_offload_update, "update_cpu_rate": machine.update_cpu_rate}
    t0 = time.perf_counter()
    tasks = S.task_graph(ocfg, machine.gpu_count)
    items = S.ledger_items(tasks, omach, oprof)
    makespan = S.run(items)
    dt = time.perf_counter() - t0
    return {"seconds": round(dt, 4), "tasks": len(tasks), "items": len(items), "makespan_ns": makespan,
            "cores": 1, "what": "task graph + swap plan + event-driven estimate (pure-Python restatement of the "
                                "reference planner, oracle/schedule.py), single core"}


def run_reference(args) -> None:
    """Reference arm: the reference has no training runtime, so
    the path's CPU implementation is the torch-CPU fp32 port of one Harmony
    iteration.  It runs ONE full-depth iteration at D = 4 (BASELINE.md's
    recipe for c3) on all host threads -- minutes of CPU work, so the
    driver's --steps / --warmup are not repeated: the line reports the steps
    that actually ran (1, no warm-up)."""
    world, rank, _ = _dist()
    if rank != 0:
        return
    import torch
    from paper_2202_01306_b200 import MachineModel  # noqa: F401
    import paper_2202_01306_b200 as H
    from paper_2202_01306_b200.model import GPT_PRESETS, gpt_machine, gpt_profiles
    preset, per_gpu, u, lpp, alpha_gib, mode, *_ = WORKLOADS[args.workload]
    spec = GPT_PRESETS[preset]
    threads = len(os.sched_getaffinity(0))
    D = per_gpu * args.gpus
    R = spec.n_layer
    packs = tuple((i, min(i + lpp, R) - 1) for i in range(0, R, lpp))
    machine = gpt_machine(args.gpus, alpha_bytes=alpha_gib << 30)
    prof = gpt_profiles(spec)
    graph = H.generate_task_graph(H.Configuration(u, packs, u, packs, D, H.Mode(mode)), machine, prof)
    plan = planner_port_seconds(graph, machine, prof)
    sample_d = min(4, D)
    it = cpu_port_iteration(spec, sample_d, threads)
    v = it["value"]
    line = {"impl": "reference", "metric": "samples/s (Harmony layer-pack training, GPT-2 XL)"
            if preset == "gpt2-xl" else f"samples/s (Harmony layer-pack training, {spec.name})", "value": v,
            "unit": "samples/s", "n_gpus": args.gpus, "steps": 1, "warmup": 0,
            "ms_per_step": 1000.0 * it["seconds"], "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": _config(args.workload, spec, mode, lpp, u, alpha_gib, D, args.gpus,
                              (WORKLOADS[args.workload][6:] or ("fp32",))[0]),
            "sample": f"iteration at D={sample_d} (of the workload's D={D}): the per-sample work is the same, "
                      f"the per-iteration Adam is amortised over {sample_d} instead of {D} samples",
            "requested": {"steps": args.steps, "warmup": args.warmup},
            "cpu_baseline": {k: it[k] for k in ("value", "unit", "cores", "kind", "sample")},
            "planner_port": plan, "torch_threads": torch.get_num_threads(),
            "e2e": {"value": v, "unit": "samples/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def _config(workload, spec, mode, lpp, u, alpha_gib, D, world, payload) -> dict:
    return {"workload": f"{workload}: {spec.name} Harmony-{mode.upper()}, packs of {lpp} layers, "
                        f"u_f=u_b={u}, alpha={alpha_gib} GiB/GPU",
            "global_batch": D, "seq_len": getattr(spec, "seq_len", None), "parallelism": f"harmony-{mode}{world}",
            "l2": "inputs larger than L2 (W and K stream from host every step)",
            "w_payload": payload if payload == "fp32" else
            "bf16 planes (SURVEY 8f4b fast mode: forward W rows differ from the reference ledger)",
            "dp_update": _dp_update(workload) if _dp_update(workload) == "replicated" else
            "sharded (SURVEY 8f row-4 fast mode: U rows carry one shard each at N > 1)"}


def run_native(args) -> None:
    import numpy as np
    import torch

    world, rank, local = _dist()
    torch.cuda.set_device(local)
    if world > 1:
        import torch.distributed as dist
        if SHARE_GPU:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_2202_01306_b200 as H
    from paper_2202_01306_b200 import ops
    from paper_2202_01306_b200.cnn import CNN_PRESETS, cnn_profiles, synthetic_images
    from paper_2202_01306_b200.model import GPT_PRESETS, gpt_machine, gpt_profiles, synthetic_batch
    from paper_2202_01306_b200.runtime import HarmonyRuntime

    preset, per_gpu, u, lpp, alpha_gib, mode, *_ = WORKLOADS[args.workload]
    if args.alpha_gib:
        alpha_gib = args.alpha_gib
    is_cnn = preset in CNN_PRESETS
    spec = CNN_PRESETS[preset] if is_cnn else GPT_PRESETS[preset]
    D = per_gpu * world
    R = spec.n_layer
    packs = tuple((i, min(i + lpp, R) - 1) for i in range(0, R, lpp))
    cfg = H.Configuration(u, packs, u, packs, D, H.Mode(mode))
    pcie, pcie_conc = _pcie_rates(world, rank)
    machine = gpt_machine(world, alpha_bytes=alpha_gib << 30, pcie_gbs=min(pcie["h2d"], pcie["d2h"]) * 1e9)
    prof = cnn_profiles(spec) if is_cnn else gpt_profiles(spec)
    graph = H.generate_task_graph(cfg, machine, prof)
    dp_update = _dp_update(args.workload)
    skip = _host_precheck(spec, world, mode, HarmonyRuntime.stash_bytes_for(graph, prof), dp_update)
    if skip:
        if rank == 0:
            print(json.dumps({"metric": f"samples/s (Harmony layer-pack training, {spec.name})", "value": None,
                              "unit": "samples/s", "n_gpus": world, "skipped": skip,
                              "config": {"workload": args.workload}}), flush=True)
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()
        return
    payload = (WORKLOADS[args.workload][6:] or ("fp32",))[0]
    rt = HarmonyRuntime(spec, alpha_bytes=alpha_gib << 30, device=local, w_payload=payload, dp_update=dp_update)
    sim = H.simulate(graph, machine, prof, w_fwd_bytes=rt.w_fwd_bytes(), dp_update=dp_update)
    # weights drawn on the GPU (seconds, also with 8 ranks initialising at once);
    # the CPU generator is what the parity tests use
    pp_multi = mode == "pp" and world > 1
    shard_multi = mode == "dp" and dp_update == "sharded" and world > 1
    if pp_multi or shard_multi:
        # Harmony-PP / sharded DP: one pinned host copy of W / K (/ stash) shared
        # by every rank (rank 0 creates and initialises it)
        import torch.distributed as dist
        name = [f"hm_bench_{os.getpid()}" if rank == 0 else None]
        dist.broadcast_object_list(name, src=0)
        stash = HarmonyRuntime.stash_bytes_for(graph, prof)
        if rank == 0:
            rt.share_arenas(name[0], True, stash)
            rt.init_weights(0, device=None if is_cnn else "cuda")
        dist.barrier()
        if rank != 0:
            rt.share_arenas(name[0], False, stash)
    else:
        rt.init_weights(0, device=None if is_cnn else "cuda")
    if world > 1 and mode == "dp":
        import torch.distributed as dist
        if SHARE_GPU:
            rt.init_ipc_reduce(world, rank)
        else:
            obj = [HarmonyRuntime.nccl_unique_id() if rank == 0 else None]
            dist.broadcast_object_list(obj, src=0)
            rt.init_comm(obj[0], world, rank)
    rt.load(graph, machine, prof, rank=rank)
    if pp_multi or shard_multi or (SHARE_GPU and world > 1):  # device counters (PP: activation buffers) of every peer
        blobs = [None] * world
        dist.all_gather_object(blobs, rt.ipc_export())
        for b in blobs:
            rt.ipc_import(b)
        dist.barrier()
    lo, hi = rt.sample_range()
    if is_cnn:
        img_all, labc_all = synthetic_images(spec, D)
        tok_c, lab_c = img_all[lo:hi].contiguous(), labc_all[lo:hi].contiguous()
    else:
        tok_all, lab_all = synthetic_batch(spec, D)
        tok_c, lab_c = torch.from_numpy(tok_all[lo:hi]), torch.from_numpy(lab_all[lo:hi])
    in_bytes = tok_c.numel() * tok_c.element_size() + lab_c.numel() * lab_c.element_size()
    tok_d = tok_c.cuda()
    lab_d = lab_c.cuda()
    tok_p = tok_c.pin_memory()
    lab_p = lab_c.pin_memory()

    for _ in range(args.warmup):
        rt.step(tok_d, lab_d)
    _barrier(world)
    torch.cuda.synchronize()
    launches0 = ops.launch_count()
    with ClockSampler(local) as clocks:
        losses, t_dev = rt.run_steps(args.steps, tok_d, lab_d)
    torch.cuda.synchronize()
    launches = ops.launch_count() - launches0
    cnt = rt.counters()
    rep = rt.report()
    ledgers = [rep.ledger]
    if world > 1:  # the plan's ledger is the union of the ranks' executed rows
        import torch.distributed as dist
        ledgers = [None] * world
        dist.all_gather_object(ledgers, rep.ledger)
    ledger_ok = sorted(r for led in ledgers for r in led) == sorted(sim.ledger)
    # stream utilisation of the last timed iteration (measured CUDA events)
    busy = {"h2d": 0, "d2h": 0, "compute": 0, "update": 0}
    for e in rep.trace:
        key = ("compute" if e.resource.endswith(".compute") else "update" if e.resource.endswith(".update")
               else "h2d" if e.resource.endswith(".swap_in") else "d2h" if e.resource.endswith(".swap_out") else None)
        if key:
            busy[key] += e.end_ns - e.start_ns
    util = {k: round(v / max(1, cnt["iteration_ns"]), 4) for k, v in busy.items()}
    # achieved link rate of the swap streams while they move data (bytes / busy time
    # of the last timed iteration's transfers, measured CUDA events)
    moved = {"h2d": 0, "d2h": 0}
    for r in rep.ledger:
        if r[4] in ("cpu_gpu_swap", "message_passing") and r[7] == rank:
            moved["h2d" if r[1] == 0 else "d2h"] += r[6]
    swap_gbs = {k: round(moved[k] / busy[k], 2) if busy[k] else None for k in moved}
    _barrier(world)
    # per-kernel CUDA-event timings: one extra iteration with an event pair
    # around every kernel launch (kept out of the timed steps above, whose
    # value it would perturb)
    rt.set_profiling(True)
    rt.step(tok_d, lab_d)  # records the profiled graph
    rt.set_profiling(True)  # reset stats
    rt.step(tok_d, lab_d)
    kstats = rt.kernel_stats()
    kl = rt.kernel_launches()
    gemm_groups = _gemm_groups(kl)
    gk = kl[(kl[:, 0] == 0) & (kl[:, 4] > 0)]
    gemm_span_tflops = float(gk[:, 1].sum() / (gk[:, 4].sum() / 1e3) / 1e12) if len(gk) else 0.0
    prof_iter_ns = rt.counters()["iteration_ns"]
    gemm_shapes = rt.gemm_shapes()
    rt.set_profiling(False)
    # the GEMM's own rate: every shape of the iteration replayed back to back in
    # a CUDA graph (CUDA events around whole replays; no event nodes between
    # launches), weighted by how often the iteration launches it
    gemm_replay = []
    for shp, count in gemm_shapes:
        # best of three replays: right after the pipelined run a replay has read
        # up to 45% slow on the MN-major-B shapes of one box (the same shapes
        # replayed standalone, tools/gemm_shapes.py, did not)
        us = min(ops.gemm_replay_us(shp, reps=32) for _ in range(3))
        gemm_replay.append({"m": shp[0], "n": shp[1], "k": shp[2], "a_mn": shp[3], "b_mn": shp[4], "epi": shp[5],
                            "count": count, "us": round(us, 2),
                            "tflops": round(2.0 * shp[0] * shp[1] * shp[2] / (us * 1e-6) / 1e12, 1)})
    rp_flops = sum(2.0 * r["m"] * r["n"] * r["k"] * r["count"] for r in gemm_replay)
    rp_us = sum(r["us"] * r["count"] for r in gemm_replay)
    gemm_replay_tflops = rp_flops / (rp_us * 1e-6) / 1e12 if rp_us else 0.0
    gemm_replay.sort(key=lambda r: -r["us"] * r["count"])
    t_total = _max_over_ranks(t_dev, world)
    # e2e: tokens from pinned host memory every step, per-step losses read back
    _barrier(world)
    _, t_e2e = rt.run_steps(args.steps, tok_p, lab_p) if is_cnn else rt.run_steps(args.steps, tok_p.numpy(),
                                                                                   lab_p.numpy())
    t_e2e = _max_over_ranks(t_e2e, world)

    samples_per_step = D
    value = samples_per_step * args.steps / t_total
    e2e_value = samples_per_step * args.steps / t_e2e
    pk = _peaks()
    # dominant kernel: the tcgen05 GEMM (tensor-bound)
    g = kstats["gemm"]
    gemm_tflops = g["flops"] / (g["ms"] / 1e3) / 1e12 if g["ms"] else 0.0
    roof_tflops = gemm_tflops if is_cnn else gemm_replay_tflops
    ad = kstats["adam"]
    adam_gbs = ad["bytes"] / (ad["ms"] / 1e3) / 1e9 if ad["ms"] else 0.0
    # iteration roofline: compute at tensor peak vs PCIe H2D / D2H at measured link bandwidth
    flops = step_flops(graph, spec) / world
    swap_in = sum(r[6] for r in sim.ledger if r[1] == 0 and r[4] in ("cpu_gpu_swap", "message_passing") and r[7] == rank)
    swap_out = sum(r[6] for r in sim.ledger if r[1] == 2 and r[4] in ("cpu_gpu_swap", "message_passing") and r[7] == rank)
    t_compute = flops / (pk["bf16"] * 1e12)
    t_h2d = swap_in / (pcie["h2d"] * 1e9)
    t_d2h = swap_out / (pcie["d2h"] * 1e9)
    t_bidir = (swap_in + swap_out) / (pcie["bidir"] * 1e9)  # the link's two directions share ~92 GB/s
    # multi-GPU terms: the host root complex (every rank's swaps
    # at the aggregate concurrent rate), NCCL (ring volume at the measured bus
    # bandwidth), NVLink peer hand-offs (none under Harmony-DP)
    tot_in = sum(r[6] for r in sim.ledger if r[1] == 0 and r[4] in ("cpu_gpu_swap", "message_passing"))
    tot_out = sum(r[6] for r in sim.ledger if r[1] == 2 and r[4] in ("cpu_gpu_swap", "message_passing"))
    root_h2d = _sum_over_ranks(pcie_conc["h2d"], world)
    root_d2h = _sum_over_ranks(pcie_conc["d2h"], world)
    t_root = max(tot_in / (root_h2d * 1e9), tot_out / (root_d2h * 1e9)) if world > 1 else 0.0
    busbw = _nccl_busbw(world)
    t_nccl = cnt["nccl_bytes"] / (busbw * 1e9) if world > 1 and busbw else 0.0
    p2p = sum(r[6] for r in sim.ledger if r[4] == "peer2peer")
    t_phase = phase_bound_s(graph, sim.ledger, pcie, rank)
    t_phase = _max_over_ranks(t_phase, world)
    t_roof = max(t_compute, _max_over_ranks(max(t_h2d, t_d2h, t_bidir), world), t_root, t_nccl)
    ms_step = 1000.0 * t_total / args.steps
    clk = clocks.summary()
    share = {k: round(v["ms"] / (prof_iter_ns / 1e6), 4) for k, v in kstats.items()}
    line = {
        "metric": "samples/s (Harmony layer-pack training, GPT-2 XL)" if preset == "gpt2-xl"
                  else f"samples/s (Harmony layer-pack training, {spec.name})",
        "value": round(value, 3),
        "unit": "samples/s",
        "n_gpus": world,
        "steps": args.steps,
        "warmup": args.warmup,
        "ms_per_step": round(ms_step, 3),
        "higher_is_better": True,
        "scaling": "weak",
        "vs_baseline": None,
        "dtype": "bf16",
        "data": ("synthetic (images N(0,1), 3 channels zero-padded to 64, labels U[0,classes) seed 1234; "
                 "He-normal weights seed 0)") if is_cnn else
                "synthetic (tokens U[0,V) seed 1234; weights N(0,0.02) from a CUDA generator seeded 0)",
        "config": _config(args.workload, spec, mode, lpp, u, alpha_gib, D, world, payload),
        "swap_gb_per_iter": round((swap_in + swap_out) / 1e9, 3),
        "swap_h2d_gb": round(swap_in / 1e9, 3), "swap_d2h_gb": round(swap_out / 1e9, 3),
        "step_roofline": {"bound": ("tensor" if t_roof == t_compute else "host_root" if t_roof == t_root
                                    else "nccl" if t_roof == t_nccl else "pcie"),
                          "t_roof_ms": round(1000 * t_roof, 2),
                          "t_root_ms": round(1000 * t_root, 2), "t_nccl_ms": round(1000 * t_nccl, 2),
                          "t_nvlink_ms": 0.0, "p2p_bytes": p2p,
                          "root_gbs": {"h2d": round(root_h2d, 2), "d2h": round(root_d2h, 2)} if world > 1 else None,
                          "nccl_busbw_gbs": round(busbw, 1) if world > 1 else None,
                          "t_compute_ms": round(1000 * t_compute, 2), "t_h2d_ms": round(1000 * t_h2d, 2),
                          "t_d2h_ms": round(1000 * t_d2h, 2), "t_bidir_ms": round(1000 * t_bidir, 2),
                          "frac": round(1000 * t_roof / ms_step, 4),
                          "t_phase_ms": round(1000 * t_phase, 2),
                          "frac_phase": round(1000 * max(t_phase, t_compute) / ms_step, 4),
                          "phase_how": "sum over the forward and the backward + update windows of each window's "
                                       "own max(H2D / h2d, D2H / d2h, (H2D + D2H) / bidir) from the ledger "
                                       "(explanatory; frac above is the whole-step bound)",
                          "pcie_gbs": {k: round(v, 2) for k, v in pcie.items()},
                          "tensor_peak_tflops": pk["bf16"], "peak": pk["kind"]},
        "roofline": {"bound": "tensor", "achieved": round(roof_tflops, 1), "peak": pk["bf16"],
                     "unit": "TFLOP/s", "frac": round(roof_tflops / pk["bf16"], 4), "traffic": None,
                     "kernel": "hm::gemm::gemm_kernel (tcgen05)" + (" (implicit-GEMM 3x3 convolutions)" if is_cnn
                                                                    else ""),
                     "launches_per_step": g["launches"],
                     "share_of_step": share.get("gemm"),
                     "how": ("algorithmic 2 P 9 Cin Cout per convolution launch / its CUDA-event time in one profiled "
                             "iteration (graph event nodes around every launch; the replay below covers only the "
                             "classifier GEMM)") if is_cnn else
                            "algorithmic 2MNK per launch / the kernel's own per-launch time: each GEMM shape of one "
                            "iteration (logged while profiling it) replayed as a CUDA graph of 32 back-to-back launches "
                            "on rotating operand sets, CUDA events around whole graph replays (best of three), "
                            "weighted by the iteration's launch counts (gemm_replay)",
                     "peak_kind": "sustained (MEASURED_PEAKS bf16_tflops_sustained)",
                     "achieved_event_pairs": round(gemm_tflops, 1),
                     "event_pairs_how": "per-launch CUDA event pairs (graph event nodes) around every kernel of one "
                                        "profiled iteration: also times each graph node's launch and loses the PDL "
                                        "overlap with the neighbour",
                     "achieved_device_clock": round(gemm_span_tflops, 1),
                     "frac_device_clock": round(gemm_span_tflops / pk["bf16"], 4),
                     "device_clock_how": "same launches timed by the kernel itself: first CTA start (after "
                                         "griddepcontrol.wait) to last CTA end on %globaltimer; the event pair "
                                         "around each launch also times the graph's event nodes and loses PDL overlap",
                     **(_ncu_traffic() if args.workload == "gpt2-xl-dp" else {})},
        "kernel_shares": share,
        "gemm_by_gflop": gemm_groups,
        "gemm_replay": gemm_replay[:12],
        "stream_busy_frac": util,
        "swap_achieved_gbs": swap_gbs,
        "last_iter_ms_unpipelined_view": round(cnt["iteration_ns"] / 1e6, 2),
        "adam_hbm": {"achieved_gbs": round(adam_gbs, 1), "peak": pk["hbm"], "frac": round(adam_gbs / pk["hbm"], 4)},
        "e2e": {"value": round(e2e_value, 3), "unit": "samples/s", "h2d_bytes_per_step": int(in_bytes),
                "d2h_bytes_per_step": 8},
        "gpu_launches": int(launches),
        "clocks": clk,
        "loss": [round(_sum_over_ranks(x, world) if mode == "pp" else x, 5) for x in losses[-3:]],
        "ledger_rows": sum(len(x) for x in ledgers), "ledger_equals_plan": ledger_ok,
        "host_arena_numa_node": rt.lib.hm_runtime_numa_node(rt.handle),
        "device_bytes": cnt["device_bytes"],
        "nccl_allreduce_gb_per_iter": round(cnt["nccl_bytes"] / 1e9, 3),
    }
    if not args.no_cpu_baseline and rank == 0 and world == 1:
        # bounded sample: one measured full-depth iteration at D = 1 (GPT), one
        # sample through the whole chain (CNN)
        threads = len(os.sched_getaffinity(0))
        if is_cnn:
            line["cpu_baseline"] = cnn_port_sample(spec, threads, seconds_cap=20.0)
        else:
            it = cpu_port_iteration(spec, 1, threads)
            line["cpu_baseline"] = {k: it[k] for k in ("value", "unit", "cores", "kind", "sample")}
    if rank == 0:
        print(json.dumps(line), flush=True)
    rt.close()
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


def main() -> None:
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="native", choices=("native", "reference"))
    ap.add_argument("--workload", default="gpt2-xl-dp", choices=sorted(WORKLOADS))
    ap.add_argument("--alpha-gib", type=int, default=0)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3 and args.impl == "native":
        args.warmup = 3
    if args.impl == "native" and args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: relaunch under torchrun (the driver's own launch sets WORLD_SIZE)
        import socket
        import torch
        have = torch.cuda.device_count()
        if have < args.gpus and not SHARE_GPU:
            sys.stderr.write(f"bench.py: --gpus {args.gpus} but only {have} CUDA device(s) are visible\n")
            sys.exit(2)
        sk = socket.socket()
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
        sk.close()
        os.execv(sys.executable, [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
                                  f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
                                  f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:])
    if args.impl == "native" and int(os.environ.get("WORLD_SIZE", "1")) != args.gpus:
        sys.stderr.write(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={os.environ.get('WORLD_SIZE')}\n")
        sys.exit(2)
    # communicator set-up lines (rank count, NVLS / P2P transports) on stderr
    os.environ.setdefault("NCCL_DEBUG", "INFO")
    os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    os.environ.setdefault("NCCL_DEBUG_FILE", "/dev/stderr")
    if args.impl == "reference":
        run_reference(args)
    else:
        run_native(args)


if __name__ == "__main__":
    main()

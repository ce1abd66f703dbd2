"""``simulate``: the event-driven estimate of one iteration and its exact
swap ledger, computed by the native planner (csrc/plan.cpp).

Drop-in for `pkg/src/wrapsched/simulator.py:378-434`: same signature, same
``SimReport`` fields and byte accounting.  The plan that prices the
iteration here is the plan :func:`paper_2202_01306_b200.runtime.execute`
runs on the GPU, so estimate and execution share one ledger.
"""

from __future__ import annotations

from dataclasses import dataclass, field

from .core import MachineModel, TensorKind
from .errors import ValidationError
from .lowering import CHANNEL_OF, TENSOR_OF, NativePlan, ledger_rows, resource_name
from .profiler import ProfileSet
from .taskgraph import ChannelKind, Task, TaskGraph, TaskType


@dataclass(frozen=True)
class TraceEvent:
    resource: str
    task: int
    kind: str
    label: str
    start_ns: int
    end_ns: int


@dataclass
class SimReport:
    makespan_ns: int
    gpu_busy_ns: dict[int, int]
    gpu_idle_ns: dict[int, int]
    channel_volumes: dict[str, int]
    tensor_volumes: dict[str, dict[str, int]]
    per_gpu_volumes: dict[int, dict[str, int]]
    trace: list[TraceEvent]
    caveats: tuple[str, ...] = ()
    ledger: list[tuple] = field(default_factory=list)
    measured: bool = False

    @property
    def per_gpu_swap_bytes(self) -> dict[int, int]:
        sw = (ChannelKind.CPU_GPU_SWAP.value, ChannelKind.MESSAGE_PASSING.value)
        return {g: sum(v.get(c, 0) for c in sw) for g, v in self.per_gpu_volumes.items()}

    def tensor_total(self, tensor: TensorKind, channels: tuple[str, ...]) -> int:
        per = self.tensor_volumes.get(tensor.value, {})
        return sum(per.get(c, 0) for c in channels)

    def swap_volume(self, tensor: TensorKind) -> int:
        return self.tensor_total(tensor, (ChannelKind.CPU_GPU_SWAP.value,
                                          ChannelKind.MESSAGE_PASSING.value))


def _label(task: Task, it) -> tuple[str, str]:
    if it["is_compute"]:
        lo, hi = task.pack
        return "compute", f"{task.type.value} L{lo}-{hi} mb{int(it['member'])}"
    tensor = TENSOR_OF[int(it["tensor"])].value
    ch = CHANNEL_OF[int(it["channel"])]
    if ch is ChannelKind.PEER2PEER:
        return tensor, f"{tensor} p2p"
    return tensor, f"{tensor} {'in' if int(it['stage']) == 0 else 'out'}"


def report_from_items(graph: TaskGraph, machine: MachineModel, items, makespan: int,
                      measured: bool = False) -> SimReport:
    """Aggregate plan (or measured) items into a SimReport
    (`simulator.py:399-434`)."""
    n = machine.gpu_count
    busy = {g: 0 for g in range(n)}
    channel_volumes = {k.value: 0 for k in ChannelKind}
    tensor_volumes: dict[str, dict[str, int]] = {}
    per_gpu: dict[int, dict[str, int]] = {g: {} for g in range(n)}
    trace = []
    for it in items:
        task = graph.tasks[int(it["task"])]
        kind, label = _label(task, it)
        res0 = resource_name(int(it["res"][0]), n)
        trace.append(TraceEvent(res0, int(it["task"]), kind, label, int(it["start_ns"]),
                                int(it["end_ns"])))
        if it["is_compute"]:
            if res0.startswith("gpu"):
                busy[int(it["gpu"])] += int(it["end_ns"] - it["start_ns"]) if measured else int(it["duration_ns"])
            continue
        ch = CHANNEL_OF[int(it["channel"])].value
        tn = TENSOR_OF[int(it["tensor"])].value
        nb = int(it["nbytes"])
        channel_volumes[ch] += nb
        tensor_volumes.setdefault(tn, {}).setdefault(ch, 0)
        tensor_volumes[tn][ch] += nb
        bucket = per_gpu[int(it["gpu"])]
        bucket[ch] = bucket.get(ch, 0) + nb
    trace.sort(key=lambda e: (e.start_ns, e.resource, e.task, e.end_ns))
    caveats = []
    if graph.mode.value == "dp":
        if measured:
            caveats.append("data-parallel gradient all-reduce runs on NCCL and is reported "
                           "separately; the ledger counts only CPU-GPU and peer traffic")
        else:
            caveats.append("data-parallel gradient synchronization is modeled as a zero-cost "
                           "CPU-side reduction; only CPU-GPU swap traffic is accounted")
    return SimReport(makespan_ns=int(makespan), gpu_busy_ns=busy,
                     gpu_idle_ns={g: int(makespan) - b for g, b in busy.items()},
                     channel_volumes=channel_volumes, tensor_volumes=tensor_volumes,
                     per_gpu_volumes=per_gpu, trace=trace, caveats=tuple(caveats),
                     ledger=ledger_rows(items, n), measured=measured)


def simulate(graph: TaskGraph, machine: MachineModel | None = None,
             profiles: ProfileSet | None = None, *, check_memory: bool = False,
             w_fwd_bytes=None, dp_update: str = "replicated") -> SimReport:
    """Estimate one training iteration (drop-in for `simulator.simulate`).
    ``w_fwd_bytes`` (extension, default None = the reference): per-layer W
    bytes forward tasks move under the runtime's bf16 swap-payload mode
    (``HarmonyRuntime.w_fwd_bytes()``).  ``dp_update`` (extension, default
    the reference): "sharded" prices the Harmony-DP sharded update (rank g's
    U task moves / updates only shard g of the pack's K and W)."""
    machine = machine or graph.machine
    if profiles is None:
        raise ValidationError("profiles are required")
    if machine.gpu_count != graph.machine.gpu_count:
        raise ValidationError("machine does not match the graph's GPU count")
    graph.validate()
    plan = NativePlan(graph, machine, profiles, w_fwd_bytes=w_fwd_bytes, dp_update=dp_update)
    try:
        if check_memory:
            check_memory_fit(graph, machine, profiles)
        makespan = plan.simulate()
        items = plan.items()
    finally:
        plan.close()
    return report_from_items(graph, machine, items, makespan)


def estimate_makespan(graph: TaskGraph, machine: MachineModel, profiles: ProfileSet) -> int:
    """Makespan only (the search's inner loop): no trace or report assembly."""
    plan = NativePlan(graph, machine, profiles)
    try:
        return plan.simulate()
    finally:
        plan.close()


def task_mem_bytes(task: Task, profiles: ProfileSet) -> int:
    if task.type is TaskType.U:
        return 0
    u = max(task.group)
    lo, hi = task.pack
    mem = profiles.pack_mem_bytes(task.type.value, lo, hi, u)
    if task.type is TaskType.F:
        mem += profiles.x_bytes(lo, u)
    return mem


def check_memory_fit(graph: TaskGraph, machine: MachineModel, profiles: ProfileSet) -> None:
    """Resident task plus one prefetched task must fit alpha
    (`simulator.py:437-463`)."""
    per_dev: dict[tuple[str, int], list[Task]] = {}
    for t in graph.tasks:
        if t.device[0] == "gpu":
            per_dev.setdefault(t.device, []).append(t)
    for dev, ts in per_dev.items():
        for a, b in zip(ts, ts[1:]):
            need = task_mem_bytes(a, profiles) + task_mem_bytes(b, profiles)
            if need > machine.gpu_mem_capacity:
                raise ValidationError(
                    f"tasks {a.index} and {b.index} overflow gpu{dev[1]} memory "
                    f"({need} > {machine.gpu_mem_capacity}) with prefetch")


# ---------------------------------------------------------------------------
# Python mirror of the native plan's duration model and list scheduler.
#
# The planner itself lives in csrc/plan.cpp; these helpers restate two of its
# pieces in Python so a caller can price a task or run a hand-built item
# graph without the library — the reference exposes the same three helpers
# (`simulator.py:86-147`, `:347-375`) and its own tests import them.
# ---------------------------------------------------------------------------

def _xfer_ns(nbytes: int, bw: int) -> int:
    """ceil(nbytes * 1e9 / bw) — plan.cpp `xfer_ns`."""
    return -(-int(nbytes) * 1_000_000_000 // int(bw))


def _compute_duration(task: Task, u: int, profiles: ProfileSet,
                      machine: MachineModel) -> int:
    """Nanoseconds one member (microbatch ``u``) of ``task`` occupies its GPU,
    the rule plan.cpp `Ctx::compute_ns` applies (unsharded update)."""
    lo, hi = task.pack
    if task.type is TaskType.F:
        return profiles.pack_time_ns("F", lo, hi, u)
    if task.type is TaskType.B:
        fwd = profiles.pack_time_ns("F", lo, hi, u) if task.recompute else 0
        return profiles.pack_time_ns("B", lo, hi, u) + fwd
    layers = range(lo, hi + 1)
    if machine.cpu_offload_update:
        return sum(_xfer_ns(profiles.w_bytes(L), machine.update_cpu_rate) for L in layers)
    return sum(profiles.time_ns("U", L, 1) for L in layers)


class _Item:
    """One schedulable unit: a compute member or one tensor transfer.

    ``resources`` are held for ``duration`` once every predecessor has
    released it; ``key`` orders items that become ready at the same time
    (plan.cpp `Item` + its ready-queue ordering)."""

    __slots__ = ("key", "resources", "duration", "task", "kind", "label", "tensor",
                 "channel", "nbytes", "gpu", "idx", "pending", "ready", "dependents",
                 "start", "end")

    def __init__(self, key, resources, duration, task, kind, label,
                 tensor=None, channel=None, nbytes=0, gpu=None):
        self.key, self.resources, self.duration = key, tuple(resources), int(duration)
        self.task, self.kind, self.label = task, kind, label
        self.tensor, self.channel, self.nbytes, self.gpu = tensor, channel, nbytes, gpu
        self.idx = -1
        self.pending = 0            # predecessors not yet scheduled
        self.ready = 0              # earliest start the predecessors allow
        self.dependents: list[tuple[_Item, bool]] = []
        self.start = self.end = -1


def _link(dep: _Item | None, item: _Item, at_start: bool = False) -> None:
    """``item`` waits for ``dep`` to finish (or only to start, ``at_start``)."""
    if dep is not None:
        dep.dependents.append((item, at_start))
        item.pending += 1


def _run(items: list[_Item]) -> None:
    """Greedy list schedule: pop the ready item with the smallest
    (ready time, key), start it once all its resources are free, release its
    dependents.  Raises DeadlockError when a cycle strands items — the check
    plan.cpp reports as HM_ERR_DEADLOCK."""
    import heapq

    from .errors import DeadlockError

    free_at: dict = {}
    queue = [(0, it.key, n) for n, it in enumerate(items) if it.pending == 0]
    heapq.heapify(queue)
    scheduled = 0
    while queue:
        ready, _, n = heapq.heappop(queue)
        it = items[n]
        it.start = max([ready] + [free_at.get(r, 0) for r in it.resources])
        it.end = it.start + it.duration
        for r in it.resources:
            free_at[r] = it.end
        scheduled += 1
        for child, at_start in it.dependents:
            child.ready = max(child.ready, it.start if at_start else it.end)
            child.pending -= 1
            if child.pending == 0:
                heapq.heappush(queue, (child.ready, child.key, child.idx))
    if scheduled != len(items):
        raise DeadlockError(f"{len(items) - scheduled} of {len(items)} work items never "
                            "became runnable: the dependency graph has a cycle")

"""The per-iteration task schedule (paper Algorithm 3): F / B / U tasks over
layer packs and microbatch groups, wrap-around device binding and the
channel of every tensor movement.

This is the *program* the native runtime executes.  Structure, binding and
channel wiring follow `pkg/src/wrapsched/taskgraph.py:211-400` exactly, down
to dict insertion order, because the swap ledger's row order is derived from
it (`simulator.py:180-260`):

* PP: slot i of ``p_f + reversed(p_b)`` runs on GPU ``i mod N``; the B task
  of reversed slot r has index ``|P_F| + 2r`` and is followed by its jit U
  task on ``("cpu", gpu)``; every non-shared B pack's input is stashed by the
  F task holding its head layer (MESSAGE_PASSING) and recomputed.
* DP: every GPU replays the whole pack sequence on its ``gpu_shares`` slice
  with zero-copy (SHARED_MEMORY) activation hand-offs.

A U task's device is ``("cpu", k)`` for parity with the reference's model of
the update lane; the runtime executes it on GPU k's update stream with the
fused Adam kernel.
"""

from __future__ import annotations

from dataclasses import dataclass, field
from enum import Enum

from .core import (Configuration, LayerChain, MachineModel, Mode, Pack, TensorKind,
                   gpu_shares, microbatch_groups)
from .errors import InvalidConfigurationError, UnroutableBranchError, ValidationError
from .profiler import ProfileSet


class TaskType(str, Enum):
    F = "F"
    B = "B"
    U = "U"


class ChannelKind(str, Enum):
    CPU_GPU_SWAP = "cpu_gpu_swap"
    PEER2PEER = "peer2peer"
    MESSAGE_PASSING = "message_passing"
    SHARED_MEMORY = "shared_memory"


@dataclass(frozen=True)
class Channel:
    kind: ChannelKind
    src_task: int | None = None
    dst_task: int | None = None
    src_layer: int | None = None


Device = tuple[str, int]


@dataclass
class Task:
    index: int
    pack: Pack
    type: TaskType
    group: tuple[int, ...]
    device: Device
    inputs: dict[TensorKind, dict[int, Channel]] = field(default_factory=dict)
    outputs: dict[TensorKind, dict[int, Channel]] = field(default_factory=dict)
    recompute: bool = False

    @property
    def layers(self) -> range:
        return range(self.pack[0], self.pack[1] + 1)


@dataclass
class TaskGraph:
    tasks: list[Task]
    mode: Mode
    machine: MachineModel
    minibatch: int
    config: Configuration | None = None

    @property
    def gpu_count(self) -> int:
        return self.machine.gpu_count

    def validate(self) -> None:
        """Structural checks of `taskgraph.py:123-158`."""
        n = len(self.tasks)
        for i, t in enumerate(self.tasks):
            if t.index != i:
                raise ValidationError(f"task {i} carries index {t.index}")
            if t.device[0] not in ("gpu", "cpu") or not 0 <= t.device[1] < self.gpu_count:
                raise ValidationError(f"task {i} bound to unknown device {t.device}")
            for tensor, entries in t.inputs.items():
                for ch in entries.values():
                    if ch.src_task is None:
                        continue
                    if not 0 <= ch.src_task < n:
                        raise ValidationError(f"task {i} input from unknown task {ch.src_task}")
                    if ch.src_task >= i:
                        raise ValidationError(
                            f"task {i} consumes {tensor.value} from non-earlier task {ch.src_task}")
                    if (ch.kind is ChannelKind.PEER2PEER
                            and self.tasks[ch.src_task].device == t.device):
                        raise ValidationError(f"peer channel between colocated tasks {ch.src_task}->{i}")
            for tensor, entries in t.outputs.items():
                for ch in entries.values():
                    if ch.dst_task is not None and not i < ch.dst_task < n:
                        raise ValidationError(f"task {i} outputs {tensor.value} to invalid task {ch.dst_task}")
            if t.type is TaskType.U and self.config is not None:
                prev = self.tasks[i - 1] if i else None
                if prev is None or prev.type is not TaskType.B:
                    raise ValidationError(f"update task {i} does not follow a backward task")
                if t.device != ("cpu", prev.device[1]):
                    raise ValidationError(f"update task {i} is not colocated with its backward task")

    def device_order(self) -> dict[str, list[int]]:
        order: dict[str, list[int]] = {}
        for t in self.tasks:
            order.setdefault(f"{t.device[0]}{t.device[1]}", []).append(t.index)
        return order


def unroll_schedule(graph: TaskGraph) -> dict[str, list[int]]:
    """Per-device execution order (`taskgraph.py:167-169`)."""
    return graph.device_order()


def _check_chain(cfg: Configuration, chain: LayerChain) -> None:
    if not set(range(cfg.layer_count)) <= set(chain.layers):
        raise ValidationError("chain does not cover the configured layers")
    for ann in chain.relay_annotations:
        if ann.destination not in chain.layers or ann.source not in chain.layers:
            raise UnroutableBranchError(f"relay {ann.source}->{ann.destination} has no chain endpoint")
        if chain.position(ann.destination) <= chain.position(ann.source):
            raise UnroutableBranchError(f"relay {ann.source}->{ann.destination} has no downstream consumer")


def _route(src: Device, dst: Device, **kw) -> Channel:
    """Colocated hand-offs are zero-copy, others go peer-to-peer
    (`taskgraph.py:187-192`)."""
    kind = ChannelKind.SHARED_MEMORY if src == dst else ChannelKind.PEER2PEER
    return Channel(kind, **kw)


def _boundary(chain: LayerChain, prev_tail: int, head: int, src_task: int,
              src_dev: Device, dst_dev: Device, grad: bool) -> dict[int, Channel]:
    """Trunk tensor plus relay payloads crossing one pack boundary
    (`taskgraph.py:195-208`)."""
    out = {(prev_tail if grad else head): _route(src_dev, dst_dev, src_task=src_task)}
    synthetic = set(chain.synthetic_ids)
    for s in chain.boundary_sources(chain.position(prev_tail)):
        if s == prev_tail or s in synthetic:
            continue
        out[s] = _route(src_dev, dst_dev, src_task=src_task, src_layer=s)
    return out


def _weights_in(pack: Pack) -> dict[int, Channel]:
    return {L: Channel(ChannelKind.CPU_GPU_SWAP) for L in range(pack[0], pack[1] + 1)}


def _update(index: int, pack: Pack, gpu: int, b_index: int) -> Task:
    """jit-update task: W and dW in place from its B task, K swapped in,
    W and K swapped out (`taskgraph.py:324-343`)."""
    layers = range(pack[0], pack[1] + 1)
    shm = lambda: {L: Channel(ChannelKind.SHARED_MEMORY, src_task=b_index) for L in layers}
    swp = lambda: {L: Channel(ChannelKind.CPU_GPU_SWAP) for L in layers}
    return Task(index=index, pack=pack, type=TaskType.U, group=(1,), device=("cpu", gpu),
                inputs={TensorKind.W: shm(), TensorKind.DW: shm(), TensorKind.K: swp()},
                outputs={TensorKind.W: swp(), TensorKind.K: swp()})


def _containing(packs, layer: int, base: int = 0) -> int:
    for j, (lo, hi) in enumerate(packs):
        if lo <= layer <= hi:
            return base + j
    raise InvalidConfigurationError(f"layer {layer} not covered by p_f")


def _pp(cfg: Configuration, machine: MachineModel, chain: LayerChain) -> list[Task]:
    n = machine.gpu_count
    pf, pb = cfg.p_f, cfg.p_b
    nf, nb = len(pf), len(pb)
    gf = microbatch_groups(cfg.minibatch, cfg.u_f)
    gb = microbatch_groups(cfg.minibatch, cfg.u_b)
    f_dev = [("gpu", j % n) for j in range(nf)]
    rev = list(range(nb - 1, -1, -1))
    b_idx = {q: nf + 2 * r for r, q in enumerate(rev)}
    b_dev = {q: ("gpu", (nf + r) % n) for r, q in enumerate(rev)}
    synthetic = set(chain.synthetic_ids)

    tasks: list[Task] = []
    for j, pack in enumerate(pf):
        ins: dict[TensorKind, dict[int, Channel]] = {TensorKind.W: _weights_in(pack)}
        if j > 0:
            ins[TensorKind.X] = _boundary(chain, pf[j - 1][1], pack[0], j - 1,
                                          f_dev[j - 1], f_dev[j], grad=False)
        tail = pack[1]
        if j < nf - 1:
            dst, dst_dev = j + 1, f_dev[j + 1]
        else:
            dst, dst_dev = b_idx[nb - 1], b_dev[nb - 1]
        y = {tail: _route(f_dev[j], dst_dev, dst_task=dst)}
        if j < nf - 1:
            for s in chain.boundary_sources(chain.position(tail)):
                if s != tail and s not in synthetic:
                    y[s] = _route(f_dev[j], dst_dev, dst_task=dst, src_layer=s)
        outs: dict[TensorKind, dict[int, Channel]] = {TensorKind.Y: y}
        for q in range(nb - 1):
            head = pb[q][0]
            if pack[0] <= head <= pack[1]:
                outs.setdefault(TensorKind.SX, {})[head] = Channel(
                    ChannelKind.MESSAGE_PASSING, dst_task=b_idx[q])
        tasks.append(Task(j, pack, TaskType.F, gf, f_dev[j], ins, outs))

    for r, q in enumerate(rev):
        idx = nf + 2 * r
        pack = pb[q]
        shared = q == nb - 1
        dev = b_dev[q]
        ins = {TensorKind.W: _weights_in(pack)}
        outs = {}
        if shared:
            ins[TensorKind.Y] = {pack[1]: _route(f_dev[nf - 1], dev, src_task=nf - 1)}
        else:
            ins[TensorKind.DY] = _boundary(chain, pack[1], pack[1], b_idx[q + 1],
                                           b_dev[q + 1], dev, grad=True)
            ins[TensorKind.SX] = {pack[0]: Channel(ChannelKind.MESSAGE_PASSING,
                                                   src_task=_containing(pf, pack[0]))}
        if q > 0:
            outs[TensorKind.DX] = {pack[0]: _route(dev, b_dev[q - 1], dst_task=b_idx[q - 1])}
        tasks.append(Task(idx, pack, TaskType.B, gb, dev, ins, outs, recompute=not shared))
        tasks.append(_update(idx + 1, pack, dev[1], idx))
    return tasks


def _dp(cfg: Configuration, machine: MachineModel, chain: LayerChain) -> list[Task]:
    pf, pb = cfg.p_f, cfg.p_b
    nf, nb = len(pf), len(pb)
    tasks: list[Task] = []
    for gpu, share in enumerate(gpu_shares(cfg.minibatch, machine.gpu_count)):
        if share == 0:
            continue
        gf = microbatch_groups(share, min(cfg.u_f, share))
        gb = microbatch_groups(share, min(cfg.u_b, share))
        base = len(tasks)
        dev = ("gpu", gpu)
        for j, pack in enumerate(pf):
            ins: dict[TensorKind, dict[int, Channel]] = {TensorKind.W: _weights_in(pack)}
            if j > 0:
                ins[TensorKind.X] = {pack[0]: Channel(ChannelKind.SHARED_MEMORY, src_task=base + j - 1)}
            outs: dict[TensorKind, dict[int, Channel]] = {}
            for q in range(nb - 1):
                head = pb[q][0]
                if pack[0] <= head <= pack[1]:
                    outs.setdefault(TensorKind.SX, {})[head] = Channel(
                        ChannelKind.MESSAGE_PASSING, dst_task=base + nf + 2 * (nb - 1 - q))
            tasks.append(Task(base + j, pack, TaskType.F, gf, dev, ins, outs))
        for r, q in enumerate(range(nb - 1, -1, -1)):
            idx = base + nf + 2 * r
            pack = pb[q]
            shared = q == nb - 1
            ins = {TensorKind.W: _weights_in(pack)}
            if shared:
                ins[TensorKind.Y] = {pack[1]: Channel(ChannelKind.SHARED_MEMORY, src_task=base + nf - 1)}
            else:
                ins[TensorKind.DY] = {pack[1]: Channel(ChannelKind.SHARED_MEMORY, src_task=idx - 2)}
                ins[TensorKind.SX] = {pack[0]: Channel(ChannelKind.MESSAGE_PASSING,
                                                       src_task=_containing(pf, pack[0], base))}
            tasks.append(Task(idx, pack, TaskType.B, gb, dev, ins, {}, recompute=not shared))
            tasks.append(_update(idx + 1, pack, gpu, idx))
    return tasks


def generate_task_graph(cfg: Configuration, machine: MachineModel, profiles: ProfileSet,
                        chain: LayerChain | None = None) -> TaskGraph:
    """Build and validate one iteration's task graph (`taskgraph.py:211-236`)."""
    cfg.validate()
    if profiles.layer_count < cfg.layer_count:
        raise InvalidConfigurationError(
            f"profiles cover {profiles.layer_count} layers, configuration needs {cfg.layer_count}")
    chain = chain if chain is not None else LayerChain.linear(cfg.layer_count)
    _check_chain(cfg, chain)
    tasks = _pp(cfg, machine, chain) if cfg.mode is Mode.PP else _dp(cfg, machine, chain)
    graph = TaskGraph(tasks=tasks, mode=cfg.mode, machine=machine,
                      minibatch=cfg.minibatch, config=cfg)
    graph.validate()
    return graph

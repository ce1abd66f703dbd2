"""Lower a TaskGraph + ProfileSet + MachineModel into the flat C tables of
``hm_plan_build`` (include/harmony_b200.h) and wrap the resulting native plan.

This is the boundary between the Python planner API (drop-in with the
reference) and the native runtime: Python builds the graph once per job, the
extension owns the per-item swap plan, its ledger and the execution.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _native as N
from .core import MachineModel, TensorKind
from .errors import MissingProfileError, ValidationError
from .profiler import ProfileSet
from .taskgraph import ChannelKind, TaskGraph, TaskType

TENSOR_ID = {TensorKind.X: 0, TensorKind.Y: 1, TensorKind.DX: 2, TensorKind.DY: 3,
             TensorKind.W: 4, TensorKind.DW: 5, TensorKind.K: 6, TensorKind.SX: 7}
TENSOR_OF = {v: k for k, v in TENSOR_ID.items()}
CHANNEL_ID = {ChannelKind.CPU_GPU_SWAP: 0, ChannelKind.PEER2PEER: 1,
              ChannelKind.MESSAGE_PASSING: 2, ChannelKind.SHARED_MEMORY: 3}
CHANNEL_OF = {v: k for k, v in CHANNEL_ID.items()}
TYPE_ID = {TaskType.F: 0, TaskType.B: 1, TaskType.U: 2}
RES_NAMES = ("compute", "swap_in", "swap_out", "p2p_in", "p2p_out", "update", "root_out", "root_in")


def resource_name(res_id: int, gpu_count: int) -> str:
    kind, gpu = divmod(int(res_id), gpu_count)
    if kind == 5:
        return f"cpu{gpu}.update"
    if kind in (6, 7):
        return f"host.{RES_NAMES[kind]}"
    return f"gpu{gpu}.{RES_NAMES[kind]}"


def _arr(values, ctype):
    a = (ctype * max(1, len(values)))()
    a[:len(values)] = values
    return a


class NativePlan:
    """Owns an ``hm_plan*`` and the ctypes tables it was built from."""

    def __init__(self, graph: TaskGraph, machine: MachineModel, profiles: ProfileSet,
                 need_time: bool = True, w_fwd_bytes=None, dp_update: str = "replicated") -> None:
        """``w_fwd_bytes``: per-layer W bytes a forward task moves, for the
        runtime's bf16 swap-payload mode (None = the reference's W bytes).
        ``dp_update``: "replicated" (the reference: every Harmony-DP rank
        updates its own replica) or "sharded" (hm_machine.dp_sharded_update:
        rank g updates shard g of each pack; fast mode, not the reference
        ledger at N > 1)."""
        if dp_update not in ("replicated", "sharded"):
            raise ValidationError(f"dp_update must be 'replicated' or 'sharded' (got {dp_update!r})")
        if dp_update == "sharded" and graph.mode.value != "dp":
            raise ValidationError("the sharded update applies to Harmony-DP graphs only")
        lib = N.lib()
        self.graph = graph
        self.machine = machine
        tasks = graph.tasks
        n = len(tasks)
        self._tasks = (N.hm_task * max(1, n))()
        groups: list[int] = []
        entries: list[tuple] = []
        layers_needed = 0
        u_top = 1
        for t in tasks:
            rec = self._tasks[t.index]
            rec.index, rec.type, rec.lo, rec.hi = t.index, TYPE_ID[t.type], t.pack[0], t.pack[1]
            rec.dev_kind = 0 if t.device[0] == "gpu" else 1
            rec.dev_id = t.device[1]
            rec.recompute = 1 if t.recompute else 0
            rec.group_off, rec.group_len = len(groups), len(t.group)
            groups.extend(t.group)
            u_top = max(u_top, max(t.group))
            layers_needed = max(layers_needed, t.pack[1] + 1)
            rec.in_off = len(entries)
            for tensor, ents in t.inputs.items():
                for layer, ch in ents.items():
                    entries.append((TENSOR_ID[tensor], layer, CHANNEL_ID[ch.kind],
                                    -1 if ch.src_task is None else ch.src_task,
                                    -1 if ch.src_layer is None else ch.src_layer))
                    layers_needed = max(layers_needed, layer + 1,
                                        (ch.src_layer or 0) + 1)
            rec.in_len = len(entries) - rec.in_off
            rec.out_off = len(entries)
            for tensor, ents in t.outputs.items():
                for layer, ch in ents.items():
                    entries.append((TENSOR_ID[tensor], layer, CHANNEL_ID[ch.kind],
                                    -1 if ch.dst_task is None else ch.dst_task,
                                    -1 if ch.src_layer is None else ch.src_layer))
                    layers_needed = max(layers_needed, layer + 1, (ch.src_layer or 0) + 1)
            rec.out_len = len(entries) - rec.out_off
        self._groups = _arr(groups, C.c_int32)
        self._entries = (N.hm_entry * max(1, len(entries)))()
        for i, e in enumerate(entries):
            self._entries[i] = N.hm_entry(*e)

        group_of = [machine.p2p_group_of(g) for g in range(machine.gpu_count)]
        self._group_of = _arr(group_of, C.c_int32)
        self._machine = N.hm_machine(machine.gpu_count, 1 if machine.cpu_offload_update else 0,
                                     machine.pcie_bandwidth, machine.root_link_bandwidth,
                                     machine.p2p_bandwidth, machine.update_cpu_rate,
                                     C.cast(self._group_of, C.POINTER(C.c_int32)),
                                     1 if dp_update == "sharded" else 0)
        layers = max(layers_needed, 1)
        tab = profiles.tables(layers, u_top, need_time=need_time)
        self._tab = {}
        for key in ("x", "y", "t_f", "t_b", "t_u"):
            src = {"t_f": "tF", "t_b": "tB", "t_u": "tU"}.get(key, key)
            if src not in tab:
                self._tab[key] = None
                continue
            flat = np.ascontiguousarray(np.asarray(tab[src], dtype=np.int64).reshape(-1))
            self._tab[key] = flat
        for key in ("w", "dw", "k"):
            self._tab[key] = np.ascontiguousarray(np.asarray(tab[key], dtype=np.int64))

        def ptr(a):
            if a is None:
                return C.POINTER(C.c_int64)()
            return a.ctypes.data_as(C.POINTER(C.c_int64))

        self._tab["w_f"] = None
        if w_fwd_bytes is not None:
            wf = np.zeros(layers, dtype=np.int64) - 1
            wf[:min(layers, len(w_fwd_bytes))] = np.asarray(w_fwd_bytes, dtype=np.int64)[:layers]
            self._tab["w_f"] = wf
        self._profile = N.hm_profile(layers, u_top, *(ptr(self._tab[k]) for k in
                                                      ("x", "y", "w", "dw", "k", "t_f", "t_b", "t_u", "w_f")))
        status = C.c_int32(0)
        handle = lib.hm_plan_build(self._tasks, n, C.cast(self._groups, C.POINTER(C.c_int32)),
                                   self._entries, C.byref(self._machine), C.byref(self._profile),
                                   C.byref(status))
        if not handle:
            msg = N.last_error()
            if status.value == -5:
                raise MissingProfileError(msg)
            N.check(status.value)
        self.handle = handle
        self._simulated = False

    def simulate(self) -> int:
        ms = C.c_int64(0)
        N.check(N.lib().hm_plan_simulate(self.handle, C.byref(ms)))
        self._simulated = True
        return ms.value

    def items(self) -> np.ndarray:
        lib = N.lib()
        n = lib.hm_plan_item_count(self.handle)
        buf = np.zeros(n, dtype=N.ITEM_DTYPE)
        N.check(lib.hm_plan_items(self.handle, buf.ctypes.data, n))
        return buf

    def edges(self) -> np.ndarray:
        lib = N.lib()
        n = lib.hm_plan_edge_count(self.handle)
        dep = (C.c_int32 * max(1, n))()
        item = (C.c_int32 * max(1, n))()
        st = (C.c_int32 * max(1, n))()
        N.check(lib.hm_plan_edges(self.handle, dep, item, st, n))
        return np.array([(dep[i], item[i], st[i]) for i in range(n)], dtype=np.int64).reshape(-1, 3)

    def close(self) -> None:
        if getattr(self, "handle", None):
            N.lib().hm_plan_free(self.handle)
            self.handle = None

    def __del__(self) -> None:
        try:
            self.close()
        except Exception:
            pass


def ledger_rows(items: np.ndarray, gpu_count: int) -> list[tuple]:
    """Ledger in the oracle's comparison form (SURVEY §8c recipe):
    (task, stage, member, tensor, channel, resources, nbytes, gpu), sorted."""
    rows = []
    for it in items:
        if it["is_compute"]:
            continue
        res = tuple(resource_name(r, gpu_count) for r in it["res"][: it["n_res"]])
        rows.append((int(it["task"]), int(it["stage"]), int(it["member"]),
                     TENSOR_OF[int(it["tensor"])].value, CHANNEL_OF[int(it["channel"])].value,
                     res, int(it["nbytes"]), int(it["gpu"])))
    return sorted(rows)

"""ORACLE (test infrastructure only -- never imported by the product path).

Pure-Python CPU restatement of the reference's task schedule and swap plan,
operating on plain dicts so it shares no code with the product:

* ``task_graph``      <- taskgraph.generate_task_graph / _pp_tasks / _dp_tasks
                         (pkg/src/wrapsched/taskgraph.py:211-236, 244-321, 346-400)
* ``ledger_items``    <- simulator._build_items (simulator.py:150-336)
* ``run``             <- simulator._run (simulator.py:347-375)

Pinned against golden vectors generated from the reference itself
(oracle/make_golden.py -> tests/golden/schedule_ledger.json) and against the
reference tests' hand-traced values (tests/test_oracle.py).
Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline may use it.
"""

from __future__ import annotations

import heapq

NS = 1_000_000_000
TNAME = {"X": "X", "Y": "Y", "dX": "dX", "dY": "dY", "W": "W", "dW": "dW", "K": "K", "sX": "sX"}


def groups_of(total: int, u: int) -> list[int]:
    """core.microbatch_groups (core.py:332-345)."""
    q, r = divmod(total, u)
    return [u] * q + ([r] if r else [])


def shares(d: int, n: int) -> list[int]:
    """core.gpu_shares (core.py:348-351)."""
    q, r = divmod(d, n)
    return [q + 1 if k < r else q for k in range(n)]


def _ch(kind, src=None, dst=None, src_layer=None):
    return {"kind": kind, "src": src, "dst": dst, "src_layer": src_layer}


def _local(a, b, **kw):
    """taskgraph._p2p_or_local (taskgraph.py:187-192)."""
    return _ch("shared_memory" if a == b else "peer2peer", **kw)


def task_graph(cfg: dict, n_gpus: int) -> list[dict]:
    """Linear-chain task graph (taskgraph.py:244-321 PP, 346-400 DP).

    ``cfg`` = {u_f, p_f, u_b, p_b, minibatch, mode}; packs are [lo, hi]."""
    pf = [tuple(p) for p in cfg["p_f"]]
    pb = [tuple(p) for p in cfg["p_b"]]
    nf, nb = len(pf), len(pb)

    def upd(idx, pack, gpu, b):  # taskgraph.py:324-343
        L = range(pack[0], pack[1] + 1)
        return {"index": idx, "pack": pack, "type": "U", "group": [1], "device": ("cpu", gpu),
                "recompute": False,
                "inputs": [("W", {l: _ch("shared_memory", src=b) for l in L}),
                           ("dW", {l: _ch("shared_memory", src=b) for l in L}),
                           ("K", {l: _ch("cpu_gpu_swap") for l in L})],
                "outputs": [("W", {l: _ch("cpu_gpu_swap") for l in L}),
                            ("K", {l: _ch("cpu_gpu_swap") for l in L})]}

    def win(pack):
        return {l: _ch("cpu_gpu_swap") for l in range(pack[0], pack[1] + 1)}

    def f_of(layer, base=0):
        for j, (lo, hi) in enumerate(pf):
            if lo <= layer <= hi:
                return base + j
        raise ValueError(layer)

    tasks = []
    if cfg["mode"] == "pp":
        gf, gb = groups_of(cfg["minibatch"], cfg["u_f"]), groups_of(cfg["minibatch"], cfg["u_b"])
        fdev = [("gpu", j % n_gpus) for j in range(nf)]
        rev = list(reversed(range(nb)))
        bidx = {q: nf + 2 * r for r, q in enumerate(rev)}
        bdev = {q: ("gpu", (nf + r) % n_gpus) for r, q in enumerate(rev)}
        for j, pack in enumerate(pf):
            ins = [("W", win(pack))]
            if j > 0:
                ins.append(("X", {pack[0]: _local(fdev[j - 1], fdev[j], src=j - 1)}))
            dst, ddev = (j + 1, fdev[j + 1]) if j < nf - 1 else (bidx[nb - 1], bdev[nb - 1])
            outs = [("Y", {pack[1]: _local(fdev[j], ddev, dst=dst)})]
            sx = {}
            for q in range(nb - 1):
                if pack[0] <= pb[q][0] <= pack[1]:
                    sx[pb[q][0]] = _ch("message_passing", dst=bidx[q])
            if sx:
                outs.append(("sX", sx))
            tasks.append({"index": j, "pack": pack, "type": "F", "group": gf, "device": fdev[j],
                          "recompute": False, "inputs": ins, "outputs": outs})
        for r, q in enumerate(rev):
            idx, pack, dev = nf + 2 * r, pb[q], bdev[q]
            shared = q == nb - 1
            ins = [("W", win(pack))]
            outs = []
            if shared:
                ins.append(("Y", {pack[1]: _local(fdev[nf - 1], dev, src=nf - 1)}))
            else:
                ins.append(("dY", {pack[1]: _local(bdev[q + 1], dev, src=bidx[q + 1])}))
                ins.append(("sX", {pack[0]: _ch("message_passing", src=f_of(pack[0]))}))
            if q > 0:
                outs.append(("dX", {pack[0]: _local(dev, bdev[q - 1], dst=bidx[q - 1])}))
            tasks.append({"index": idx, "pack": pack, "type": "B", "group": gb, "device": dev,
                          "recompute": not shared, "inputs": ins, "outputs": outs})
            tasks.append(upd(idx + 1, pack, dev[1], idx))
        return tasks
    for gpu, share in enumerate(shares(cfg["minibatch"], n_gpus)):
        if share == 0:
            continue
        gf = groups_of(share, min(cfg["u_f"], share))
        gb = groups_of(share, min(cfg["u_b"], share))
        base = len(tasks)
        dev = ("gpu", gpu)
        for j, pack in enumerate(pf):
            ins = [("W", win(pack))]
            if j > 0:
                ins.append(("X", {pack[0]: _ch("shared_memory", src=base + j - 1)}))
            sx = {}
            for q in range(nb - 1):
                if pack[0] <= pb[q][0] <= pack[1]:
                    sx[pb[q][0]] = _ch("message_passing", dst=base + nf + 2 * (nb - 1 - q))
            tasks.append({"index": base + j, "pack": pack, "type": "F", "group": gf, "device": dev,
                          "recompute": False, "inputs": ins, "outputs": [("sX", sx)] if sx else []})
        for r, q in enumerate(reversed(range(nb))):
            idx, pack = base + nf + 2 * r, pb[q]
            shared = q == nb - 1
            ins = [("W", win(pack))]
            if shared:
                ins.append(("Y", {pack[1]: _ch("shared_memory", src=base + nf - 1)}))
            else:
                ins.append(("dY", {pack[1]: _ch("shared_memory", src=idx - 2)}))
                ins.append(("sX", {pack[0]: _ch("message_passing", src=f_of(pack[0], base))}))
            tasks.append({"index": idx, "pack": pack, "type": "B", "group": gb, "device": dev,
                          "recompute": not shared, "inputs": ins, "outputs": []})
            tasks.append(upd(idx + 1, pack, gpu, idx))
    return tasks


def xfer_ns(nbytes: int, bw: int) -> int:
    """simulator._xfer_ns (simulator.py:45-46)."""
    return (nbytes * NS + bw - 1) // bw


class Item:
    __slots__ = ("key", "res", "dur", "task", "kind", "tensor", "channel", "nbytes", "gpu",
                 "deps", "kids", "pending", "ready", "start", "end")

    def __init__(self, key, res, dur, task, kind, tensor=None, channel=None, nbytes=0, gpu=None):
        self.key, self.res, self.dur, self.task, self.kind = key, res, dur, task, kind
        self.tensor, self.channel, self.nbytes, self.gpu = tensor, channel, nbytes, gpu
        self.kids, self.pending, self.ready, self.start, self.end = [], 0, 0, -1, -1


def ledger_items(tasks: list[dict], machine: dict, prof: dict) -> list[Item]:
    """simulator._build_items (simulator.py:150-336) over plain tables.

    ``machine`` = {gpu_count, pcie, root, p2p_group_of: [..], cpu_offload_update,
    update_cpu_rate}; ``prof`` = {x, y: [[layer][u]], w, dw, k: [layer],
    tF, tB, tU: [[layer][u]]}."""
    pcie, root = machine["pcie"], machine["root"]
    swap_bw = min(pcie, root)
    grp = machine["p2p_group_of"]
    items: list[Item] = []
    seq = 0

    def eb(tensor, layer, ch, u):  # simulator.py:118-130
        if tensor == "W":
            return prof["w"][layer]
        if tensor == "dW":
            return prof["dw"][layer]
        if tensor == "K":
            return prof["k"][layer]
        if ch["src_layer"] is not None:
            return prof["y"][ch["src_layer"]][u]
        if tensor in ("X", "sX", "dX"):
            return prof["x"][layer][u]
        return prof["y"][layer][u]

    def cdur(t, u):  # simulator.py:133-147
        lo, hi = t["pack"]
        if t["type"] == "F":
            return sum(prof["tF"][l][u] for l in range(lo, hi + 1))
        if t["type"] == "B":
            d = sum(prof["tB"][l][u] for l in range(lo, hi + 1))
            if t["recompute"]:
                d += sum(prof["tF"][l][u] for l in range(lo, hi + 1))
            return d
        if machine["cpu_offload_update"]:
            return sum(xfer_ns(prof["w"][l], machine["update_cpu_rate"]) for l in range(lo, hi + 1))
        return sum(prof["tU"][l][1] for l in range(lo, hi + 1))

    def add(it):
        items.append(it)
        return it

    def link(dep, it, at_start=False):
        if dep is None:
            return
        dep.kids.append((it, at_start))
        it.pending += 1

    def p2p_res(a, b):  # simulator.py:339-344
        r = (f"gpu{a}.p2p_out", f"gpu{b}.p2p_in")
        if grp[a] != grp[b]:
            r += ("host.root_in", "host.root_out")
        return r

    members: dict[int, list[Item]] = {}
    first: dict[int, Item] = {}
    mp_out: dict[tuple, list[Item]] = {}
    prev_dev: dict[tuple, dict] = {}
    by_index = {t["index"]: t for t in tasks}
    for t in tasks:
        gpu = t["device"][1]
        prev = prev_dev.get(t["device"])
        upd = t["type"] == "U"
        tin, gate0, mgate, shm = [], [], {}, []
        swap: dict[str, int] = {}
        for tensor, entries in t["inputs"]:
            by_src: dict[int, int] = {}
            aligned: dict[int, list[int]] = {}
            for layer, ch in entries.items():
                if ch["kind"] == "cpu_gpu_swap":
                    swap[tensor] = swap.get(tensor, 0) + eb(tensor, layer, ch, t["group"][0])
                elif ch["kind"] == "shared_memory":
                    src = by_index[ch["src"]]
                    shm.append((src, src["group"] == t["group"]))
                elif ch["kind"] == "message_passing":
                    nb = sum(eb(tensor, layer, ch, u) for u in t["group"])
                    if nb == 0:
                        gate0.append(members[ch["src"]][-1])
                        continue
                    seq += 1
                    it = add(Item((t["index"], 0, 0, seq), (f"gpu{gpu}.swap_in", "host.root_out"),
                                  xfer_ns(nb, swap_bw), t["index"], tensor, tensor,
                                  "message_passing", nb, gpu))
                    for leg in mp_out.get((ch["src"], t["index"], layer), ()):
                        link(leg, it)
                    tin.append(it)
                else:  # peer2peer
                    src = by_index[ch["src"]]
                    if src["group"] == t["group"]:
                        per = aligned.setdefault(ch["src"], [0] * len(t["group"]))
                        for g, u in enumerate(t["group"]):
                            per[g] += eb(tensor, layer, ch, u)
                    else:
                        by_src[ch["src"]] = by_src.get(ch["src"], 0) + sum(
                            eb(tensor, layer, ch, u) for u in t["group"])
            for s, per in aligned.items():
                res = p2p_res(by_index[s]["device"][1], gpu)
                bw = pcie if len(res) == 2 else swap_bw
                for g, nb in enumerate(per):
                    if nb == 0:
                        mgate.setdefault(g, []).append(members[s][g])
                        continue
                    seq += 1
                    it = add(Item((t["index"], 0, g, seq), res, xfer_ns(nb, bw), t["index"], tensor,
                                  tensor, "peer2peer", nb, gpu))
                    link(members[s][g], it)
                    mgate.setdefault(g, []).append(it)
            for s, nb in by_src.items():
                if nb == 0:
                    gate0.append(members[s][-1])
                    continue
                res = p2p_res(by_index[s]["device"][1], gpu)
                bw = pcie if len(res) == 2 else swap_bw
                seq += 1
                it = add(Item((t["index"], 0, 0, seq), res, xfer_ns(nb, bw), t["index"], tensor,
                              tensor, "peer2peer", nb, gpu))
                link(members[s][-1], it)
                tin.append(it)
        for tensor, nb in sorted(swap.items()):
            if nb == 0:
                continue
            seq += 1
            tin.append(add(Item((t["index"], 0, 0, seq), (f"gpu{gpu}.swap_in", "host.root_out"),
                                xfer_ns(nb, swap_bw), t["index"], tensor, tensor, "cpu_gpu_swap",
                                nb, gpu)))
        window = first.get(t["index"] - 1) if upd else (first[prev["index"]] if prev else None)
        for it in tin:
            link(window, it, True)
        comps = []
        res = f"cpu{gpu}.update" if t["device"][0] == "cpu" else f"gpu{gpu}.compute"
        for g, u in enumerate(t["group"] if not upd else [1]):
            seq += 1
            it = add(Item((t["index"], 1, g, seq), (res,), cdur(t, u), t["index"], "compute", gpu=gpu))
            if g == 0:
                if prev is not None:
                    link(members[prev["index"]][-1], it)
                for d in tin + gate0:
                    link(d, it)
                for src, al in shm:
                    if not al:
                        link(members[src["index"]][-1], it)
            else:
                link(comps[g - 1], it)
            for src, al in shm:
                if al:
                    link(members[src["index"]][g], it)
            for d in mgate.get(g, ()):
                link(d, it)
            comps.append(it)
        members[t["index"]] = comps
        first[t["index"]] = comps[0]
        prev_dev[t["device"]] = t
        out_swap: dict[str, int] = {}
        for tensor, entries in t["outputs"]:
            for layer, ch in entries.items():
                if ch["kind"] == "message_passing":
                    for g, u in enumerate(t["group"]):
                        nb = eb(tensor, layer, ch, u)
                        if nb == 0:
                            continue
                        seq += 1
                        it = add(Item((t["index"], 2, g, seq), (f"gpu{gpu}.swap_out", "host.root_in"),
                                      xfer_ns(nb, swap_bw), t["index"], tensor, tensor,
                                      "message_passing", nb, gpu))
                        link(comps[g], it)
                        mp_out.setdefault((t["index"], ch["dst"], layer), []).append(it)
                elif ch["kind"] == "cpu_gpu_swap":
                    out_swap[tensor] = out_swap.get(tensor, 0) + eb(tensor, layer, ch, t["group"][0])
        for tensor, nb in sorted(out_swap.items()):
            if nb == 0:
                continue
            seq += 1
            it = add(Item((t["index"], 2, 0, seq), (f"gpu{gpu}.swap_out", "host.root_in"),
                          xfer_ns(nb, swap_bw), t["index"], tensor, tensor, "cpu_gpu_swap", nb, gpu))
            link(comps[-1], it)
    return items


def run(items: list[Item]) -> int:
    """simulator._run (simulator.py:347-375); returns the makespan."""
    busy: dict[str, int] = {}
    heap = [(0, it.key, i) for i, it in enumerate(items) if it.pending == 0]
    heapq.heapify(heap)
    index = {id(it): i for i, it in enumerate(items)}
    done = 0
    while heap:
        ready, _, i = heapq.heappop(heap)
        it = items[i]
        start = max([ready] + [busy.get(r, 0) for r in it.res])
        it.start, it.end = start, start + it.dur
        for r in it.res:
            busy[r] = it.end
        done += 1
        for kid, at_start in it.kids:
            kid.ready = max(kid.ready, start if at_start else it.end)
            kid.pending -= 1
            if kid.pending == 0:
                heapq.heappush(heap, (kid.ready, kid.key, index[id(kid)]))
    if done != len(items):
        raise RuntimeError("deadlock")
    return max((it.end for it in items), default=0)


def ledger_rows(items: list[Item]) -> list[tuple]:
    """SURVEY §8c comparison form: sorted (task, stage, member, tensor,
    channel, resources, nbytes, gpu) over non-compute items."""
    return sorted((it.task, it.key[1], it.key[2], it.tensor, it.channel, tuple(it.res), it.nbytes,
                   it.gpu) for it in items if it.kind != "compute")


def unroll(tasks: list[dict]) -> dict[str, list[int]]:
    """taskgraph.unroll_schedule (taskgraph.py:160-169)."""
    out: dict[str, list[int]] = {}
    for t in tasks:
        out.setdefault(f"{t['device'][0]}{t['device'][1]}", []).append(t["index"])
    return out

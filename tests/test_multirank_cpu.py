"""Multi-process (gloo, world_size 2, CPU) checks of the Harmony-DP / PP host
logic: every rank derives the same global plan, its own task subset and
sample range; the ranks' executed-ledger slices partition the global ledger;
the per-pack all-reduce sequence is identical on every rank (NCCL requires
the same collective order)."""

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, mode, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2202_01306_b200 as H
        from paper_2202_01306_b200.lowering import NativePlan, ledger_rows
        from paper_2202_01306_b200.model import GPT_PRESETS, gpt_machine, gpt_profiles
        spec = GPT_PRESETS["tiny"]
        prof = gpt_profiles(spec)
        mach = gpt_machine(world, alpha_bytes=4 << 30)
        packs = ((0, 1), (2, 3))
        D = 10
        g = H.generate_task_graph(H.Configuration(2, packs, 2, packs, D, H.Mode(mode)), mach, prof)
        plan = NativePlan(g, mach, prof)
        plan.simulate()
        items = plan.items()
        mine = items[items["gpu"] == rank]
        rows = ledger_rows(mine, world)
        my_tasks = [t.index for t in g.tasks if t.device[1] == rank]
        if mode == "dp":
            sh = H.gpu_shares(D, world)
            rng = (sum(sh[:rank]), sum(sh[:rank + 1]))
        else:
            rng = (0, D)
        # U tasks in order = the all-reduce sequence (packs) on this rank
        ar_seq = [g.tasks[i].pack for i in my_tasks if g.tasks[i].type is H.TaskType.U]
        gathered = [None] * world
        dist.all_gather_object(gathered, {"rows": rows, "tasks": my_tasks, "range": rng, "ar": ar_seq,
                                          "total": ledger_rows(items, world)})
        if rank == 0:
            q.put(gathered)
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("mode", ["dp", "pp"])
def test_two_rank_plan_partition(mode):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, mode, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    a, b = out
    assert a["total"] == b["total"]                      # same global plan everywhere
    assert sorted(a["rows"] + b["rows"]) == a["total"]   # rank slices partition the ledger
    assert not set(a["tasks"]) & set(b["tasks"])
    if mode == "dp":
        assert a["range"] == (0, 5) and b["range"] == (5, 10)
        assert a["ar"] == b["ar"]                        # identical collective order
        assert any(r[3] == "sX" for r in a["rows"]) and any(r[3] == "sX" for r in b["rows"])
    else:
        assert any(r[4] == "peer2peer" for r in a["rows"] + b["rows"])

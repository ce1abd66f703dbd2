"""Harmony-DP with N=2 data-parallel ranks, one process per rank, both on one
GPU.  NCCL cannot place two ranks on one device, so the per-pack gradient sum
runs through the runtime's CUDA-IPC backend (hm_runtime_init_ipc_reduce: each
rank sums both ranks' pack gradients through the mapped peer pools, in rank
order, ordered by device-side counters) -- the same action, placement and
ordering as the NCCL all-reduce the multi-GPU path uses.

Checks (taskgraph.py:346-400: per-GPU task copies over gpu_shares):
* the union of the ranks' executed ledgers equals the planner's ledger;
* the ranks' losses sum to the oracle's single-device loss, and every rank's
  replica of W and K matches the torch-CPU oracle run on the whole minibatch
  (per-layer weight deltas, Adam m / v) -- even and uneven shares;
* both replicas hold identical bits after training (same summed gradients)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp
from conftest import collect_or_fail

pytestmark = pytest.mark.gpu


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, D, math, q, update="replicated", shm=""):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2202_01306_b200 as H
        from paper_2202_01306_b200.model import GPT_PRESETS, gpt_profiles, synthetic_batch
        from paper_2202_01306_b200.runtime import HarmonyRuntime
        spec = GPT_PRESETS["tiny"]
        prof = gpt_profiles(spec)
        mach = H.MachineModel(gpu_count=world, gpu_mem_capacity=4 << 30, pcie_bandwidth=55_000_000_000)
        packs = ((0, 1), (2, 3))
        g = H.generate_task_graph(H.Configuration(2, packs, 2, packs, D, H.Mode.DP), mach, prof)
        torch.cuda.set_device(0)
        rt = HarmonyRuntime(spec, alpha_bytes=4 << 30, device=0, math=math, dp_update=update)
        if update == "sharded":  # one host arena for all ranks (rank 0 creates and initialises it)
            stash = HarmonyRuntime.stash_bytes_for(g, prof)
            if rank == 0:
                rt.share_arenas(shm, True, stash)
                rt.init_weights(0)
            dist.barrier()
            if rank != 0:
                rt.share_arenas(shm, False, stash)
        else:
            rt.init_weights(0)  # same seed on every rank: identical replicas
        w0 = rt.w.copy()
        rt.init_ipc_reduce(world, rank)
        rt.load(g, mach, prof, rank=rank)
        blobs = [None] * world
        dist.all_gather_object(blobs, rt.ipc_export())
        for b in blobs:
            rt.ipc_import(b)
        dist.barrier()
        tok, lab = synthetic_batch(spec, D)
        lo, hi = rt.sample_range()
        losses = [rt.step(tok[lo:hi], lab[lo:hi]) for _ in range(2)]
        losses += rt.run_steps(2, tok[lo:hi], lab[lo:hi])[0]  # pipelined
        torch.cuda.synchronize()
        dist.barrier()
        out = {"rank": rank, "losses": losses, "ledger": rt.report().ledger, "w": rt.w.copy(), "k": rt.k.copy(),
               "w0": w0, "w_off": rt.w_off.copy(), "nccl_bytes": rt.counters()["nccl_bytes"],
               "rank_waits": rt.counters()["rank_waits"]}
        gathered = [None] * world
        dist.all_gather_object(gathered, out)
        if rank == 0:
            q.put({"ranks": gathered, "sim_ledger": H.simulate(g, mach, prof, dp_update=update).ledger,
                   "ref_ledger": H.simulate(g, mach, prof).ledger})
        dist.barrier()
        rt.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("D,math,update", [(8, "bf16", "replicated"), (7, "bf16", "replicated"),
                                           (8, "fp32", "replicated"), (8, "fp32", "sharded"),
                                           (7, "bf16", "sharded")])
def test_dp_two_ranks_one_gpu(D, math, update):
    """Replicated (the reference) and sharded (SURVEY 8f row 4 fast mode:
    reduce-scattered gradients, rank g updates shard g of each pack in one
    shared host arena) Harmony-DP."""
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    shm = f"hm_dp_test_{os.getpid()}_{D}_{math}"
    procs = [ctx.Process(target=_worker, args=(r, 2, port, D, math, q, update, shm)) for r in range(2)]
    for p in procs:
        p.start()
    res = collect_or_fail(q, procs, 300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    r0, r1 = sorted(res["ranks"], key=lambda x: x["rank"])
    assert sorted(r0["ledger"] + r1["ledger"]) == sorted(res["sim_ledger"])
    assert r0["nccl_bytes"] > 0
    if update == "replicated":
        # per-rank host replicas: no transfer waits on another rank's counters
        # (the NCCL path imports no peer pools, so such a wait could never be met)
        assert r0["rank_waits"] == 0 and r1["rank_waits"] == 0
    else:
        # shared arena: W swap-ins wait for every rank's shard W-out of the last
        # iteration; K and W-out rows carry one shard each, so the union of the
        # ranks' ledgers moves |K| and |W| once per pack instead of once per rank
        assert r0["rank_waits"] > 0 and r1["rank_waits"] > 0
        def vol(led, tensor, stage):
            return sum(r[6] for r in led if r[3] == tensor and r[1] == stage)
        union = r0["ledger"] + r1["ledger"]
        for tensor, stage in (("K", 0), ("K", 2), ("W", 2)):
            assert 2 * vol(union, tensor, stage) == vol(res["ref_ledger"], tensor, stage)
        assert vol(union, "W", 0) == vol(res["ref_ledger"], "W", 0)
    # both replicas: the same summed gradient, the same Adam -> the same bits
    assert np.array_equal(r0["w"].view(np.uint32), r1["w"].view(np.uint32))
    assert np.array_equal(r0["k"].view(np.uint32), r1["k"].view(np.uint32))
    from oracle.gpt_cpu import GPTOracle
    from paper_2202_01306_b200.model import GPT_PRESETS, synthetic_batch
    from test_parity_gpu import BF16_TOL, FP32_TOL, per_layer_rel
    spec = GPT_PRESETS["tiny"]
    o = GPTOracle(spec, r0["w0"], r0["w_off"])
    tok, lab = synthetic_batch(spec, D)
    ref = [o.step(tok, lab, [2] * (D // 2) + ([D % 2] if D % 2 else [])) for _ in range(4)]
    tol = FP32_TOL if math == "fp32" else BF16_TOL
    for a, b, r in zip(r0["losses"], r1["losses"], ref):
        assert abs((a + b) - r) / r < tol["loss"], (a, b, r)
    off = r0["w_off"]
    dw = per_layer_rel(r0["w"], o.w.numpy(), off, r0["w0"])
    m = per_layer_rel(r0["k"][0::2], o.m.numpy(), off)
    v = per_layer_rel(r0["k"][1::2], o.v.numpy(), off)
    print(f"DP N=2 D={D} math={math}: dW {max(dw):.2e} m {max(m):.2e} v {max(v):.2e}")
    assert max(dw) < tol["dw"] and max(m) < tol["m"] and max(v) < tol["v"]

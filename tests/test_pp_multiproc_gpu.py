"""Harmony-PP with N=2 pipeline ranks, one process per rank, both on one GPU
(CUDA IPC and stream memory operations work between processes on the same
device).  Checks: the union of the ranks' executed ledgers equals the
planner's ledger (including the peer2peer X / Y / dY rows), and loss and
weights match the torch-CPU oracle -- for step-by-step and pipelined runs,
at the tiny c1 shape and at the c4 (GPT-40B) layer shape at reduced depth
(d=8192, 64 heads of 128, seq 128, 2 steps): loss within 1e-3 at every step, per-layer
weight deltas / Adam moments within the stated tolerances
(tests/test_parity_gpu.py)."""

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


SPECS = {
    "tiny": dict(preset="tiny", lr=1e-4, alpha=4 << 30),
    # the 40B config's layer (805 M parameters, 3.2 GB of fp32 W per layer)
    # (fp32-operand parity mode: per-layer updates within 1e-3; in the bf16 mode Adam's
    # first steps turn operand rounding into sign flips of near-zero gradients)
    "wide": dict(spec=(4, 8192, 64, 128, 1024), lr=1e-5, alpha=70 << 30, steps=2, math="fp32"),
}


def _spec(name):
    from paper_2202_01306_b200.model import GPT_PRESETS, GPTSpec
    c = SPECS[name]
    return GPT_PRESETS[c["preset"]] if "preset" in c else GPTSpec(*c["spec"], causal=True, name="gpt-40b-layers")


def _worker(rank, world, port, shm, pipelined, name, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2202_01306_b200 as H
        from paper_2202_01306_b200.model import GPT_PRESETS, gpt_profiles, synthetic_batch
        from paper_2202_01306_b200.runtime import HarmonyRuntime
        spec = _spec(name)
        lr, alpha = SPECS[name]["lr"], SPECS[name]["alpha"]
        prof = gpt_profiles(spec)
        mach = H.MachineModel(gpu_count=world, gpu_mem_capacity=alpha, pcie_bandwidth=55_000_000_000)
        pf = ((0, 0), (1, 1), (2, 3))
        pb = ((0, 1), (2, 3))
        g = H.generate_task_graph(H.Configuration(4, pf, 4, pb, 8, H.Mode.PP), mach, prof)
        torch.cuda.set_device(0)
        rt = HarmonyRuntime(spec, alpha_bytes=alpha, device=0, lr=lr, math=SPECS[name].get("math", "bf16"))
        stash = HarmonyRuntime.stash_bytes_for(g, prof)
        if rank == 0:
            rt.share_arenas(shm, True, stash)
            rt.init_weights(0, device="cuda" if name != "tiny" else None)
        dist.barrier()
        if rank != 0:
            rt.share_arenas(shm, False, stash)
        w0 = rt.w.copy() if rank == 0 else None
        rt.load(g, mach, prof, rank=rank)
        blobs = [None] * world
        dist.all_gather_object(blobs, rt.ipc_export())
        for b in blobs:
            rt.ipc_import(b)
        dist.barrier()
        tok, lab = synthetic_batch(spec, 8)
        steps = SPECS[name].get("steps", 3)
        if pipelined:
            losses, _ = rt.run_steps(steps, tok, lab)
        else:
            losses = []
            for _ in range(steps):
                losses.append(rt.step(tok, lab))
        torch.cuda.synchronize()
        dist.barrier()
        rep = rt.report()
        out = {"rank": rank, "losses": losses, "ledger": rep.ledger, "p2p": rt.counters()["p2p_bytes"],
               "rank_waits": rt.counters()["rank_waits"]}
        if rank == 0:  # weights travel as files (GBs at the 40B layer shape)
            d = os.environ.get("TMPDIR", "/tmp")
            out["w_final"] = os.path.join(d, f"{shm}_w_final.npy")
            out["w0"] = os.path.join(d, f"{shm}_w0.npy")
            np.save(out["w_final"], rt.w)
            np.save(out["w0"], w0)
            del w0
        gathered = [None] * world
        dist.all_gather_object(gathered, out)
        if rank == 0:
            sim = H.simulate(g, mach, prof)
            q.put({"ranks": gathered, "sim_ledger": sim.ledger, "w_off": rt.w_off})
        dist.barrier()
        rt.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("name,pipelined", [("tiny", False), ("tiny", True), ("wide", True)])
def test_pp_two_ranks_one_gpu(name, pipelined):
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    shm = f"hm_pp_test_{os.getpid()}_{int(pipelined)}"
    port = _port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, shm, pipelined, name, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = collect_or_fail(q, procs, 900)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    r0, r1 = sorted(res["ranks"], key=lambda x: x["rank"])
    # activations and the shared host arenas order the ranks through device counters
    assert r0["rank_waits"] > 0 and r1["rank_waits"] > 0
    for key in ("w0", "w_final"):
        path = r0[key]
        r0[key] = np.load(path)
        os.unlink(path)
    assert sorted(r0["ledger"] + r1["ledger"]) == res["sim_ledger"]
    assert any(row[4] == "peer2peer" for row in res["sim_ledger"])
    # oracle
    from oracle.gpt_cpu import GPTOracle
    from paper_2202_01306_b200.model import synthetic_batch
    from test_parity_gpu import BF16_TOL, FP32_TOL, per_layer_rel
    spec = _spec(name)
    o = GPTOracle(spec, r0["w0"], res["w_off"], lr=SPECS[name]["lr"])
    tok, lab = synthetic_batch(spec, 8)
    ref = [o.step(tok, lab, [8]) for _ in range(SPECS[name].get("steps", 3))]
    # the rank running the last forward task owns the loss; the other reports 0
    losses = [max(a, b) for a, b in zip(r0["losses"], r1["losses"])]
    assert min(min(r0["losses"]), min(r1["losses"])) == 0.0
    tol = FP32_TOL if SPECS[name].get("math") == "fp32" else BF16_TOL
    for a, b in zip(losses, ref):
        assert abs(a - b) / b < tol["loss"], (losses, ref)
    dw = per_layer_rel(r0["w_final"], o.w.numpy(), res["w_off"], r0["w0"])
    print(f"PP N=2 {name}: loss {losses} vs {ref}; per-layer dW rel {['%.1e' % x for x in dw]}")
    # north_star's weight check: the weights after K steps within 1e-3 relative
    w_rel = float(np.linalg.norm(r0["w_final"] - o.w.numpy()) / np.linalg.norm(o.w.numpy()))
    assert w_rel < 1e-3, w_rel
    # the stricter per-layer update delta, at north_star's 1e-3 in the fp32-operand
    # mode too (its accumulating GEMMs sum K in chunks of <= 1024 in TMEM: the
    # 4-layer d = 8192 chain measured 5.0e-4 .. 1.3e-3 with one long chain)
    assert max(dw) < tol["dw"], dw

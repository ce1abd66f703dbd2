"""The multi-rank bench path on one GPU (HM_BENCH_SHARE_GPU=1: N ranks on
cuda:0, gloo control plane, CUDA-IPC gradient sum in place of NCCL): the
launcher spawns the ranks, the ranks' executed ledgers union to the plan,
timing is the max over ranks and rank 0 prints one JSON line with n_gpus = N.
Harmony-DP (replicated and sharded update) and Harmony-PP."""

import json
import os
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("workload,n", [("tiny-dp", 2), ("tiny-dp-shard", 2), ("tiny", 2), ("tiny-dp", 3)])
def test_bench_ranks_share_one_gpu(workload, n):
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    env = dict(os.environ, HM_BENCH_SHARE_GPU="1", NCCL_DEBUG="WARN")
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", str(n), "--workload", workload,
                        "--steps", "3", "--warmup", "3", "--no-cpu-baseline"],
                       env=env, capture_output=True, text=True, timeout=600, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]  # rank 0 only
    d = json.loads(lines[0])
    assert d["n_gpus"] == n and d["steps"] == 3
    assert d["ledger_equals_plan"] is True
    assert d["value"] > 0 and d["gpu_launches"] > 0
    assert d["config"]["parallelism"].endswith(str(n))

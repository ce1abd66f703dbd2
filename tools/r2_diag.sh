set -u
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -m pytest tests/test_kernels_gpu.py -q -x > gpurun_out/d_k.log 2>&1; tail -1 gpurun_out/d_k.log
python -m pytest tests/test_parity_gpu.py -q -s > gpurun_out/d_par.log 2>&1; grep -E "math=|passed|failed" gpurun_out/d_par.log | head -30
python tools/parity_flip_diag.py > gpurun_out/flip_kcap.jsonl 2>&1
python tools/attn_perf.py 4 1024 25 64 1 50 > gpurun_out/d_perf.jsonl 2>&1
echo done

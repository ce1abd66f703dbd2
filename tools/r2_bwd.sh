set -u
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_kernels_gpu.py -q -x -k "attn or attention" > gpurun_out/bwd_tests.log 2>&1; tail -1 gpurun_out/bwd_tests.log
timeout 1200 python -m pytest tests/test_parity_gpu.py tests/test_runtime_gpu.py -q -k "wide" > gpurun_out/bwd_par.log 2>&1; tail -1 gpurun_out/bwd_par.log
timeout 120 python tools/attn_perf.py 4 1024 64 128 1 20 > gpurun_out/bwd_perf.jsonl 2>&1
timeout 120 python tools/attn_perf.py 2 2048 64 128 1 10 >> gpurun_out/bwd_perf.jsonl 2>&1
HM_ATTN_FWD=t timeout 120 python tools/attn_perf.py 4 1024 25 64 1 20 >> gpurun_out/bwd_perf.jsonl 2>&1
echo done

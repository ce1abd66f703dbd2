set -u
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -m pytest tests/test_kernels_gpu.py tests/test_runtime_gpu.py -q -x > gpurun_out/tr_tests.log 2>&1; tail -3 gpurun_out/tr_tests.log
python tools/attn_perf.py 4 1024 25 64 1 50 > gpurun_out/tr_perf.jsonl 2>&1
python tools/attn_perf.py 16 1024 25 64 1 20 >> gpurun_out/tr_perf.jsonl 2>&1
python tools/attn_perf.py 8 512 16 64 0 20 >> gpurun_out/tr_perf.jsonl 2>&1
python tools/attn_perf.py 4 1024 64 128 1 20 >> gpurun_out/tr_perf.jsonl 2>&1
echo done

set -u
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_kernels_gpu.py -q -x -k "attn or attention" > gpurun_out/tr_tests.log 2>&1; tail -1 gpurun_out/tr_tests.log
timeout 120 python tools/attn_perf.py 4 1024 25 64 1 50 > gpurun_out/tr_perf.jsonl 2>&1
timeout 120 python tools/attn_perf.py 16 1024 25 64 1 20 >> gpurun_out/tr_perf.jsonl 2>&1
timeout 120 python tools/attn_perf.py 8 512 16 64 0 20 >> gpurun_out/tr_perf.jsonl 2>&1
timeout 900 python bench.py --workload gpt2-xl-dp-d64 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/tr_d64.json 2> gpurun_out/tr_d64.err
echo done

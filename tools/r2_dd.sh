set -u
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_kernels_gpu.py -q -x -k "attention_fwd_bwd" > gpurun_out/r2dd_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r2dd_tests.log
for shape in "4 1024 25 64 1" "8 512 16 64 0" "16 1024 25 64 1" "8 1024 25 64 1"; do
  timeout 60 python tools/attn_perf.py $shape >> gpurun_out/r2dd_attn_perf.jsonl 2>>gpurun_out/r2dd_attn_perf.err
done
HM_ATTN_TRACE=1 timeout 60 python tools/attn_perf.py 4 1024 25 64 1 1 > gpurun_out/r2dd_trace.log 2>&1
echo done

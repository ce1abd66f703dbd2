# attention backward issue order: parity, timing, phase trace
set -u
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_kernels_gpu.py -q -x -k "attention" > gpurun_out/r2o_attn_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r2o_attn_tests.log
for shape in "4 1024 25 64 1" "8 512 16 64 0" "1 1024 25 64 1" "16 1024 25 64 1"; do
  timeout 120 python tools/attn_perf.py $shape >> gpurun_out/r2o_attn_perf.jsonl 2>>gpurun_out/r2o_attn_perf.err
done
HM_ATTN_TRACE=1 timeout 120 python tools/attn_perf.py 4 1024 25 64 1 1 > gpurun_out/r2o_trace.log 2>&1
echo done

# persistent head_dim-64 forward with per-tile S buffers: parity + timing + trace
set -u
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 300 python -m pytest tests/test_kernels_gpu.py -q -x -k "attention_fwd_bwd and 64" > gpurun_out/r2w_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r2w_tests.log
for shape in "4 1024 25 64 1" "8 512 16 64 0" "1 1024 25 64 1" "16 1024 25 64 1"; do
  timeout 60 python tools/attn_perf.py $shape >> gpurun_out/r2w_attn_perf.jsonl 2>>gpurun_out/r2w_attn_perf.err
done
HM_ATTN_TRACE=1 timeout 60 python tools/attn_perf.py 4 1024 25 64 1 1 > gpurun_out/r2w_trace.log 2>&1
timeout 600 python -m pytest tests/test_kernels_gpu.py -q -k "attention" > gpurun_out/r2w_tests_all.log 2>&1
echo "rc=$?" >> gpurun_out/r2w_tests_all.log
echo done

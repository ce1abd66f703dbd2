# head_dim-128 tcgen05 attention: parity tests + timing vs the mma.sync kernels
set -u
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_kernels_gpu.py -q -x -k attention > gpurun_out/r2b_attn_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r2b_attn_tests.log
for shape in "4 1024 64 128 1" "1 1024 64 128 1" "8 512 16 128 0" "4 1024 25 64 1"; do
  timeout 120 python tools/attn_perf.py $shape >> gpurun_out/r2b_attn_perf.jsonl 2>>gpurun_out/r2b_attn_perf.err
  HM_ATTN=mma HM_ATTN_BWD=mma timeout 120 python tools/attn_perf.py $shape >> gpurun_out/r2b_attn_perf.jsonl 2>>gpurun_out/r2b_attn_perf.err
done
echo done

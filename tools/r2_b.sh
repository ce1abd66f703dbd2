# round-2 checks: head_dim-128 attention, DP (replicated + sharded) on one GPU, bench, reference arm
set -u
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_kernels_gpu.py -q -k attention > gpurun_out/r2b_attn_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r2b_attn_tests.log
for shape in "4 1024 64 128 1" "1 1024 64 128 1" "8 512 16 128 0" "4 1024 25 64 1"; do
  timeout 120 python tools/attn_perf.py $shape >> gpurun_out/r2b_attn_perf.jsonl 2>>gpurun_out/r2b_attn_perf.err
  HM_ATTN=mma HM_ATTN_BWD=mma timeout 120 python tools/attn_perf.py $shape >> gpurun_out/r2b_attn_perf.jsonl 2>>gpurun_out/r2b_attn_perf.err
done
timeout 900 python -m pytest tests/test_dp_multiproc_gpu.py tests/test_pp_multiproc_gpu.py -q > gpurun_out/r2b_mp_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r2b_mp_tests.log
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r2b_bench.json 2> gpurun_out/r2b_bench.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r2b_bench_ref.json 2> gpurun_out/r2b_bench_ref.err
echo done

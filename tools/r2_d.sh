set -u
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
(df -h /dev/shm; free -g; nproc) > gpurun_out/r2d_box.txt 2>&1
PYTHONFAULTHANDLER=1 timeout 700 python -m pytest tests/test_pp_multiproc_gpu.py -q -x -k wide -s > gpurun_out/r2d_wide.log 2>&1
echo "rc=$?" >> gpurun_out/r2d_wide.log
timeout 900 python -m pytest tests/test_profiling.py tests/test_bench_multirank_gpu.py -q > gpurun_out/r2d_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r2d_tests.log
for mode in q t; do
  HM_ATTN_FWD=$mode timeout 120 python tools/attn_perf.py 4 1024 25 64 1 >> gpurun_out/r2d_attn_perf.jsonl 2>>gpurun_out/r2d_attn_perf.err
  HM_ATTN_FWD=$mode timeout 120 python tools/attn_perf.py 8 512 16 64 0 >> gpurun_out/r2d_attn_perf.jsonl 2>>gpurun_out/r2d_attn_perf.err
done
for shape in "4 1024 64 128 1" "1 1024 64 128 1" "8 512 16 128 0"; do
  timeout 120 python tools/attn_perf.py $shape >> gpurun_out/r2d_attn_perf.jsonl 2>>gpurun_out/r2d_attn_perf.err
done
for w in resnet-1026-dp vgg-416-dp; do
  timeout 900 python bench.py --workload $w --steps 3 --warmup 3 > gpurun_out/r2d_bench_$w.json 2> gpurun_out/r2d_bench_$w.err
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_tc128 -c 2 \
  -o gpurun_out/r2d_attn128 python tools/attn_perf.py 4 1024 64 128 1 2 > gpurun_out/r2d_ncu128.log 2>&1
HM_ATTN_FWD=t timeout 600 ncu --set full --clock-control none --import-source on -k regex:fwd_kernel -c 1 \
  -o gpurun_out/r2d_attn64t python tools/attn_perf.py 4 1024 25 64 1 2 > gpurun_out/r2d_ncu64t.log 2>&1
bash tools/sanitize.sh
echo done

set -u
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python bench.py --steps 6 --warmup 3 --no-cpu-baseline > gpurun_out/bb.json 2> gpurun_out/bb.err
for e in 0 4 2 1; do
  HM_ATTN_ICVT=$e timeout 120 python tools/attn_perf.py 4 1024 25 64 1 50 >> gpurun_out/icvt_perf.jsonl 2>&1
  HM_ATTN_ICVT=$e timeout 120 python tools/attn_perf.py 16 1024 25 64 1 20 >> gpurun_out/icvt_perf.jsonl 2>&1
  HM_ATTN_ICVT=$e timeout 120 python tools/attn_perf.py 8 512 16 64 0 20 >> gpurun_out/icvt_perf.jsonl 2>&1
done
HM_ATTN_ICVT=1 timeout 600 python -m pytest tests/test_kernels_gpu.py -q -x -k "attn or attention" > gpurun_out/icvt_tests.log 2>&1; tail -1 gpurun_out/icvt_tests.log
echo done

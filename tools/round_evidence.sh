#!/bin/bash
# Run on the GPU box: tests, smoke, bench, launch list and one full ncu capture
# of the dominant kernel; everything lands in gpurun_out/ (copy to profiles/).
set -u
cd "$(dirname "$0")/.."
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/ev_tests.log 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/ev_smoke.log 2>&1
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/ev_bench.json 2> gpurun_out/ev_bench.err
timeout 300 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/ev_bench_ref.json 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 12000 --csv \
  --log-file gpurun_out/ev_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ev_ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 3000 -c 4 \
  -o gpurun_out/ev_gemm python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/ev_ncu_full.log 2>&1
echo done

# round-2 evidence on HEAD: GPU suite, smoke, bench + reference arm, attention perf, ncu launch list
set -u
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2e_box.txt 2>&1
(free -g; nproc) >> gpurun_out/r2e_box.txt 2>&1
timeout 2700 python -m pytest tests -m gpu -q --durations=40 > gpurun_out/r2e_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r2e_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2e_smoke.log 2>&1
echo "rc=$?" >> gpurun_out/r2e_smoke.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r2e_bench.json 2> gpurun_out/r2e_bench.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/r2e_bench_ref.json 2> gpurun_out/r2e_bench_ref.err
for shape in "4 1024 25 64 1" "8 512 16 64 0" "4 1024 64 128 1" "1 1024 64 128 1" "8 512 16 128 0"; do
  timeout 120 python tools/attn_perf.py $shape >> gpurun_out/r2e_attn_perf.jsonl 2>>gpurun_out/r2e_attn_perf.err
done
for mode in q t; do
  HM_ATTN_FWD=$mode timeout 120 python tools/attn_perf.py 4 1024 25 64 1 >> gpurun_out/r2e_attn_perf_fwdvar.jsonl 2>>gpurun_out/r2e_attn_perf.err
done
echo done

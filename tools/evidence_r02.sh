# round-2 evidence on HEAD: GPU suite, smoke, bench + reference arm, ncu launch list,
# ncu --set full of in-step GEMM launches, compute-bound workloads
set -u
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/fin_box.txt 2>&1
timeout 2700 python -m pytest tests -m gpu -q --durations=20 > gpurun_out/fin_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/fin_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/fin_smoke.log 2>&1
echo "rc=$?" >> gpurun_out/fin_smoke.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/fin_bench.json 2> gpurun_out/fin_bench.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/fin_bench_ref.json 2> gpurun_out/fin_bench_ref.err
for w in gpt2-xl-dp-d64 bert-large-pp; do
  timeout 900 python bench.py --workload $w --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/fin_bench_$w.json 2> gpurun_out/fin_bench_$w.err
done
for shape in "4 1024 25 64 1" "8 512 16 64 0" "16 1024 25 64 1" "4 1024 64 128 1"; do
  timeout 60 python tools/attn_perf.py $shape >> gpurun_out/fin_attn_perf.jsonl 2>>gpurun_out/fin_attn_perf.err
done
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -c 12000 --csv \
  --log-file gpurun_out/fin_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/fin_ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:gemm_kernel -s 3000 -c 4 \
  -o gpurun_out/fin_gemm python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/fin_ncu_full.log 2>&1
echo done

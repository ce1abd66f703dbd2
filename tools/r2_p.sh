# evidence on HEAD: GPU suite, smoke, default bench, reference arm, kernel timings
set -u
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/r2p_box.txt 2>&1
timeout 2700 python -m pytest tests -m gpu -q --durations=30 > gpurun_out/r2p_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r2p_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2p_smoke.log 2>&1
echo "rc=$?" >> gpurun_out/r2p_smoke.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r2p_bench.json 2> gpurun_out/r2p_bench.err
timeout 300 python tools/kernel_perf.py ln >> gpurun_out/r2p_ln_perf.jsonl 2>>gpurun_out/r2p_kp.err
for shape in "4 1024 25 64 1" "8 512 16 64 0" "4 1024 64 128 1"; do
  timeout 120 python tools/attn_perf.py $shape >> gpurun_out/r2p_attn_perf.jsonl 2>>gpurun_out/r2p_attn_perf.err
done
timeout 900 python bench.py --workload vgg-416-dp --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2p_bench_vgg.json 2> gpurun_out/r2p_bench_vgg.err
echo done

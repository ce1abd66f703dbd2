set -u
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 2700 python -m pytest tests -m gpu -q > gpurun_out/f4_tests.log 2>&1; echo "tests rc=$?" >> gpurun_out/f4_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f4_smoke.log 2>&1; echo "rc=$?" >> gpurun_out/f4_smoke.log
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/f4_bench.json 2> gpurun_out/f4_bench.err
for shape in "4 1024 25 64 1" "8 512 16 64 0" "16 1024 25 64 1" "4 1024 64 128 1"; do
  timeout 60 python tools/attn_perf.py $shape >> gpurun_out/f4_attn_perf.jsonl 2>>gpurun_out/f4_attn_perf.err
done
echo done

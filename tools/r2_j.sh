# new default head_dim-64 forward: parity (variants), ncu of fwd64 and the head_dim-64 backward, bench
set -u
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_kernels_gpu.py -q -k "attention" > gpurun_out/r2j_attn_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r2j_attn_tests.log
timeout 600 ncu --set full --clock-control none --import-source on --kernel-name-base demangled \
  -k regex:"attn_fwd64|attn_tc::bwd" -c 2 -o gpurun_out/r2j_attn64 python tools/attn_perf.py 4 1024 25 64 1 2 > gpurun_out/r2j_ncu.log 2>&1
timeout 900 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2j_bench.json 2> gpurun_out/r2j_bench.err
timeout 900 python bench.py --workload gpt2-xl-dp-d64 --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/r2j_bench_d64.json 2> gpurun_out/r2j_bench_d64.err
echo done

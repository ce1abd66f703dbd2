set -u
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_kernels_gpu.py -q -k "layernorm" > gpurun_out/r2z_ln_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r2z_ln_tests.log
timeout 300 python tools/kernel_perf.py ln >> gpurun_out/r2z_ln_perf.jsonl 2>>gpurun_out/r2z_ln.err
echo done

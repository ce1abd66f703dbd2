set -u
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_kernels_gpu.py -q -k "layernorm" > gpurun_out/r2ff_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r2ff_tests.log
echo done

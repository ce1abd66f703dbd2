set -u
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_kernels_gpu.py -q -k "attention" > gpurun_out/r2cc_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r2cc_tests.log
echo done

set -u
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_pp_multiproc_gpu.py -q -k wide --durations=5 > gpurun_out/r2c_wide.log 2>&1
echo "rc=$?" >> gpurun_out/r2c_wide.log
timeout 2400 python -m pytest tests -m gpu -q -k "not wide" --durations=30 > gpurun_out/r2c_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r2c_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2c_smoke.log 2>&1
echo done

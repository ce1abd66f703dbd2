set -u
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python -m pytest tests/test_kernels_gpu.py -q -x -k "gemm" > gpurun_out/g_tests.log 2>&1; tail -3 gpurun_out/g_tests.log
python tools/gemm_shapes.py new > gpurun_out/g_new.jsonl 2>&1
HM_GEMM_EFF192PM=0.1 python tools/gemm_shapes.py old > gpurun_out/g_old.jsonl 2>&1
echo done

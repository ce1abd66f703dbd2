# GEMM direct epilogue: parity (GEMM + conv tests) and A/B timing
set -u
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_kernels_gpu.py -q -x -k "gemm or conv" > gpurun_out/r2ee_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r2ee_tests.log
for e in tma direct; do
  if [ $e = tma ]; then export HM_GEMM_EPI=tma; else unset HM_GEMM_EPI; fi
  timeout 120 python tools/gemm_epi_ab.py 4096 6400 1600 | sed "s/^{/{\"mode\": \"$e\", /" >> gpurun_out/r2ee_epi.jsonl 2>>gpurun_out/r2ee.err
  timeout 120 python tools/gemm_epi_ab.py 4096 1600 1600 | sed "s/^{/{\"mode\": \"$e\", /" >> gpurun_out/r2ee_epi.jsonl 2>>gpurun_out/r2ee.err
  timeout 300 python tools/gemm_shapes.py $e >> gpurun_out/r2ee_shapes.jsonl 2>>gpurun_out/r2ee.err
done
unset HM_GEMM_EPI
timeout 900 python -m pytest tests/test_runtime_gpu.py -q -x -k "tiny or cnn" > gpurun_out/r2ee_rt.log 2>&1
echo "rc=$?" >> gpurun_out/r2ee_rt.log
echo done

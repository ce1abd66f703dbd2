# head_dim-64 forward (HM_ATTN_FWD=f) parity + timing; GEMM stream-K (ACC_F32) parity + A/B
set -u
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_kernels_gpu.py -q -x -k "every_variant and f" > gpurun_out/r2i_attn_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r2i_attn_tests.log
for mode in q f; do
  for shape in "4 1024 25 64 1" "8 512 16 64 0" "1 1024 25 64 1"; do
    HM_ATTN_FWD=$mode timeout 120 python tools/attn_perf.py $shape >> gpurun_out/r2i_attn_perf.jsonl 2>>gpurun_out/r2i_attn_perf.err
  done
done
timeout 900 python -m pytest tests/test_kernels_gpu.py -q -x -k "gemm" > gpurun_out/r2i_gemm_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r2i_gemm_tests.log
HM_GEMM_STREAMK=0 timeout 300 python tools/gemm_shapes.py nosk >> gpurun_out/r2i_gemm_shapes.jsonl 2>>gpurun_out/r2i_gemm.err
timeout 300 python tools/gemm_shapes.py auto >> gpurun_out/r2i_gemm_shapes.jsonl 2>>gpurun_out/r2i_gemm.err
HM_ATTN_FWD=f timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_fwd64 -c 1 \
  -o gpurun_out/r2i_fwd64 python tools/attn_perf.py 4 1024 25 64 1 2 > gpurun_out/r2i_ncu.log 2>&1
echo done

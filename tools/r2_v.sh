set -u
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
HM_ATTN_TRACE=1 timeout 120 python tools/attn_perf.py 4 1024 25 64 1 1 > gpurun_out/r2v_fwd_trace.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k regex:gemm_kernel -s 3 -c 1 \
  -o gpurun_out/r2v_gemm_gelu python tools/gemm_shapes.py ncu 1 > gpurun_out/r2v_ncu_gemm.log 2>&1
echo done

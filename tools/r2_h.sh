# head_dim-64 forward with rotating S buffers (HM_ATTN_FWD=f): parity + timing
set -u
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_kernels_gpu.py -q -x -k "every_variant and (f or q)" > gpurun_out/r2h_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r2h_tests.log
for mode in q t f; do
  for shape in "4 1024 25 64 1" "8 512 16 64 0" "1 1024 25 64 1"; do
    HM_ATTN_FWD=$mode timeout 120 python tools/attn_perf.py $shape >> gpurun_out/r2h_attn_perf.jsonl 2>>gpurun_out/r2h_attn_perf.err
  done
done
HM_ATTN_FWD=f timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_fwd64 -c 1 \
  -o gpurun_out/r2h_fwd64 python tools/attn_perf.py 4 1024 25 64 1 2 > gpurun_out/r2h_ncu.log 2>&1
timeout 900 python -m pytest tests/test_pp_multiproc_gpu.py -q -k wide -s > gpurun_out/r2h_wide.log 2>&1
echo "rc=$?" >> gpurun_out/r2h_wide.log
echo done

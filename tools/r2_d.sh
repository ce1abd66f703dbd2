# attention profiles (ncu, one fwd + one bwd of the head_dim-128 kernels and the
# head_dim-64 default / 't' forward), d64 't' vs default timing, sanitizers
set -u
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for mode in q t; do
  HM_ATTN_FWD=$mode timeout 120 python tools/attn_perf.py 4 1024 25 64 1 >> gpurun_out/r2d_attn_perf.jsonl 2>>gpurun_out/r2d_attn_perf.err
  HM_ATTN_FWD=$mode timeout 120 python tools/attn_perf.py 8 512 16 64 0 >> gpurun_out/r2d_attn_perf.jsonl 2>>gpurun_out/r2d_attn_perf.err
done
timeout 600 ncu --set full --clock-control none --import-source on -k regex:attn_tc128 -c 2 \
  -o gpurun_out/r2d_attn128 python tools/attn_perf.py 4 1024 64 128 1 2 > gpurun_out/r2d_ncu128.log 2>&1
HM_ATTN_FWD=t timeout 600 ncu --set full --clock-control none --import-source on -k regex:fwd_kernel -c 1 \
  -o gpurun_out/r2d_attn64t python tools/attn_perf.py 4 1024 25 64 1 2 > gpurun_out/r2d_ncu64t.log 2>&1
bash tools/sanitize.sh
echo done

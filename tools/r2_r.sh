set -u
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
HM_ATTN_TRACE=1 timeout 120 python tools/attn_perf.py 4 1024 25 64 1 1 > gpurun_out/r2r_trace.log 2>&1
echo done

# LayerNorm backward with wide rows in registers: parity (every variant) + graph-timed A/B
set -u
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_kernels_gpu.py -q -k "layernorm" > gpurun_out/r2n_ln_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r2n_ln_tests.log
timeout 300 python tools/kernel_perf.py ln >> gpurun_out/r2n_ln_perf.jsonl 2>>gpurun_out/r2n_ln.err
HM_LN_BWD=w timeout 300 python tools/kernel_perf.py ln >> gpurun_out/r2n_ln_perf.jsonl 2>>gpurun_out/r2n_ln.err
echo done
HM_ATTN_TRACE=1 timeout 120 python tools/attn_perf.py 4 1024 25 64 1 1 > gpurun_out/r2n_trace.log 2>&1
HM_ATTN_TRACE=1 timeout 120 python tools/attn_perf.py 8 512 16 64 0 1 >> gpurun_out/r2n_trace.log 2>&1
echo done2

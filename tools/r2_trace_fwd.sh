set -u
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
python tools/attn_perf.py 4 1024 25 64 1 50 > gpurun_out/tr_perf.jsonl 2>&1
python tools/attn_perf.py 16 1024 25 64 1 20 >> gpurun_out/tr_perf.jsonl 2>&1
HM_ATTN_TRACE=1 python tools/attn_perf.py 4 1024 25 64 1 2 > /dev/null 2> gpurun_out/tr_fwd64.log
HM_ATTN_TRACE=1 python tools/attn_perf.py 16 1024 25 64 1 2 > /dev/null 2> gpurun_out/tr_fwd64_16.log
echo done

set -u
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for e in 0 8 4 2; do
  HM_ATTN_EMU=$e timeout 120 python tools/attn_perf.py 4 1024 25 64 1 50 >> gpurun_out/emu_perf.jsonl 2>&1
  HM_ATTN_EMU=$e timeout 120 python tools/attn_perf.py 16 1024 25 64 1 20 >> gpurun_out/emu_perf.jsonl 2>&1
  HM_ATTN_EMU=$e timeout 120 python tools/attn_perf.py 8 512 16 64 0 20 >> gpurun_out/emu_perf.jsonl 2>&1
done
HM_ATTN_EMU=4 timeout 600 python -m pytest tests/test_kernels_gpu.py -q -x -k "attn or attention" > gpurun_out/emu_tests4.log 2>&1; tail -1 gpurun_out/emu_tests4.log
HM_ATTN_EMU=2 timeout 600 python -m pytest tests/test_kernels_gpu.py -q -x -k "attn or attention" > gpurun_out/emu_tests2.log 2>&1; tail -1 gpurun_out/emu_tests2.log
echo done

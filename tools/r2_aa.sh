set -u
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
HM_ATTN_EXP_EMU=1 timeout 300 python -m pytest tests/test_kernels_gpu.py -q -x -k "attention_fwd_bwd and 64" > gpurun_out/r2aa_tests.log 2>&1
echo "rc=$?" >> gpurun_out/r2aa_tests.log
for emu in 0 1; do
for shape in "4 1024 25 64 1" "8 512 16 64 0" "16 1024 25 64 1"; do
  HM_ATTN_EXP_EMU=$emu timeout 60 python tools/attn_perf.py $shape >> gpurun_out/r2aa_attn_perf.jsonl 2>>gpurun_out/r2aa_attn_perf.err
done
done
echo done

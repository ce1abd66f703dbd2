set -u
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for k in "fwd_kernel 4 1024 25 64 1" "bwd_kernel 4 1024 25 64 1"; do
  set -- $k
  timeout 600 ncu --section SpeedOfLight --section ComputeWorkloadAnalysis --section MemoryWorkloadAnalysis --section LaunchStats \
    --metrics sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed,sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active,sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__instruction_throughput.avg.pct_of_peak_sustained_active,l1tex__data_pipe_lsu_wavefronts_mem_shared.avg.pct_of_peak_sustained_elapsed \
    --clock-control none -k regex:$1 -s 2 -c 1 -o gpurun_out/ncu_attn_$1 python tools/attn_perf.py $2 $3 $4 $5 $6 2 > gpurun_out/ncu_attn_$1.log 2>&1
  echo "$1 rc=$?"
done
echo done

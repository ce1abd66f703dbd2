# ncu of the head_dim-64 attention kernels (no SASS-patching sections: the
# instrumented replay of the setmaxnreg forward hangs)
set -u
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
SECS="--section SpeedOfLight --section ComputeWorkloadAnalysis --section WarpStateStats --section SchedulerStats --section MemoryWorkloadAnalysis --section LaunchStats --section Occupancy --section InstructionStats"
timeout 300 ncu $SECS --clock-control none --kernel-name-base demangled -k regex:"attn_tc::bwd" -c 1 \
  -o gpurun_out/r2k_bwd64 python tools/attn_perf.py 4 1024 25 64 1 2 > gpurun_out/r2k_ncu_bwd.log 2>&1
timeout 300 ncu $SECS --clock-control none --kernel-name-base demangled -k regex:"attn_fwd64" -c 1 \
  -o gpurun_out/r2k_fwd64 python tools/attn_perf.py 4 1024 25 64 1 2 > gpurun_out/r2k_ncu_fwd.log 2>&1
timeout 300 ncu --set full --import-source on --clock-control none --kernel-name-base demangled -k regex:"attn_tc::bwd" -c 1 \
  -o gpurun_out/r2k_bwd64_full python tools/attn_perf.py 4 1024 25 64 1 2 > gpurun_out/r2k_ncu_bwd_full.log 2>&1
echo done

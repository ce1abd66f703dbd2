set -u
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 60 tools/probes/mma_probe > gpurun_out/r2s_mma_probe.jsonl 2>&1
echo done

set -u
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 2400 python tools/parity_c2_full.py > gpurun_out/r2gg_c2_full.log 2>&1
echo "rc=$?" >> gpurun_out/r2gg_c2_full.log
echo done

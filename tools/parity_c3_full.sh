set -u
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 3000 python tools/parity_c3_full.py > gpurun_out/r2hh_c3_full.log 2>&1
echo "rc=$?" >> gpurun_out/r2hh_c3_full.log
echo done

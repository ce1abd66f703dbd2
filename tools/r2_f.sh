# XU-pipe probe, the 40B-layer PP test, compute-sanitizer evidence
set -u
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 60 tools/probes/xu_probe > gpurun_out/r2f_xu_probe.jsonl 2>&1
timeout 900 python -m pytest tests/test_pp_multiproc_gpu.py -q -k wide > gpurun_out/r2f_wide.log 2>&1
echo "rc=$?" >> gpurun_out/r2f_wide.log
bash tools/sanitize.sh
echo done

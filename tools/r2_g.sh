set -u
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
timeout 60 tools/probes/tmem_probe > gpurun_out/r2g_tmem_probe.jsonl 2>&1
timeout 900 python -m pytest tests/test_pp_multiproc_gpu.py -q -k wide -s > gpurun_out/r2g_wide.log 2>&1
echo "rc=$?" >> gpurun_out/r2g_wide.log
timeout 1500 /usr/local/cuda/bin/compute-sanitizer --tool racecheck --print-limit 50 --error-exitcode 9 \
  python -c "import __graft_entry__ as g; g.smoke(parts=('bf16', 'cnn'))" > gpurun_out/san_smoke_racecheck.log 2>&1
echo "exit=$?" >> gpurun_out/san_smoke_racecheck.log
echo done

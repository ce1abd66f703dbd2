# compute-sanitizer evidence: memcheck / racecheck / synccheck on smoke() and
# memcheck on the 2-process Harmony-PP test (all target processes).  Logs go to
# gpurun_out/ (copied into profiles/ by hand).
set -u
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck synccheck; do
  timeout 900 $CS --tool $tool --print-limit 50 --error-exitcode 9 \
    python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/san_smoke_$tool.log 2>&1
  echo "exit=$?" >> gpurun_out/san_smoke_$tool.log
done
# racecheck (shared-memory hazards) is slow on the three-plane fp32-operand GEMMs: the
# bf16-operand GPT iteration and the CNN iteration
timeout 1500 $CS --tool racecheck --print-limit 50 --error-exitcode 9 \
  python -c "import __graft_entry__ as g; g.smoke(parts=('bf16', 'cnn'))" > gpurun_out/san_smoke_racecheck.log 2>&1
echo "exit=$?" >> gpurun_out/san_smoke_racecheck.log
timeout 900 $CS --tool memcheck --target-processes all --print-limit 50 --error-exitcode 9 \
  python -m pytest tests/test_pp_multiproc_gpu.py -q -k "tiny and False" > gpurun_out/san_pp_memcheck.log 2>&1
echo "exit=$?" >> gpurun_out/san_pp_memcheck.log
timeout 900 $CS --tool memcheck --target-processes all --print-limit 50 --error-exitcode 9 \
  python -m pytest tests/test_dp_multiproc_gpu.py -q -k "8-fp32-sharded" > gpurun_out/san_dp_memcheck.log 2>&1
echo "exit=$?" >> gpurun_out/san_dp_memcheck.log
echo done

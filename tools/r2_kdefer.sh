set -u
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
for n in 2 0 4 1 3; do
  HM_K_DEFER=$n timeout 600 python bench.py --steps 6 --warmup 3 --no-cpu-baseline > gpurun_out/kd_$n.json 2> gpurun_out/kd_$n.err
  python - "$n" <<'PY'
import json,sys
n=sys.argv[1]
try:
    d=json.loads(open(f"gpurun_out/kd_{n}.json").read().strip().splitlines()[-1])
    print(json.dumps({"k_defer": int(n), "value": d["value"], "e2e": d["e2e"]["value"], "ms": d["ms_per_step"],
      "frac": d["step_roofline"]["frac"], "t_phase": d["step_roofline"].get("t_phase_ms"), "frac_phase": d["step_roofline"].get("frac_phase"),
      "busy": d["stream_busy_frac"], "pcie": d["step_roofline"]["pcie_gbs"], "clk": d["clocks"]["sm_mhz"], "ledger": d["ledger_equals_plan"]}))
except Exception as e:
    print("k_defer", n, "failed", e)
PY
done >> gpurun_out/kd_summary.jsonl
echo done

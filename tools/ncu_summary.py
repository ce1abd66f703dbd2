"""Summarise an `ncu --set full` capture of GEMM launches into the JSON that
bench.py reports as roofline.traffic (run here, no GPU needed):

    python tools/ncu_summary.py profiles/r01_gemm_pair_full.ncu-rep > profiles/r01_gemm_ncu_summary.json
"""
import csv, io, json, os, subprocess, sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, units, data = rows[0], rows[1], rows[2:]
col = {n: h.index(n) for n in h}
scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
launches = []
for r in data:
    rd = float(r[col["dram__bytes_read.sum"]]) * scale[units[col["dram__bytes_read.sum"]]]
    wr = float(r[col["dram__bytes_write.sum"]]) * scale[units[col["dram__bytes_write.sum"]]]
    launches.append({"kernel": r[col["Kernel Name"]].split("(")[0], "us": float(r[col["gpu__time_duration.sum"]]),
                     "dram_read": rd, "dram_write": wr,
                     "tensor_active_pct": float(r[col["sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed"]])})
n = len(launches)
print(json.dumps({"source": os.path.basename(rep), "launches": n,
                  "dram_bytes_per_launch_mean": round(sum(l["dram_read"] + l["dram_write"] for l in launches) / n),
                  "per_launch": launches}, indent=1))

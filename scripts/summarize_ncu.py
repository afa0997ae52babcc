"""Summarise an ncu report (details page minus rule text, plus key raw metrics) for profiles/."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
det = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
out = []
for row in csv.reader(io.StringIO(det)):
    if len(row) < 4 or row[-4] in ("OPT", "INF", "WRN") or row[-4] == "Rule Type":
        continue
    if row[-4].startswith(("Section", "Rule")):
        continue
    out.append("%-40s %-45s %12s %s" % (row[-4][:40], row[-3][:45], row[-1], row[-2]))
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
keys = ["Kernel Name", "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active"]
h, u, v = rows[0], rows[1], rows[2]
print("== raw ==")
for k in keys:
    if k in h:
        i = h.index(k)
        print("%-65s %s %s" % (k, v[i], u[i]))
print("== details ==")
print("\n".join(out))

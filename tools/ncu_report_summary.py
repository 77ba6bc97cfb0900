"""One-screen summary of an ncu --set full report (one kernel): headline
metrics, warp-stall shares and the SASS instruction mix.
usage: python tools/ncu_report_summary.py <report.ncu-rep> "<title line>" """
import collections
import csv
import io
import subprocess
import sys

rep, title = sys.argv[1], sys.argv[2] if len(sys.argv) > 2 else ""
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h, u, v = rows[0], rows[1], rows[2]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__inst_executed.sum"]
print("# " + title)
for k in want:
    if k in h:
        i = h.index(k)
        print(f"{k:60s} {v[i]} {u[i]}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
srows = list(csv.reader(io.StringIO(src)))
sh = srows[1]
data = srows[2:]
ie, sc = sh.index("Instructions Executed"), sh.index("Source")
cols = [c for c in sh if c.startswith("stall_") and "Not Issued" not in c]
idx = [sh.index(c) for c in cols]
tot = collections.Counter()
mix = collections.Counter()
for r in data:
    for c, i in zip(cols, idx):
        tot[c[6:]] += int(r[i] or 0)
    op = r[sc].split()
    if op:
        o = op[1] if op[0].startswith("@") and len(op) > 1 else op[0]
        mix[o.split(".")[0]] += int(r[ie] or 0)
T = sum(tot.values())
M = sum(mix.values())
print("warp stall samples (share): " + ", ".join(f"{k}={100 * n / T:.1f}%" for k, n in tot.most_common(8)))
print("instruction mix: " + ", ".join(f"{k}={100 * n / M:.1f}%" for k, n in mix.most_common(10)))

"""Key metrics per kernel from an ncu report (details page)."""
import csv
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[0]
ki, mi, vi, ui, ii = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "Metric Unit", "ID"))
want = ["Duration", "DRAM Throughput", "Memory Throughput", "Achieved Occupancy", "Theoretical Occupancy",
        "Registers Per Thread", "Compute (SM) Throughput", "L2 Hit Rate", "Executed Ipc Active", "Issue Slots Busy",
        "Warp Cycles Per Issued Instruction", "Dynamic Shared Memory Per Block", "Grid Size", "Block Size"]
seen = set()
for r in rows[1:]:
    if r[mi] in want and (r[ii], r[mi]) not in seen:
        seen.add((r[ii], r[mi]))
        print(r[ii], r[ki].split("(")[0][-28:], "|", r[mi], r[vi], r[ui])
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rr = list(csv.reader(raw.splitlines()))
hh = rr[0]
cols = [i for i, n in enumerate(hh) if n in ("dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__time_duration.sum",
                                               "lts__t_sector_hit_rate.pct", "Kernel Name")]
for r in rr[2:]:
    print([(hh[i], r[i]) for i in cols])

"""Issue-slot roofline of the rasterizer kernels (and the scatter-add for comparison) from an
ncu --set full report: warp instructions per frame, issue-active fraction, FP64 pipe use,
and the top stall reasons per issued instruction.  python tools/ncu_issue_roofline.py REP FRAMES"""
import csv
import subprocess
import sys

rep, frames = sys.argv[1], int(sys.argv[2])
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
h = rows[0]
col = {n: i for i, n in enumerate(h)}
stalls = [n for n in h if n.startswith("smsp__average_warps_issue_stalled_") and n.endswith("_per_issue_active.ratio")]
for r in rows[2:]:
    name = r[col["Kernel Name"]].split("(")[0].split("::")[-1]
    g = lambda k: float(r[col[k]].replace(",", "")) if k in col and r[col[k]] not in ("", "n/a") else float("nan")  # noqa
    inst = g("smsp__inst_executed.sum") if "smsp__inst_executed.sum" in col else g("sm__inst_executed.sum")
    dur_ms = g("gpu__time_duration.sum")
    top = sorted(((g(s), s[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]) for s in stalls),
                 reverse=True)[:5]
    print("%-22s %7.3f ms  %6.2f M warp-inst/frame  issue-active %5.1f %%  fp64 pipe %5.1f %%  IPC %4.2f" % (
        name, dur_ms, inst / frames / 1e6, g("sm__issue_active.avg.pct_of_peak_sustained_elapsed"),
        g("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
        g("sm__inst_executed.avg.per_cycle_active")))
    print("    stalls per issued instruction: " + ", ".join("%s %.2f" % (n, v) for v, n in top))

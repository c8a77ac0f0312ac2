"""Selected raw metrics of the first kernel in each ncu report, one block per report:
    python tools/ncu_metrics.py LABEL=REP [LABEL=REP ...]  (split at the last "=")"""
import csv
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "duration"),
    ("sm__inst_executed.sum", "warp instructions"),
    ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue active %"),
    ("l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_elapsed", "L1 data pipe (LSU wavefronts) % of peak"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "shared-memory wavefronts"),
    ("lts__throughput.avg.pct_of_peak_sustained_elapsed", "L2 throughput % of peak"),
    ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput % of peak"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "FP64 pipe %"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
    ("launch__registers_per_thread", "registers"),
]


def main(args):
    for arg in args:
        label, rep = arg.rsplit("=", 1)
        out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(out.splitlines()))
        h, u, v = rows[0], rows[1], rows[2]
        name = v[h.index("Kernel Name")]
        print("%s: %s" % (label, name))
        for m, what in METRICS:
            if m in h:
                i = h.index(m)
                print("    %-42s %s %s" % (what, v[i], u[i]))


if __name__ == "__main__":
    main(sys.argv[1:])

"""Per-CUDA-line summary of `ncu -i REP --page source --csv --print-source=cuda,sass`:
stall samples and executed warp instructions per source line (sorted by samples)."""
import csv
import sys

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
rows = list(csv.reader(open(path, encoding="utf-8", errors="replace")))
out = []
tot_s = tot_i = 0
for r in rows:
    if len(r) < 8 or not r[0] or r[2] != "-":
        continue
    try:
        s, ins = int(r[4]), int(r[7])
    except ValueError:
        continue
    out.append((s, ins, r[0], r[1]))
    tot_s += s
    tot_i += ins
tot_s = tot_s or 1
tot_i = tot_i or 1
print("total samples %d, warp instructions %d" % (tot_s, tot_i))
for s, ins, ln, src in sorted(out, key=lambda o: -o[0])[:top]:
    print("%5.1f%% smp %5.1f%% ins  L%-4s %s" % (100.0 * s / tot_s, 100.0 * ins / tot_i, ln, src.strip()[:100]))

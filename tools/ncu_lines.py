"""Summarize an `ncu --page source --csv --print-source=cuda,sass` dump per CUDA source line."""
import csv
import sys

path = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
rows = list(csv.reader(open(path)))
out = []
hdr = None
fname = None
for r in rows:
    if r and r[0] == "Line No":
        hdr = r
        continue
    if r and r[0] in ("File Name", "File Path"):
        fname = r[1]
        continue
    if hdr is None or not r or not r[0] or r[0] == "" or len(r) < len(hdr):
        continue
    if r[2] != "-":  # sass rows carry an address
        continue
    try:
        samples = int(r[hdr.index("Warp Stall Sampling (All Samples)")])
    except ValueError:
        continue
    stalls = {}
    for i, h in enumerate(hdr):
        if h.startswith("stall_") and "Not Issued" not in h:
            try:
                v = int(r[i])
            except ValueError:
                continue
            if v:
                stalls[h[6:]] = v
    best = sorted(stalls.items(), key=lambda kv: -kv[1])[:3]
    out.append((samples, r[0], r[1][:90], best, r[hdr.index("Instructions Executed")]))
tot = sum(o[0] for o in out) or 1
for s, ln, src, best, ins in sorted(out, key=lambda o: -o[0])[:top]:
    print("%5.1f%% L%-4s inst=%-9s %-90s %s" % (100.0 * s / tot, ln, ins, src.strip(), best))

"""Top SASS instructions by warp-stall samples from `ncu --page source --csv --print-source sass`."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]
i_src, i_s = hdr.index("Source"), hdr.index("Warp Stall Sampling (All Samples)")
data = [(float(r[i_s] or 0), r[hdr.index("Address")], r[i_src]) for r in rows[2:] if len(r) > i_s]
tot = sum(d[0] for d in data)
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
for s, a, src in sorted(data, reverse=True)[:n]:
    print(f"{s / tot * 100:5.1f}% {a} {src[:110]}")

"""Per-instruction stall breakdown from `ncu --page source --csv --print-source sass` output.

usage: python tools/sass_stalls.py <csv> [top_n] [reason]
Prints the top instructions by the given stall column (default: all samples)
with the previous 3 instructions for context.
"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1], errors="replace")))
hdr = rows[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
col = sys.argv[3] if len(sys.argv) > 3 else "Warp Stall Sampling (All Samples)"
i_src, i_s = hdr.index("Source"), hdr.index(col)
body = [r for r in rows[2:] if len(r) > i_s]
tot_all = sum(float(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0) for r in body)
reasons = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
print("total samples", tot_all)
print("by reason:", {h: int(sum(float(r[hdr.index(h)] or 0) for r in body)) for h in reasons})
order = sorted(range(len(body)), key=lambda j: -float(body[j][i_s] or 0))[:n]
for j in order:
    r = body[j]
    top = sorted(((float(r[hdr.index(h)] or 0), h[6:]) for h in reasons), reverse=True)[:2]
    print(f"{float(r[i_s] or 0) / tot_all * 100:5.1f}% [{j:5d}] {r[i_src][:70]:70s} {top}")

"""Per-role view of an `ncu --page source --csv --print-source sass` capture: for each kernel,
the MMA-issuer region (the SASS span holding the UTCHMMA instructions) against the whole
kernel -- instructions executed, stall samples, and the issuer's share of one warp's samples
(near 1 or above: the issuer is busy the whole kernel, i.e. it paces the pipeline).

usage: python tools/warp_roles.py <src.csv> <warps per CTA> [steps]
"""
import csv
import sys

path, nwarps = sys.argv[1], int(sys.argv[2])
steps = float(sys.argv[3]) if len(sys.argv) > 3 else None
rows = list(csv.reader(open(path, errors="replace")))
kernels, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = {"name": r[1], "rows": []}
        kernels.append(cur)
    elif r and r[0] == "Address":
        cur["hdr"] = r
    elif cur is not None and "hdr" in cur and len(r) >= len(cur["hdr"]) - 1:
        cur["rows"].append(r)
for k in kernels:
    h, body = k["hdr"], k["rows"]
    i_src, i_s, i_e = h.index("Source"), h.index("Warp Stall Sampling (All Samples)"), h.index("Instructions Executed")
    f = lambda r, i: float(r[i] or 0)  # noqa: E731
    mma = [j for j, r in enumerate(body) if "UTCHMMA" in r[i_src] and f(r, i_e) > 0]
    if not mma:
        continue
    lo, hi = mma[0] - 40, mma[-1] + 20
    tot_s = sum(f(r, i_s) for r in body)
    iss_s = sum(f(body[j], i_s) for j in range(lo, hi))
    iss_e = sum(f(body[j], i_e) for j in range(lo, hi))
    reasons = [x for x in h if x.startswith("stall_") and "Not Issued" not in x]
    agg = sorted(((sum(f(body[j], h.index(x)) for j in range(lo, hi)), x[6:]) for x in reasons), reverse=True)[:5]
    print(k["name"][:90])
    print(f"  issuer span SASS [{lo}, {hi}): {iss_e:.0f} warp instructions" +
          (f" = {iss_e / steps:.0f} per step" if steps else ""))
    print(f"  issuer samples {iss_s:.0f} = {iss_s / (tot_s / nwarps):.2f} x one warp's average; top stalls "
          + ", ".join(f"{n} {v:.0f}" for v, n in agg))

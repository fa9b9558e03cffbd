"""Median epilogue phase lengths (clk) per query-tile slot from an RSA_BF_TRACE dump (steps of heads >= 1)."""
import sys

import numpy as np

nw = int(sys.argv[2]) if len(sys.argv) > 2 else 12
nq = 4
a = np.fromfile(sys.argv[1], dtype=np.int64).reshape(nw, 4096)
ev = a[2][a[2] != 0]
e, t = (ev >> 48).tolist(), (ev & ((1 << 48) - 1)).tolist()
steps, cur = [], {}
for ee, tt in zip(e, t):
    if ee == 20 and cur:
        steps.append(cur)
        cur = {}
    cur[ee] = tt
steps.append(cur)
names = [("kv", 20, 21), ("dPw", 21, 22), ("dS", 22, 23), ("pread", 23, 24), ("st", 24, 25)]
rows = {q: [] for q in range(nq)}
for i in range(16, len(steps) - 1):
    s, n = steps[i], steps[i + 1]
    if 25 not in s:
        continue
    rows[i % nq].append([s[b] - s[a_] for _, a_, b in names] + [n[20] - s[25], n[20] - s[20]])
for q in range(nq):
    m = np.median(np.array(rows[q]), axis=0)
    print(f"qt{q}: " + " ".join(f"{nm}={v:.0f}" for nm, v in zip([x[0] for x in names] + ["tail", "step"], m)))
tot = steps[-1][20] - steps[16][20]
print("avg step", tot / (len(steps) - 17))

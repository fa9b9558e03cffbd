"""Decode an RSA_BF_TRACE dump: per-step epilogue phase durations and MMA issue gaps (clk)."""
import sys

import numpy as np

a = np.fromfile(sys.argv[1], dtype=np.int64).reshape(10, 4096)


def events(w):
    ev = a[w][a[w] != 0]
    return ev >> 48, ev & ((1 << 48) - 1)


e, t = events(2)
steps = []
cur = {}
for ee, tt in zip(e.tolist(), t.tolist()):
    if ee == 20 and cur:
        steps.append(cur)
        cur = {}
    cur[ee] = tt
steps.append(cur)
print("epilogue warp 2: step, start, kv-readout(20->21 incl P wait), dP wait, dS compute, p_read wait, dS store, step len")
prev = None
for i, s in enumerate(steps):
    if 25 not in s:
        continue
    ln = (s[20] - prev) if prev is not None else 0
    prev = s[20]
    print(f"{i:3d} {s[20]:8d} {s[21]-s[20]:6d} {s[22]-s[21]:6d} {s[23]-s[22]:6d} {s[24]-s[23]:6d} {s[25]-s[24]:6d} {ln:6d}")
e1, t1 = events(1)
e0, t0 = events(0)
print("producer P-issue times:", t0[e0 == 1][:40].tolist())
print("mma:", list(zip(e1[:60].tolist(), t1[:60].tolist())))

"""Per-unit timeline of fwd_factored (CTA 0, RSA_FF_TRACE) at the bench shape (B64 Z12 L512,
panel mode): for each unit of epilogue warp 2 (group 0), the clocks from unit start (event 1)
to each step's S-ready (3), to O~ ready (7) and to the unit's end (21).

usage: python tools/ff_units.py
"""
import os
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2105_13120_b200 import engine  # noqa: E402

dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(0)
q, k, v = (torch.randn((1, 64, 12, 512, 64), generator=g, device=dev).to(torch.bfloat16) for _ in range(3))
for _ in range(3):
    engine.forward(q, k, v, path="fused")
os.environ["RSA_FF_TRACE"] = "/tmp/ff_trace.bin"
engine.forward(q, k, v, path="fused")
torch.cuda.synchronize()
a = np.fromfile("/tmp/ff_trace.bin", dtype=np.int64).reshape(19, 4096)
for w in (2, 10):
    x = a[w][a[w] != 0]
    e, t = (x >> 48).tolist(), (x & ((1 << 48) - 1)).tolist()
    units, cur = [], []
    for ee, tt in zip(e, t):
        if ee == 1 and cur:
            units.append(cur)
            cur = []
        cur.append((ee, tt))
    units.append(cur)
    print(f"warp {w}: {len(units)} units")
    for u in units[:12]:
        t0 = u[0][1]
        s = [tt - t0 for ee, tt in u if ee == 3]
        o7 = [tt - t0 for ee, tt in u if ee == 7]
        e21 = [tt - t0 for ee, tt in u if ee == 21]
        print(f"  start {t0:8d}  S-ready {s}  O-ready {o7}  end {e21}")

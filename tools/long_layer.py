"""Per-kernel times of one long-sequence RSA layer (B=4, Z=12, A=64, N=1), fwd + bwd, vs the
6-byte-per-panel-element HBM bound (panel written once, read by the two backward kernels)."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2105_13120_b200 import engine  # noqa: E402

B, Z, A = 4, 12, 64
dev = torch.device("cuda", 0)
for L in [int(x) for x in (sys.argv[1:] or ["2048", "4096", "8192"])]:
    g = torch.Generator(device=dev).manual_seed(0)
    q, k, v, dO = (torch.randn((1, B, Z, L, A), generator=g, device=dev).to(torch.bfloat16) for _ in range(4))
    tm = engine.KernelTimer()
    for it in range(4):
        if it == 1:
            tm.reset()
        out, panel, rs, flag = engine.forward(q, k, v, path="auto", timer=tm)
        engine.backward(q, k, v, panel, dO, outputs=out, rowscale=rs, path="auto", timer=tm)
        del panel
    tot = tm.totals()
    pe = B * Z * L * L
    bound_us = 6 * pe / 6540e9 * 1e6
    s = sum(ms for _, ms in tot.values()) / 3 * 1e3
    print(f"L={L}: layer {s:.0f} us, 6-B panel bound {bound_us:.0f} us ({bound_us / s:.0%}); " +
          ", ".join(f"{k} {ms / n * 1e3:.0f} us x{n // 3}" for k, (n, ms) in tot.items()), flush=True)

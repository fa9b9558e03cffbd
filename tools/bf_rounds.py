"""rsa_bwd_fused time against the number of heads (one CTA per head, 148 SMs): whole rounds
(a multiple of 148 heads) against the bench shape's 768 heads = 5 rounds + a 28-head tail.

usage: python tools/bf_rounds.py
"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2105_13120_b200 import engine  # noqa: E402

dev = torch.device("cuda", 0)
L, A = 512, 64
for (b, z) in [(37, 4), (74, 4), (37, 12), (64, 12), (74, 12), (61, 12), (62, 12)]:
    g = torch.Generator(device=dev).manual_seed(0)
    q, k, v, dO = (torch.randn((1, b, z, L, A), generator=g, device=dev).to(torch.bfloat16) for _ in range(4))
    out, panel, rs, flag = engine.forward(q, k, v, path="fused")
    ts = []
    for it in range(8):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        tm = engine.KernelTimer()
        engine.backward(q, k, v, panel, dO, outputs=out, rowscale=rs, path="fused", timer=tm)
        if it >= 3:
            ts.append(tm.totals()["bwd_fused"][1] * 1e3 / tm.totals()["bwd_fused"][0])
    ts.sort()
    heads = b * z
    print(f"heads {heads:4d} = {heads / 148:.2f} rounds: bwd_fused {ts[len(ts) // 2]:.1f} us, "
          f"{ts[len(ts) // 2] / -(-heads // 148):.1f} us per round", flush=True)

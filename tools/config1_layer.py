"""Config 1's layer (B4 Z12 L512, 4 logical ranks, panel mode, single-pass backward) run a few
times without a graph: the driver for an ncu launch list of its kernels.

usage: python tools/config1_layer.py [iters] [mode]
"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
sys.path.insert(0, str(Path(__file__).resolve().parent))
from configs import layer_closure  # noqa: E402

iters = int(sys.argv[1]) if len(sys.argv) > 1 else 3
mode = sys.argv[2] if len(sys.argv) > 2 else "panel"
dev = torch.device("cuda", 0)
gen = torch.Generator(device=dev).manual_seed(512)
q, k, v, g = (torch.randn((4, 4, 12, 128, 64), generator=gen, device=dev).to(torch.bfloat16) for _ in range(4))
step = layer_closure(q, k, v, g, mode, single_pass=True if mode == "panel" else None)
for _ in range(iters):
    step()
torch.cuda.synchronize()
print("done")

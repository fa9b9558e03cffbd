"""One BERT-base RSA layer (B=64, L=512, Z=12, A=64, N=1) fwd+bwd, repeated.

Profiling driver for ncu: every fused kernel launches once per iteration.
"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2105_13120_b200 import engine  # noqa: E402

B, Z, L, A = 64, 12, 512, 64
iters = int(sys.argv[1]) if len(sys.argv) > 1 else 3
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(0)
q, k, v, dO = (torch.randn((1, B, Z, L, A), generator=g, device=dev).to(torch.bfloat16) for _ in range(4))
for _ in range(iters):
    out, panel, rowscale, flag = engine.forward(q, k, v, path="fused")
    engine.backward(q, k, v, panel, dO, outputs=out, rowscale=rowscale, path="fused")
torch.cuda.synchronize()
print("done")

"""ncu driver: one long-L panel-mode RSA layer (B=4, Z=12, A=64, L from argv, N=1) fwd + two-kernel bwd."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2105_13120_b200 import engine  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(0)
q, k, v, dO = (torch.randn((1, 4, 12, L, 64), generator=g, device=dev).to(torch.bfloat16) for _ in range(4))
for _ in range(2):
    out, panel, rs, flag = engine.forward(q, k, v, path="fused")
    engine.backward(q, k, v, panel, dO, outputs=out, rowscale=rs, path="fused", single_pass=False)
torch.cuda.synchronize()
print("done")

"""ncu driver: one stream-mode RSA layer (B=4, Z=12, A=64, L from argv, N=1) fwd+bwd, repeated."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2105_13120_b200 import engine  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 2
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(0)
q, k, v, dO = (torch.randn((1, 4, 12, L, 64), generator=g, device=dev).to(torch.bfloat16) for _ in range(4))
for _ in range(iters):
    sf = engine.forward_stream(q, k, v)
    engine.backward_stream(q, k, v, dO, sf.out, sf.rowscale, sf.rowmax)
torch.cuda.synchronize()
print("done")

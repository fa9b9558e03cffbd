"""ncu driver: config 5's Linformer forward + backward through the public API (B4 Z12 A64
L114688 Kp256, 8 logical ranks), once warm, once profiled.

usage: ncu ... python tools/prof_linformer.py"""
import math
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2105_13120_b200 import AttentionConfig, SparseAttentionConfig  # noqa: E402
from paper_2105_13120_b200.sparse_attention import (sparse_ring_attention_backward,  # noqa: E402
                                                    sparse_ring_attention_forward)
from paper_2105_13120_b200.weights import SparseWeights  # noqa: E402

n, b, z, L, a, kdim = 8, 4, 12, 114688, 64, 256
c = L // n
dev = torch.device("cuda", 0)
gen = torch.Generator(device=dev).manual_seed(0)
base = AttentionConfig(batch_size=b, seq_len=L, hidden_size=z * a, num_heads=z, head_size=a, num_devices=n)
cfg = SparseAttentionConfig(base=base, proj_dim=kdim)
q, k, v, g = (torch.randn((b, z, L, a), generator=gen, device=dev).to(torch.bfloat16) for _ in range(4))
ch = lambda t: [t[:, :, d * c:(d + 1) * c] for d in range(n)]  # noqa: E731
w = SparseWeights(*((torch.randn((kdim, L), generator=gen, device=dev) / math.sqrt(L)).to(torch.bfloat16)
                    for _ in range(2)))
for _ in range(2):
    sparse_ring_attention_forward(ch(q), ch(k), ch(v), w, cfg)
    sparse_ring_attention_backward(ch(q), ch(k), ch(v), w, cfg, ch(g))
torch.cuda.synchronize()
print("done")

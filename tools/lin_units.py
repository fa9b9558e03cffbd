"""Unit timeline of the Linformer low-rank attention (config 5: B4 Z12 L=114688 over 8 ranks,
K' = 256 keys, stream-mode fwd_factored): CTA 0's epilogue warp 2, clocks from each unit's
start to its S-ready events and the deferred O readout.

usage: python tools/lin_units.py
"""
import os
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2105_13120_b200 import AttentionConfig, SparseAttentionConfig, SparseWeights  # noqa: E402
from paper_2105_13120_b200.sparse_attention import sparse_ring_attention_forward  # noqa: E402

dev = torch.device("cuda", 0)
n, b, z, seq, a, kp = 8, 4, 12, 114688, 64, 256
gen = torch.Generator(device=dev).manual_seed(5)
seqs = [torch.randn((b, z, seq, a), generator=gen, device=dev).to(torch.bfloat16) for _ in range(3)]
sc = [list(t.chunk(n, dim=2)) for t in seqs]
s = seq ** -0.5
w = SparseWeights((torch.randn((kp, seq), generator=gen, device=dev) * s).to(torch.bfloat16),
                  (torch.randn((kp, seq), generator=gen, device=dev) * s).to(torch.bfloat16))
cfg = SparseAttentionConfig(base=AttentionConfig(batch_size=b, seq_len=seq, hidden_size=z * a, num_heads=z,
                                                 head_size=a, num_devices=n), proj_dim=kp)
for _ in range(3):
    sparse_ring_attention_forward(sc[0], sc[1], sc[2], w, cfg)
os.environ["RSA_FF_TRACE"] = "/tmp/ff_trace.bin"
sparse_ring_attention_forward(sc[0], sc[1], sc[2], w, cfg)
torch.cuda.synchronize()
tr = np.fromfile("/tmp/ff_trace.bin", dtype=np.int64).reshape(19, 4096)
for wi in (2,):
    x = tr[wi][tr[wi] != 0]
    e, t = (x >> 48).tolist(), (x & ((1 << 48) - 1)).tolist()
    units, cur = [], []
    for ee, tt in zip(e, t):
        if ee == 1 and cur:
            units.append(cur)
            cur = []
        cur.append((ee, tt))
    units.append(cur)
    starts = [u[0][1] for u in units]
    print(f"warp {wi}: {len(units)} units traced; median unit length {np.median(np.diff(starts)):.0f} clk")
    for u in units[5:15]:
        t0 = u[0][1]
        print("  ", [(ee, tt - t0) for ee, tt in u])

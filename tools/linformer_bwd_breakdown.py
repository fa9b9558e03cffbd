"""Breakdown of the Linformer backward (sparse_ring_attention_backward) at config 5:
B4 Z12 A64 L114688 Kp256, 8 logical ranks -- each stage timed with CUDA events.

usage: python tools/linformer_bwd_breakdown.py"""
import math
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2105_13120_b200 import engine, sparse_attention as sa  # noqa: E402
from paper_2105_13120_b200 import tensor_ops as ops  # noqa: E402

n, b, z, L, a, kdim = 8, 4, 12, 114688, 64, 256
c = L // n
dev = torch.device("cuda", 0)
gen = torch.Generator(device=dev).manual_seed(0)
q, k, v, g = (torch.randn((n, b, z, c, a), generator=gen, device=dev).to(torch.bfloat16) for _ in range(4))
e, f = ((torch.randn((kdim, L), generator=gen, device=dev) / math.sqrt(L)).to(torch.bfloat16) for _ in range(2))


def timed(fn, reps=5):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        out = fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps, out


ms, (kl, vl) = timed(lambda: sa._project(q, k, v, e, f, kdim))
print(f"project            {ms:.3f} ms", flush=True)
ms, res = timed(lambda: sa._low_rank_stream(q, kl, vl))
print(f"low-rank forward   {ms:.3f} ms", flush=True)
tm = engine.KernelTimer()
ms, (dq, dkl, dvl) = timed(lambda: engine.backward_stream(q, kl.unsqueeze(0), vl.unsqueeze(0), g, res.out, res.rowscale,
                                                          res.rowmax, dkv_f32=True, timer=tm))
print(f"attention backward {ms:.3f} ms  {dict((k_, round(v_[1] / v_[0], 3)) for k_, v_ in tm.totals().items())}",
      flush=True)
dkl16, dvl16 = dkl[0].to(torch.bfloat16), dvl[0].to(torch.bfloat16)
dk, dv = torch.empty_like(q), torch.empty_like(q)
ge = torch.empty((kdim, L), dtype=torch.float32, device=dev)
dk_flat = dkl16.permute(2, 0, 1, 3).reshape(kdim, b * z * a)


def proj_grads():
    for d in range(n):
        cols = slice(d * c, (d + 1) * c)
        ops.matmul(e[:, cols].transpose(0, 1), dkl16, out=dk[d])
        ops.matmul(e[:, cols].transpose(0, 1), dvl16, out=dv[d])
        ops.matmul(dk_flat, k[d].transpose(-1, -2).reshape(b * z * a, c), out=ge[:, cols])
        ops.matmul(dk_flat, v[d].transpose(-1, -2).reshape(b * z * a, c), out=ge[:, cols])


ms, _ = timed(proj_grads)
print(f"projection grads   {ms:.3f} ms (32 GEMMs)", flush=True)
ms, _ = timed(lambda: [ops.matmul(e[:, slice(d * c, (d + 1) * c)].transpose(0, 1), dkl16, out=dk[d]) for d in range(n)])
print(f"  dK = E_d^T dK'   {ms:.3f} ms (8 GEMMs)", flush=True)
ms, _ = timed(lambda: [ops.matmul(dk_flat, k[d].transpose(-1, -2).reshape(b * z * a, c),
                                  out=ge[:, slice(d * c, (d + 1) * c)]) for d in range(n)])
print(f"  dE = dK' K_d^T   {ms:.3f} ms (8 GEMMs)", flush=True)

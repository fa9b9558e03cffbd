"""Experiment driver: the stream backward's one-pass kernel against the two-kernel form at one
length (per-launch time and relative difference).

usage: [RSA_FS_DBG=<bits>] python tools/fs_exp.py [L]"""
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2105_13120_b200 import engine  # noqa: E402

L = int(sys.argv[1]) if len(sys.argv) > 1 else 8192
B, Z, A = 4, 12, 64
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(0)
q, k, v, dO = (torch.randn((1, B, Z, L, A), generator=g, device=dev).to(torch.bfloat16) for _ in range(4))
sf = engine.forward_stream(q, k, v)
dvec, gsc = engine.ops.rowdot_scale(dO, sf.out, sf.rowscale)
grads = (torch.empty_like(q), torch.empty_like(k), torch.empty_like(v))
acc = torch.empty(q.shape, dtype=torch.float32, device=dev)
ref = engine.stream_backward_kernels(q, k, v, gsc, sf.rowmax, dvec, tuple(torch.empty_like(x) for x in grads),
                                     fused=False)
for fused in (True, False):
    for _ in range(2):
        engine.stream_backward_kernels(q, k, v, gsc, sf.rowmax, dvec, grads, fused=fused, dq_acc=acc)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        engine.stream_backward_kernels(q, k, v, gsc, sf.rowmax, dvec, grads, fused=fused, dq_acc=acc)
    e1.record()
    torch.cuda.synchronize()
    err = [float((x.double() - y.double()).norm() / y.double().norm()) for x, y in zip(grads, ref)]
    print(f"L={L} dbg={os.environ.get('RSA_FS_DBG', '0')} fused={fused}: "
          f"{e0.elapsed_time(e1) / 5 * 1e3:.1f} us, rel diff vs two-kernel {['%.1e' % x for x in err]}", flush=True)

"""Experiment: the single-pass backward's last partial round of heads -- rsa_bwd_fused over the
first b_main batches and rsa_bwd_panel_fused over the rest, each timed as a replayed CUDA graph
(host launch cost excluded).  B64 Z12 L512 (the bench shape)."""
import ctypes
import sys

import torch

sys.path.insert(0, '.')
from paper_2105_13120_b200 import engine  # noqa: E402
from paper_2105_13120_b200._native import BF16, lib  # noqa: E402

dev = torch.device('cuda', 0)
g = torch.Generator(device=dev).manual_seed(0)
n, B, Z, c, A = 1, 64, 12, 512, 64
q, k, v, dO = (torch.randn((n, B, Z, c, A), generator=g, device=dev).to(torch.bfloat16) for _ in range(4))
out, panel, rs, flag = engine.forward(q, k, v, path='fused')
dvec, gsc = engine.ops.rowdot_scale(dO, out, rs)
dq, dk, dv = (torch.empty_like(q) for _ in range(3))
acc = torch.zeros((n, B, Z, c, A), dtype=torch.float32, device=dev)
L = lib()
V = engine._view


def graphed(fn, reps=10):
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        fn(s.cuda_stream)
    torch.cuda.current_stream().wait_stream(s)
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        fn(torch.cuda.current_stream().cuda_stream)
    for _ in range(3):
        gr.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        gr.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


def main(b0, b1):
    gm = engine._geom(n, b1 - b0, Z, c, A, c, 0, n)
    sl = lambda t: t[:, b0:b1]  # noqa: E731
    return lambda st: L.rsa_bwd_fused(ctypes.byref(gm), *(V(sl(t)) for t in (q, k, v, gsc, panel)),
                                      sl(dvec).data_ptr(), engine.NULL_VIEW, 0, V(sl(dq)), V(sl(dk)), V(sl(dv)), BF16, 0, st)


def tail(b0, b1, accum=0, cast=True):
    gt = engine._geom(n, b1 - b0, Z, c, A, c, 0, n)
    sl = lambda t: t[:, b0:b1]  # noqa: E731
    return lambda st: L.rsa_bwd_panel_fused(ctypes.byref(gt), *(V(sl(t)) for t in (q, k, v, gsc, panel)),
                                            sl(dvec).data_ptr(), V(sl(dk)), V(sl(dv)), BF16, 0, acc.data_ptr(), accum,
                                            V(sl(dq)) if cast else engine.NULL_VIEW, st)


print('all 64 batches rsa_bwd_fused', round(graphed(main(0, 64)), 1), flush=True)
for bm in (62, 61, 60):
    t_main = graphed(main(0, bm))
    t_tail = graphed(tail(bm, B))
    t_tail_k = graphed(tail(bm, B, accum=1, cast=False))
    both = graphed(lambda st: (main(0, bm)(st), tail(bm, B)(st)))
    print(f'b_main {bm}: main {t_main:.1f}  tail {t_tail:.1f} (kernel only {t_tail_k:.1f})  both {both:.1f} us',
          flush=True)

"""A/B of rsa_fwd_factored / rsa_bwd_fused between two builds of librsa_b200.so at the bench
shape (B64 Z12 L512, 12 layers): python tools/ab_fwd.py <libA.so> <libB.so>"""
import ctypes
import sys

import torch

sys.path.insert(0, ".")
from paper_2105_13120_b200 import engine  # noqa: E402
from paper_2105_13120_b200 import tensor_ops as ops  # noqa: E402


def run(path, reps=20):
    L = ctypes.CDLL(path)
    dev = torch.device("cuda", 0)
    gen = torch.Generator(device=dev).manual_seed(1)
    B, Z, S, A = 64, 12, 512, 64
    lay = []
    for _ in range(12):
        q, k, v, g = (torch.randn((1, B, Z, S, A), generator=gen, device=dev).to(torch.bfloat16) for _ in range(4))
        lay.append(dict(q=q, k=k, v=v, g=g, o=torch.empty_like(q), p=torch.empty((1, B, Z, S, S), dtype=torch.bfloat16,
                        device=dev), r=torch.empty((1, B, Z, S), device=dev), dq=torch.empty_like(q),
                        dk=torch.empty_like(q), dv=torch.empty_like(q)))
    flag = torch.zeros(1, dtype=torch.int32, device=dev)
    dvec = torch.empty((1, B, Z, S), device=dev)
    gs = torch.empty_like(lay[0]["q"])
    gm = engine._geom(1, B, Z, S, A, S, 0, 1)
    st = torch.cuda.current_stream().cuda_stream
    V = engine._view

    def fwd():
        for ly in lay:
            L.rsa_fwd_factored(ctypes.byref(gm), V(ly["q"]), V(ly["k"]), V(ly["v"]), V(ly["p"]), V(ly["o"]),
                               ctypes.c_void_p(ly["r"].data_ptr()), ctypes.c_void_p(flag.data_ptr()), ctypes.c_void_p(st))

    def bwd():
        for ly in lay:
            L.rsa_bwd_fused(ctypes.byref(gm), V(ly["q"]), V(ly["k"]), V(ly["v"]), V(gs), V(ly["p"]),
                            ctypes.c_void_p(dvec.data_ptr()), engine.NULL_VIEW, 0, V(ly["dq"]), V(ly["dk"]), V(ly["dv"]),
                            1, 0, ctypes.c_void_p(st))

    fwd()
    ops.rowdot_scale(lay[0]["g"], lay[0]["o"], lay[0]["r"], out=dvec, a_scaled=gs)
    res = {}
    for name, fn in (("fwd", fwd), ("bwd", bwd)):
        fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        res[name] = e0.elapsed_time(e1) / reps / 12 * 1e3
    return res


if __name__ == "__main__":
    for rnd in range(3):
        for p in sys.argv[1:]:
            print(rnd, p, {k: round(v, 2) for k, v in run(p).items()}, flush=True)

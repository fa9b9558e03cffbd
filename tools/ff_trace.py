"""Stream-forward timeline (CTA 0) from an RSA_FF_TRACE dump: per-step event offsets (clk).

usage: python tools/ff_trace.py run L      (on the GPU: writes /tmp/ff_trace.bin)
       python tools/ff_trace.py show FILE  (decodes: median per-step phase lengths per group)
Events (fwd_factored.cu FF_TRACE): 3 S ready, 40/41 chunk 0/1 in registers, 4 exps done,
5 P~ slot free, 6 P~ stored; warp 1: 10+g S issued; warp 18: 12+g P~V issued.
"""
import os
import sys
from pathlib import Path

import numpy as np

NW = 19


def show(path):
    a = np.fromfile(path, dtype=np.int64).reshape(NW, 4096)

    def ev(w):
        x = a[w][a[w] != 0]
        return (x >> 48).tolist(), (x & ((1 << 48) - 1)).tolist()

    for w in (2, 10):  # one epilogue warp of each group
        e, t = ev(w)
        steps, cur = [], {}
        for ee, tt in zip(e, t):
            if ee == 3 and cur:
                steps.append(cur)
                cur = {}
            cur[ee] = tt
        steps.append(cur)
        rows = []
        for i in range(2, len(steps) - 1):
            s, n = steps[i], steps[i + 1]
            if not all(k in s for k in (3, 40, 41, 4, 5, 6)) or 3 not in n:
                continue
            rows.append([s[40] - s[3], s[41] - s[40], s[4] - s[41], s[5] - s[4], s[6] - s[5], n[3] - s[6], n[3] - s[3]])
        m = np.median(np.array(rows), axis=0)
        print(f"warp {w}: steps {len(rows)} " + " ".join(f"{k}={v:.0f}" for k, v in
              zip(["ld0", "ld1+exp0", "exp1", "p_wait", "store", "s_wait", "step"], m)))
    for w, base in ((1, 10), (18, 12)):
        e, t = ev(w)
        for gi in (0, 1):
            ts = np.array([tt for ee, tt in zip(e, t) if ee == base + gi])
            d = np.diff(ts)
            print(f"warp {w} ev {base + gi}: n={len(ts)} median gap {np.median(d):.0f}")
    e, t = ev(2)
    ts = [tt for ee, tt in zip(e, t) if ee == 3]
    print("group-0 step (overall):", (ts[-1] - ts[0]) / (len(ts) - 1))
    # one mid-run window of absolute event times: epilogue warps 2 (group 0), 10 (group 1), MMA warps
    t0 = ts[len(ts) // 2]
    win = []
    for w in (0, 1, 2, 10, 18):
        e, t = ev(w)
        win += [(tt - t0, w, ee) for ee, tt in zip(e, t) if 0 <= tt - t0 < 7000]
    for tt, w, ee in sorted(win):
        print(f"  {tt:6d} w{w:<2d} ev{ee}")


def run(L):
    import torch
    sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
    from paper_2105_13120_b200 import engine
    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev).manual_seed(0)
    q, k, v = (torch.randn((1, 4, 12, L, 64), generator=g, device=dev).to(torch.bfloat16) for _ in range(3))
    for _ in range(2):
        engine.forward_stream(q, k, v)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        engine.forward_stream(q, k, v)
    e1.record()
    torch.cuda.synchronize()
    print(f"fwd_stream L={L}: {e0.elapsed_time(e1) / 10 * 1e3:.1f} us", flush=True)
    os.environ["RSA_FF_TRACE"] = "/tmp/ff_trace.bin"
    engine.forward_stream(q, k, v)
    torch.cuda.synchronize()
    del os.environ["RSA_FF_TRACE"]
    show("/tmp/ff_trace.bin")


if __name__ == "__main__":
    if sys.argv[1] == "run":
        run(int(sys.argv[2]) if len(sys.argv) > 2 else 4096)
    else:
        show(sys.argv[2])

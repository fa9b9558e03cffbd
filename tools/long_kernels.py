"""Per-kernel times of one long-sequence RSA layer, panel and stream mode, against each
kernel's own bound: HBM bytes (panel traffic) or tensor flops (stream recompute).

usage: python tools/long_kernels.py [L ...]        (B=4, Z=12, A=64, every origin resident)
"""
import json
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2105_13120_b200 import engine  # noqa: E402

B, Z, A = 4, 12, 64
HBM, TC = 6539.9e9, 1383.5e12
dev = torch.device("cuda", 0)


def run(L, n=1):
    c = L // n
    g = torch.Generator(device=dev).manual_seed(0)
    q, k, v, dO = (torch.randn((n, B, Z, c, A), generator=g, device=dev).to(torch.bfloat16) for _ in range(4))
    pe = B * Z * L * L
    res = {"seq_len": L, "ranks": n}
    for mode in ("panel", "panel_2k", "stream", "stream_2k"):
        os.environ["RSA_B200_DETERMINISTIC"] = "1" if mode == "panel_2k" else "0"
        tm = engine.KernelTimer()
        for it in range(3):
            if it == 1:
                tm.reset()
            if mode.startswith("panel"):
                out, panel, rs, flag = engine.forward(q, k, v, path="fused", timer=tm)
                engine.backward(q, k, v, panel, dO, outputs=out, rowscale=rs, path="fused", timer=tm,
                                single_pass=False)
                del panel
            else:
                with tm("fwd_stream"):
                    sf = engine.forward_stream(q, k, v)
                engine.backward_stream(q, k, v, dO, sf.out, sf.rowscale, sf.rowmax, timer=tm,
                                       fused=mode == "stream")
        tot = tm.totals()
        ker = {}
        for name, (cnt, ms) in tot.items():
            us = ms / cnt * 1e3
            ker[name] = {"us": round(us, 1)}
            if name in ("fwd_factored", "bwd_dkdv", "bwd_dq", "bwd_panel_fused"):  # 2 bytes per panel element
                ker[name]["hbm_frac"] = round(2 * pe / HBM * 1e6 / us, 3)
            if name in ("fwd_stream", "bwd_kv_stream", "bwd_q_stream", "fwd_factored", "bwd_stream_fused"):
                prods = {"fwd_stream": 2, "fwd_factored": 2, "bwd_kv_stream": 4, "bwd_q_stream": 3,
                         "bwd_stream_fused": 5}[name]
                ker[name]["tc_frac_incl_recompute"] = round(prods * 2 * pe * A / TC * 1e6 / us, 3)
        res[mode] = {"layer_us": round(sum(v["us"] for v in ker.values()), 1), "kernels": ker}
        torch.cuda.empty_cache()
    return res


if __name__ == "__main__":
    out = [run(int(x)) for x in (sys.argv[1:] or ["2048", "8192"])]
    for r in out:
        print(json.dumps(r), flush=True)

"""Sequence-length sweep and max trainable sequence length on one B200 (BASELINE config 3).

BERT-base attention stack (Z=12, A=64), batch B=4 (config 3's fixed batch), 12 layers
forward then backward with every layer's saved panel resident, as in a training step.
For each L: tokens/s of the stack (device-resident synthetic inputs, CUDA events).  The
max L is the largest multiple of 1024 whose working set fits in HBM (checked by running
it), found by bisection between the largest measured L and an analytic upper bound.

usage: python tools/seq_sweep.py [--layers 12] [--batch 4] [--out gpurun_out/seq_sweep.json]
"""
import argparse
import json
import math
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2105_13120_b200 import engine  # noqa: E402

Z, A = 12, 64


def run(L, B, layers, steps, dev):
    """One fwd+bwd stack at sequence length L; returns ms per step (raises on OOM)."""
    gen = torch.Generator(device=dev).manual_seed(L)
    shp = (1, B, Z, L, A)
    q, k, v, g = (torch.randn(shp, generator=gen, device=dev).to(torch.bfloat16) for _ in range(4))
    saved = []
    flag = torch.zeros(1, dtype=torch.int32, device=dev)
    panels = [torch.empty((1, B, Z, L, L), dtype=torch.bfloat16, device=dev) for _ in range(layers)]
    scales = [torch.empty((1, B, Z, L), dtype=torch.float32, device=dev) for _ in range(layers)]
    outs = [torch.empty(shp, dtype=torch.bfloat16, device=dev) for _ in range(layers)]
    grads = tuple(torch.empty(shp, dtype=torch.bfloat16, device=dev) for _ in range(3))
    dvec = torch.empty((1, B, Z, L), dtype=torch.float32, device=dev)
    gs = torch.empty(shp, dtype=torch.bfloat16, device=dev)

    def step():
        for i in range(layers):  # (shared q/k/v across layers: memory goes to the saved panels)
            engine.forward(q, k, v, path="fused", flag=flag, out=outs[i], panel=panels[i], rowscale=scales[i])
        for i in reversed(range(layers)):
            engine.backward(q, k, v, panels[i], g, outputs=outs[i], rowscale=scales[i], path="fused", grads=grads,
                            dvec=dvec, grad_scaled=gs)

    step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        step()
    e1.record()
    torch.cuda.synchronize()
    if int(flag.item()):
        raise RuntimeError(f"flag {int(flag.item())} at L={L}")
    del saved
    return e0.elapsed_time(e1) / steps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=12)
    ap.add_argument("--batch", type=int, default=4)
    ap.add_argument("--lengths", default="2048,4096,8192")
    ap.add_argument("--out", default="gpurun_out/seq_sweep.json")
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    free, total = torch.cuda.mem_get_info(dev)
    rows = []
    for L in [int(x) for x in args.lengths.split(",")]:
        ms = run(L, args.batch, args.layers, 2, dev)
        rows.append({"seq_len": L, "ms_per_step": ms, "tokens_per_s": args.batch * L / (ms / 1e3)})
        print(json.dumps(rows[-1]), flush=True)
        torch.cuda.empty_cache()
    # bytes per L^2 of the saved panels (bf16) plus the transient row vectors: the bound
    per_l2 = args.layers * args.batch * Z * 2
    hi = int(math.sqrt(total / per_l2)) // 1024 * 1024 + 1024
    lo = max(r["seq_len"] for r in rows)
    best = None
    while hi - lo > 1024:
        mid = (lo + hi) // 2 // 1024 * 1024
        try:
            t0 = time.time()
            ms = run(mid, args.batch, args.layers, 1, dev)
            best = {"seq_len": mid, "ms_per_step": ms, "tokens_per_s": args.batch * mid / (ms / 1e3)}
            print("fits", json.dumps(best), f"({time.time() - t0:.1f} s)", flush=True)
            lo = mid
        except torch.OutOfMemoryError:
            print("OOM at", mid, flush=True)
            hi = mid
        torch.cuda.empty_cache()
    res = {"workload": f"BERT-base attention stack, {args.layers} layers fwd+bwd, B={args.batch}, Z={Z}, A={A}, "
                       "every layer's factored panel saved (training step), N=1 (whole sequence on one GPU)",
           "hbm_total_bytes": total, "sweep": rows, "max_seq_len": best or {"seq_len": lo}}
    Path(args.out).parent.mkdir(parents=True, exist_ok=True)
    Path(args.out).write_text(json.dumps(res, indent=1))
    print(json.dumps(res["max_seq_len"]))


if __name__ == "__main__":
    main()

"""Panel vs stream mode on one B200: BERT-base attention stack (Z=12, A=64, B=4 -- BASELINE
config 3's fixed batch), 12 layers forward then backward as in a training step, every
layer's activations saved (q, k, v, O, and the panel or the two row statistics).

* sweep: ms/step, tokens/s and peak HBM for both modes at each L (device-resident inputs);
* max L: the panel mode's largest L is bounded by the L^2 panels (bisection, as
  tools/seq_sweep.py); the stream mode's saved state is linear in L, so its bound is the
  per-token bytes measured here.  The stream max is then PROVEN by allocating all 12
  layers' saved state at that L and running one full layer fwd+bwd there (a whole
  12-layer step at ~0.5M tokens is minutes of O(L^2) compute).

usage: python tools/stream_sweep.py [--lengths 2048,4096,8192,16384] [--out gpurun_out/stream_sweep.json]
"""
import argparse
import json
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2105_13120_b200 import engine  # noqa: E402

Z, A = 12, 64


def layer_state(L, B, layers, mode, dev, gen):
    shp = (1, B, Z, L, A)
    st = []
    for _ in range(layers):
        d = {x: torch.randn(shp, generator=gen, device=dev).to(torch.bfloat16) for x in ("q", "k", "v")}
        d["o"] = torch.empty(shp, dtype=torch.bfloat16, device=dev)
        d["r"] = torch.empty((1, B, Z, L), dtype=torch.float32, device=dev)
        if mode == "panel":
            d["p"] = torch.empty((1, B, Z, L, L), dtype=torch.bfloat16, device=dev)
        else:
            d["m"] = torch.empty((1, B, Z, L), dtype=torch.float32, device=dev)
        st.append(d)
    return st


def run(L, B, layers, mode, steps, dev, run_layers=None):
    """ms per step of `run_layers` (default all) layers fwd+bwd with `layers` layers' state resident."""
    torch.cuda.reset_peak_memory_stats(dev)
    gen = torch.Generator(device=dev).manual_seed(L)
    shp = (1, B, Z, L, A)
    st = layer_state(L, B, layers, mode, dev, gen)
    g = torch.randn(shp, generator=gen, device=dev).to(torch.bfloat16)
    grads = tuple(torch.empty(shp, dtype=torch.bfloat16, device=dev) for _ in range(3))
    dvec = torch.empty((1, B, Z, L), dtype=torch.float32, device=dev)
    gs = torch.empty(shp, dtype=torch.bfloat16, device=dev)
    flag = torch.zeros(1, dtype=torch.int32, device=dev)
    act = st[: run_layers or layers]

    def step():
        for d in act:
            if mode == "panel":
                engine.forward(d["q"], d["k"], d["v"], path="fused", flag=flag, out=d["o"], panel=d["p"],
                               rowscale=d["r"])
            else:
                engine.forward_stream(d["q"], d["k"], d["v"], flag=flag, out=d["o"], rowscale=d["r"], rowmax=d["m"])
        for d in reversed(act):
            if mode == "panel":
                engine.backward(d["q"], d["k"], d["v"], d["p"], g, outputs=d["o"], rowscale=d["r"], path="fused",
                                grads=grads, dvec=dvec, grad_scaled=gs)
            else:
                engine.backward_stream(d["q"], d["k"], d["v"], g, d["o"], d["r"], d["m"], grads=grads, dvec=dvec,
                                       grad_scaled=gs)

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
    peak = torch.cuda.max_memory_allocated(dev)
    del st
    return e0.elapsed_time(e1) / steps, peak


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--layers", type=int, default=12)
    ap.add_argument("--batch", type=int, default=4)
    ap.add_argument("--lengths", default="2048,4096,8192,16384")
    ap.add_argument("--prove-max", type=int, default=1)
    ap.add_argument("--out", default="gpurun_out/stream_sweep.json")
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    free, total = torch.cuda.mem_get_info(dev)
    rows = []
    B = args.batch
    for L in [int(x) for x in args.lengths.split(",")]:
        row = {"seq_len": L}
        for mode in ("panel", "stream"):
            try:
                ms, peak = run(L, B, args.layers, mode, 2, dev)
                row[mode] = {"ms_per_step": ms, "tokens_per_s": B * L / (ms / 1e3), "peak_bytes": peak}
            except torch.OutOfMemoryError:
                row[mode] = "OOM"
            torch.cuda.empty_cache()
        rows.append(row)
        print(json.dumps(row), flush=True)
    # stream-mode bytes per token from the two largest measured points (linear in L)
    pts = [(r["seq_len"], r["stream"]["peak_bytes"]) for r in rows if isinstance(r["stream"], dict)]
    (l0, p0), (l1, p1) = pts[-2], pts[-1]
    per_token = (p1 - p0) / (l1 - l0)
    budget = free * 0.97
    l_max = int((budget - (p1 - per_token * l1)) / per_token) // 4096 * 4096
    res = {"workload": f"BERT-base attention stack, {args.layers} layers fwd+bwd, B={B}, Z={Z}, A={A}, every "
                       "layer's q, k, v, O and panel (panel mode) or row statistics (stream mode) saved, N=1",
           "hbm_total_bytes": total, "hbm_free_bytes": free, "sweep": rows,
           "stream_bytes_per_token": per_token, "stream_max_seq_len_estimate": l_max}
    if args.prove_max:
        t0 = time.time()
        try:
            ms, peak = run(l_max, B, args.layers, "stream", 1, dev, run_layers=1)
            res["stream_max_proof"] = {"seq_len": l_max, "layers_resident": args.layers, "layers_run": 1,
                                       "ms_one_layer_fwd_bwd": ms, "peak_bytes": peak,
                                       "est_ms_12_layer_step": ms * args.layers, "wall_s": time.time() - t0}
        except torch.OutOfMemoryError as exc:
            res["stream_max_proof"] = {"seq_len": l_max, "oom": str(exc)[:200]}
        print(json.dumps(res.get("stream_max_proof")), flush=True)
    Path(args.out).parent.mkdir(parents=True, exist_ok=True)
    Path(args.out).write_text(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()

"""BERT encoder training step on one B200 through EncoderLayer.

L encoder layers (MHA by ring self-attention + GELU MLP, residuals; no layer norm -- the
reference has none) forward then backward with saved activations, synthetic bf16
inputs and output gradient, random weights at the reference's scales.  Reports tokens/s
and the share of the step spent in the RSA kernels (timed on their own, same shapes).

usage: python tools/bert_step.py [--model base|large] [--batch 64] [--seq 512] [--ranks 1]
"""
import argparse
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2105_13120_b200 import AttentionConfig, engine  # noqa: E402
from paper_2105_13120_b200.encoder import EncoderLayer, EncoderWeights  # noqa: E402

MODELS = {"base": (12, 768, 12), "large": (24, 1024, 16)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--model", default="base", choices=sorted(MODELS))
    ap.add_argument("--batch", type=int, default=64)
    ap.add_argument("--seq", type=int, default=512)
    ap.add_argument("--ranks", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    layers_n, h, z = MODELS[args.model]
    n, b, seq = args.ranks, args.batch, args.seq
    cfg = AttentionConfig(batch_size=b, seq_len=seq, hidden_size=h, num_heads=z, head_size=h // z, num_devices=n)
    dev = torch.device("cuda", 0)
    gen = torch.Generator(device=dev).manual_seed(0)
    rs = (2 * layers_n) ** -0.5  # residual-branch scaling: no layer norm in the reference
    layers = [EncoderLayer(cfg, EncoderWeights.random(cfg, dev, gen, residual_scale=rs)) for _ in range(layers_n)]
    x0 = torch.randn((n, b, seq // n, h), generator=gen, device=dev).to(torch.bfloat16)
    gy = torch.randn((n, b, seq // n, h), generator=gen, device=dev).to(torch.bfloat16)

    def step():
        x = x0
        for ly in layers:
            x = ly.forward(x, check=False)
        g = gy
        for ly in reversed(layers):
            g, _ = ly.backward(g)
        return x

    for _ in range(2):
        step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        step()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    flags = [int(ly.flag.item()) for ly in layers]
    if any(flags):
        raise RuntimeError(f"layer status flags {flags} (1: non-finite score, 2: factored-panel fallback needed)")
    # the RSA kernels alone at this layer's shapes
    c = seq // n
    q, k, v, d = (torch.randn((n, b, z, c, h // z), generator=gen, device=dev).to(torch.bfloat16) for _ in range(4))

    def rsa():
        f = engine.forward(q, k, v, path="auto")
        engine.backward(q, k, v, f.panel, d, outputs=f.out, rowscale=f.rowscale, path="auto")

    for _ in range(2):
        rsa()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(args.steps):
        rsa()
    e1.record()
    torch.cuda.synchronize()
    rsa_ms = e0.elapsed_time(e1) / args.steps * layers_n
    res = {"model": f"BERT-{args.model} encoder ({layers_n} layers, H={h}, Z={z})", "batch": b, "seq_len": seq,
           "ring_ranks": n, "ms_per_step": ms, "tokens_per_s": b * seq / (ms / 1e3),
           "rsa_ms_per_step": rsa_ms, "rsa_share": rsa_ms / ms,
           "note": "training step = every layer fwd then bwd with saved activations; synthetic data, random init"}
    print(json.dumps(res), flush=True)
    if args.out:
        Path(args.out).write_text(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()

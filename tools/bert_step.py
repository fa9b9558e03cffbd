"""BERT encoder training step on one B200 through EncoderLayer.

L encoder layers (MHA by ring self-attention + GELU MLP, residuals; no layer norm -- the
reference has none) forward then backward with saved activations, synthetic bf16
inputs and output gradient, random weights at the reference's scales.  Reports tokens/s
and the share of the step spent in the RSA kernels (timed on their own, same shapes).

usage: python tools/bert_step.py [--model base|large] [--batch 64] [--seq 512] [--ranks 1] [--mlm]

--mlm times the whole masked-LM model step instead (paper_2105_13120_b200.bert.BertMLM):
token + position embeddings, the encoder stack, the tied-weight MLM head over the 15%
masked positions, mean cross-entropy, and every gradient -- the paper's BERT training step
 on synthetic token ids.
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
    ap.add_argument("--mlm", action="store_true")
    ap.add_argument("--vocab", type=int, default=30522)
    args = ap.parse_args()
    if args.mlm:
        return mlm(args)
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


def mlm(args):
    from paper_2105_13120_b200.bert import BertMLM

    layers_n, h, z = MODELS[args.model]
    n, b, seq = args.ranks, args.batch, args.seq
    cfg = AttentionConfig(batch_size=b, seq_len=seq, hidden_size=h, num_heads=z, head_size=h // z, num_devices=n)
    dev = torch.device("cuda", 0)
    gen = torch.Generator(device=dev).manual_seed(0)
    model = BertMLM(cfg, layers_n, vocab=args.vocab, device=dev, generator=gen)
    ids = torch.randint(1000, args.vocab, (n, b, seq // n), generator=gen, device=dev, dtype=torch.int32)
    rows = ids.numel()
    n_mask = max(1, int(0.15 * rows))
    mask_rows = torch.randperm(rows, generator=gen, device=dev)[:n_mask].sort().values
    targets = ids.view(-1)[mask_rows].clone()
    ids.view(-1)[mask_rows] = 103  # [MASK]
    for _ in range(2):
        loss, _ = model.step(ids, mask_rows, targets)
    torch.cuda.synchronize()
    losses = []
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        loss, grads = model.step(ids, mask_rows, targets)
        losses.append(loss)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / args.steps
    lv = [float(x) for x in losses]
    res = {"model": f"BERT-{args.model} masked LM ({layers_n} layers, H={h}, Z={z}, vocab {args.vocab})", "batch": b,
           "seq_len": seq, "ring_ranks": n, "masked_tokens": n_mask, "ms_per_step": ms,
           "tokens_per_s": b * seq / (ms / 1e3), "loss": lv[-1], "loss_finite": all(x == x and abs(x) < 1e4 for x in lv),
           "note": "whole training step: embeddings, encoder (RSA + MLP), MLM head on masked rows, cross-entropy, "
                   "every gradient; synthetic ids, random init (no optimizer update)"}
    print(json.dumps(res), flush=True)
    if args.out:
        Path(args.out).write_text(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()

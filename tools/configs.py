"""One-GPU measurements of BASELINE.json's configs (besides bench.py's headline config 2).

  config 1  single RSA layer fwd+bwd, H=768 Z=12 L=512 B=4, sequence over 4 logical ranks
  config 4  BERT-large attention (Z=16, A=64) single layer fwd+bwd at L=16384, B=4, the
            sequence over 8 logical ranks (the per-box work of the paper's 8-GPU run)
  config 5  Linformer sequence-parallel fwd+bwd at L=114688 (8 x 14336), B=4, Z=12, Kp=256,
            8 logical ranks

Device-resident synthetic inputs, CUDA events, median of `--iters` after warm-up.
(Config 3's sweep and max length: tools/seq_sweep.py.)
usage: python tools/configs.py [--out gpurun_out/configs.json]
"""
import argparse
import json
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2105_13120_b200 import AttentionConfig, SparseAttentionConfig, SparseWeights, engine  # noqa: E402
from paper_2105_13120_b200.sparse_attention import (sparse_ring_attention_backward,  # noqa: E402
                                                    sparse_ring_attention_forward)


def timed(fn, iters, warmup=2):
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(iters):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return statistics.median(ts)


def layer_closure(q, k, v, g, mode, single_pass=None):
    """One RSA layer fwd+bwd on preallocated buffers (graph-capturable)."""
    n, b, z, c, a = q.shape
    dev = q.device
    flag = torch.zeros(1, dtype=torch.int32, device=dev)
    out = torch.empty_like(q)
    rs = torch.empty((n, b, z, c), dtype=torch.float32, device=dev)
    grads = tuple(torch.empty_like(q) for _ in range(3))
    dvec = torch.empty((n, b, z, c), dtype=torch.float32, device=dev)
    gs = torch.empty_like(q)
    if mode == "stream":
        m = torch.empty_like(rs)

        def step():
            engine.forward_stream(q, k, v, flag=flag, out=out, rowscale=rs, rowmax=m)
            engine.backward_stream(q, k, v, g, out, rs, m, grads=grads, dvec=dvec, grad_scaled=gs)
        return step
    panel = torch.empty((n, b, z, c, n * c), dtype=torch.bfloat16, device=dev)

    def step():
        engine.forward(q, k, v, path="fused", flag=flag, out=out, panel=panel, rowscale=rs)
        engine.backward(q, k, v, panel, g, outputs=out, rowscale=rs, path="fused", grads=grads, dvec=dvec,
                        grad_scaled=gs, single_pass=single_pass)
    return step


def graphed(fn):
    fn()
    torch.cuda.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        fn()
    return gr.replay


def rsa_layer(n, b, z, seq, a, iters, dev, graph=False):
    c = seq // n
    gen = torch.Generator(device=dev).manual_seed(seq)
    q, k, v, g = (torch.randn((n, b, z, c, a), generator=gen, device=dev).to(torch.bfloat16) for _ in range(4))
    res = {}
    variants = [("panel", None), ("stream", None)]
    if engine.single_pass_supported(n, b, z, c, a):
        variants = [("panel", True), ("panel", False), ("stream", None)]
    for mode, sp in variants:
        name = mode if sp is None else f"{mode}_{'bwd_fused' if sp else 'bwd_dkdv_dq'}"
        fn = layer_closure(q, k, v, g, mode, sp)
        ms = timed(fn, iters)
        res[name] = {"ms_per_layer_fwd_bwd": ms, "tokens_per_s": b * seq / (ms / 1e3)}
        if graph:
            ms_g = timed(graphed(fn), iters)
            res[name]["graph_ms_per_layer_fwd_bwd"] = ms_g
            res[name]["graph_tokens_per_s"] = b * seq / (ms_g / 1e3)
        torch.cuda.empty_cache()
    return res


def linformer(n, b, z, seq, a, kp, iters, dev):
    c = seq // n
    gen = torch.Generator(device=dev).manual_seed(5)
    ch = [[torch.randn((b, z, c, a), generator=gen, device=dev).to(torch.bfloat16) for _ in range(n)]
          for _ in range(4)]
    s = seq ** -0.5
    w = SparseWeights((torch.randn((kp, seq), generator=gen, device=dev) * s).to(torch.bfloat16),
                      (torch.randn((kp, seq), generator=gen, device=dev) * s).to(torch.bfloat16))
    base = AttentionConfig(batch_size=b, seq_len=seq, hidden_size=z * a, num_heads=z, head_size=a, num_devices=n)
    cfg = SparseAttentionConfig(base=base, proj_dim=kp)
    # chunks as views of whole-sequence tensors (zero copy: the API runs the sequence as one
    # resident rank) ...
    seqs = [torch.cat(x, dim=2) for x in ch]
    sc = [list(t.chunk(n, dim=2)) for t in seqs]
    fwd_ms = timed(lambda: sparse_ring_attention_forward(sc[0], sc[1], sc[2], w, cfg), iters)
    bwd_ms = timed(lambda: sparse_ring_attention_backward(sc[0], sc[1], sc[2], w, cfg, sc[3]), iters)
    # ... and independent contiguous per-rank chunks, as scatter_sequence returns them (stacked
    # into [N][B][Z][c][A] first)
    fwd_ms_sep = timed(lambda: sparse_ring_attention_forward(ch[0], ch[1], ch[2], w, cfg), iters)
    bwd_ms_sep = timed(lambda: sparse_ring_attention_backward(ch[0], ch[1], ch[2], w, cfg, ch[3]), iters)
    del seqs, sc
    # the device path without the list API's chunk stacking: projections, then the fused attention
    from paper_2105_13120_b200 import sparse_attention as spm

    q, k, v = (torch.stack(x) for x in ch[:3])
    proj_ms = timed(lambda: spm._project(q, k, v, w.key_proj, w.value_proj, kp), iters)
    k16, v16 = spm._project(q, k, v, w.key_proj, w.value_proj, kp)
    attn_ms = timed(lambda: spm.low_rank_attention(q, k16, v16), iters)
    # algorithmic HBM bytes of the forward: read q, k, v and write O (bf16), E/F blocks
    fwd_bytes = 4 * 2 * b * z * seq * a + 2 * 2 * kp * seq
    return {"ms_fwd_api": fwd_ms, "ms_bwd_api_incl_recompute": bwd_ms,
            "ms_fwd_api_separate_chunks": fwd_ms_sep, "ms_bwd_api_separate_chunks": bwd_ms_sep,
            "tokens_per_s_fwd_api": b * seq / (fwd_ms / 1e3),
            "tokens_per_s_fwd_bwd_api": b * seq / ((fwd_ms + bwd_ms) / 1e3),
            "ms_fwd_projections": proj_ms, "ms_fwd_low_rank_attention": attn_ms,
            "fwd_device_ms": proj_ms + attn_ms, "fwd_alg_bytes": fwd_bytes,
            "fwd_hbm_frac": fwd_bytes / ((proj_ms + attn_ms) / 1e3) / 6539.9e9}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--iters", type=int, default=5)
    ap.add_argument("--out", default="gpurun_out/configs.json")
    args = ap.parse_args()
    dev = torch.device("cuda", 0)
    res = {}
    res["config1"] = {"shape": "B4 Z12 A64 L512, N=4 logical ranks",
                      **rsa_layer(4, 4, 12, 512, 64, max(args.iters, 20), dev, graph=True)}
    print(json.dumps(res["config1"]), flush=True)
    res["config4"] = {"shape": "BERT-large attention Z16 A64 L16384 B4, N=8 logical ranks (c=2048)",
                      **rsa_layer(8, 4, 16, 16384, 64, args.iters, dev)}
    print(json.dumps(res["config4"]), flush=True)
    res["config5"] = {"shape": "Linformer B4 Z12 A64 L114688 Kp256, N=8 logical ranks",
                      **linformer(8, 4, 12, 114688, 64, 256, args.iters, dev)}
    print(json.dumps(res["config5"]), flush=True)
    Path(args.out).parent.mkdir(parents=True, exist_ok=True)
    Path(args.out).write_text(json.dumps(res, indent=1))


if __name__ == "__main__":
    main()

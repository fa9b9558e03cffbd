"""Tensor-parallel comparator behind ``ringseq.tensor_parallel``.

The paper frames sequence parallelism against Megatron-style tensor parallelism:
weights partitioned, activations replicated (ringseq/tensor_parallel.py:1-8).  Same
names, signatures, result shapes and errors as the reference:

* ``split_mlp_weights(w, n_devices)`` -> ``ColumnRowSplitWeights``      (:40-51)
* ``split_attention_heads(w, cfg, n_devices)`` -> list[AttentionWeights] (:54-76)
* ``tensor_parallel_mlp(x, w, cfg, *, executor=None)`` -> (output, ledger)       (:79-96)
* ``tensor_parallel_attention(x, w, cfg, *, executor=None)`` -> (output, ledger) (:99-122)

Every device's shard is resident on this GPU.  A device's attention over its heads is
independent of the others', so all heads run in one launch of the fused RSA kernels
(one ring rank, the whole sequence); the row-partitioned output projection of each
device is an rsa_gemm, and the partials are summed in ascending device order in fp32 --
the all-reduce, which the ledger charges with the reference's convention
(2E(N-1)/N elements per device, ringseq/cluster.py:320-359).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np
import torch

from . import tensor_ops as ops
from .cluster import CommLedger, resolve_executor
from .config import AttentionConfig
from .errors import ConfigError, ShapeError
from .weights import AttentionWeights

__all__ = ["ColumnRowSplitWeights", "split_mlp_weights", "split_attention_heads", "tensor_parallel_mlp",
           "tensor_parallel_attention", "validate_tensor_parallel"]


@dataclass(frozen=True)
class ColumnRowSplitWeights:
    """Per-device MLP shards: up columns (H, 4H/N) and down rows (4H/N, H)."""

    up_columns: list
    down_rows: list


def validate_tensor_parallel(cfg: AttentionConfig) -> None:
    """ringseq/config.py:59-69: heads and the feed-forward width must split evenly."""
    if cfg.num_heads % cfg.num_devices != 0:
        raise ConfigError(f"num_heads={cfg.num_heads} not divisible by num_devices={cfg.num_devices}")
    if (4 * cfg.hidden_size) % cfg.num_devices != 0:
        raise ConfigError(f"feed-forward width {4 * cfg.hidden_size} not divisible by num_devices={cfg.num_devices}")


def _cols(m, lo, hi):
    return m[:, lo:hi].contiguous() if isinstance(m, torch.Tensor) else np.ascontiguousarray(np.asarray(m)[:, lo:hi])


def _rows(m, lo, hi):
    return m[lo:hi].contiguous() if isinstance(m, torch.Tensor) else np.ascontiguousarray(np.asarray(m)[lo:hi])


def split_mlp_weights(w, n_devices: int) -> ColumnRowSplitWeights:
    """Shard the feed-forward weights; concatenating the shards reconstructs them."""
    width = w.up.shape[1]
    if width % n_devices != 0:
        raise ConfigError(f"feed-forward width {width} not divisible by num_devices={n_devices}")
    step = width // n_devices
    return ColumnRowSplitWeights(
        up_columns=[_cols(w.up, d * step, (d + 1) * step) for d in range(n_devices)],
        down_rows=[_rows(w.down, d * step, (d + 1) * step) for d in range(n_devices)],
    )


def split_attention_heads(w, cfg: AttentionConfig, n_devices: int) -> list:
    """Device d keeps the input-projection columns and output-projection rows of heads
    [d*Z/N, (d+1)*Z/N); head h is the channel slice [h*A, (h+1)*A)."""
    if cfg.num_heads % n_devices != 0:
        raise ConfigError(f"num_heads={cfg.num_heads} not divisible by num_devices={n_devices}")
    out = []
    for d in range(n_devices):
        lo = d * (cfg.num_heads // n_devices) * cfg.head_size
        hi = (d + 1) * (cfg.num_heads // n_devices) * cfg.head_size
        out.append(AttentionWeights(wq=_cols(w.wq, lo, hi), wk=_cols(w.wk, lo, hi), wv=_cols(w.wv, lo, hi),
                                    wo=_rows(w.wo, lo, hi)))
    return out


def _input(x, cfg: AttentionConfig):
    expect = (cfg.batch_size, cfg.seq_len, cfg.hidden_size)
    shape = tuple(x.shape) if hasattr(x, "shape") else np.asarray(x).shape
    if shape != expect:
        raise ShapeError(f"x has shape {shape}, expected {expect}")
    dev = x.device if isinstance(x, torch.Tensor) and x.is_cuda else ops.default_device()
    return ops.to_device(x, dev)


def _all_reduce_ledger(cfg: AttentionConfig) -> CommLedger:
    ledger = CommLedger(cfg.num_devices)
    if cfg.num_devices > 1:
        elements = cfg.batch_size * cfg.seq_len * cfg.hidden_size
        for d in range(cfg.num_devices):
            ledger.record_allreduce(d, elements)
    return ledger


def tensor_parallel_mlp(x, w, cfg: AttentionConfig, *, executor: str | None = None):
    """Column/row-split feed-forward block with replicated input (ringseq/tensor_parallel.py:79-96).
    Returns (output (B, L, H) bf16 -- every device's copy is the same -- and the ledger)."""
    resolve_executor(executor)
    validate_tensor_parallel(cfg)
    xd = _input(x, cfg)
    shards = split_mlp_weights(w, cfg.num_devices)
    out = torch.empty(xd.shape, dtype=torch.float32, device=xd.device)
    for d in range(cfg.num_devices):  # partials summed in ascending device order (the all-reduce)
        up = ops.to_device(shards.up_columns[d], xd.device)
        down = ops.to_device(shards.down_rows[d], xd.device)
        hidden = ops.gelu(ops.matmul(xd, up))
        ops.matmul(hidden, down, out=out, accumulate=d > 0)
    return out.to(torch.bfloat16), _all_reduce_ledger(cfg)


def tensor_parallel_attention(x, w, cfg: AttentionConfig, *, executor: str | None = None):
    """Heads split across devices, input replicated (ringseq/tensor_parallel.py:99-122).
    Returns (output (B, L, H) bf16, ledger)."""
    from .ring_attention import _forward_checked

    resolve_executor(executor)
    validate_tensor_parallel(cfg)
    xd = _input(x, cfg)
    b, seq, z, a, n = cfg.batch_size, cfg.seq_len, cfg.num_heads, cfg.head_size, cfg.num_devices
    shards = split_attention_heads(w, cfg, n)
    dev = xd.device
    wq, wk, wv = (torch.cat([ops.to_device(getattr(s, m), dev) for s in shards], dim=1) for m in ("wq", "wk", "wv"))

    def heads(m):  # (B, L, Z*A) -> [1][B][Z][L][A]: every head over the whole sequence
        return ops.matmul(xd, m, out_dtype=torch.bfloat16).view(b, seq, z, a).permute(0, 2, 1, 3).unsqueeze(0) \
            .contiguous()

    res = _forward_checked(heads(wq), heads(wk), heads(wv), "auto")
    merged = res.out[0].permute(0, 2, 1, 3).reshape(b, seq, z * a)  # merge_heads
    out = torch.empty((b, seq, cfg.hidden_size), dtype=torch.float32, device=dev)
    per = (z // n) * a
    for d in range(n):  # row-partitioned output projections, summed in ascending device order
        ops.matmul(merged[..., d * per:(d + 1) * per], ops.to_device(shards[d].wo, dev), out=out, accumulate=d > 0)
    return out.to(torch.bfloat16), _all_reduce_ledger(cfg)

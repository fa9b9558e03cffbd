"""Sequence-sharded Linformer attention behind the ``ringseq.sparse_attention`` API.

Drop-in counterparts of ringseq/sparse_attention.py:37-149:

* ``split_projection_columns(proj, n_devices)``        (:47-56)
* ``sparse_ring_attention_forward(q, k, v, weights, cfg, *, executor=None)``
  -> ``SparseRingForward(outputs, shape_logs, ledger)`` (:74-133)
* ``full_length_dims(shape_logs, cfg)``                (:136-149)

Protocol per rank d (all arithmetic in sm_100a kernels via ``tensor_ops``):
K'_d = E[:, d-block] K_d and V'_d = F[:, d-block] V_d (tcgen05 GEMMs with the
projection shared across the B*Z heads through a stride-0 batch), the
partials summed across ranks (the reference's N-1 ring-accumulate hops,
:59-71, i.e. an all-reduce), then local low-rank attention softmax(Q_d K'^T /
sqrt(A)) V'.  With every rank resident on one GPU the sum is one fp32
accumulation over the ranks' partial GEMMs (every rank gets the same total;
the reference's totals differ only in addition grouping); across GPUs it is
one NCCL all-reduce of the concatenated [K'; V'] buffer
(``distributed.SpmdRing.linformer_forward``).

The ledger charges the reference's ring-accumulate convention:
2(N-1)*B*Z*K*A elements per rank (ringseq/cost_model.py:160-168).
"""

from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np
import torch

from . import tensor_ops as ops
from .cluster import CommLedger, resolve_executor
from .config import SparseAttentionConfig
from .errors import ShapeError

__all__ = ["SparseRingForward", "split_projection_columns", "sparse_ring_attention_forward", "full_length_dims"]


@dataclass
class SparseRingForward:
    """Per-rank (B, Z, L/N, A) outputs, per-rank allocation shape logs, ledger."""

    outputs: list
    shape_logs: list
    ledger: CommLedger


def _shape(x) -> tuple:
    return tuple(x.shape) if hasattr(x, "shape") else np.asarray(x).shape


def split_projection_columns(proj, n_devices: int) -> list:
    """Split a (K, L) projection into N contiguous (K, L/N) column blocks."""
    shape = _shape(proj)
    if len(shape) != 2:
        raise ShapeError(f"projection must be 2-D, got shape {shape}")
    if shape[1] % n_devices:
        raise ShapeError(f"projection length {shape[1]} not divisible by device count {n_devices}")
    w = shape[1] // n_devices
    if isinstance(proj, torch.Tensor):
        return [proj[:, i * w:(i + 1) * w].contiguous() for i in range(n_devices)]
    arr = np.asarray(proj, dtype=np.float64)
    return [np.ascontiguousarray(arr[:, i * w:(i + 1) * w]) for i in range(n_devices)]


def _stack(chunks, device) -> torch.Tensor:
    out = torch.empty((len(chunks),) + _shape(chunks[0]), dtype=torch.bfloat16, device=device)
    for d, c in enumerate(chunks):
        out[d].copy_(ops.to_device(c, device))
    return out


def sparse_ring_attention_forward(q_chunks, k_chunks, v_chunks, weights, cfg: SparseAttentionConfig, *,
                                  executor: str | None = None) -> SparseRingForward:
    """Projected attention on sequence-partitioned (B, Z, L/N, A) chunks (ringseq/sparse_attention.py:74-133)."""
    resolve_executor(executor)
    base = cfg.base
    n = base.num_devices
    expect = base.chunk_shape()
    q_chunks, k_chunks, v_chunks = list(q_chunks), list(k_chunks), list(v_chunks)
    for name, chunks in (("q_chunks", q_chunks), ("k_chunks", k_chunks), ("v_chunks", v_chunks)):
        if len(chunks) != n:
            raise ShapeError(f"{name}: got {len(chunks)} chunks for {n} devices")
        for i, c in enumerate(chunks):
            if _shape(c) != expect:
                raise ShapeError(f"{name}[{i}] has shape {_shape(c)}, expected {expect}")
    proj_shape = (cfg.proj_dim, base.seq_len)
    kp_shape, vp_shape = _shape(weights.key_proj), _shape(weights.value_proj)
    if kp_shape != proj_shape or vp_shape != proj_shape:
        raise ShapeError(f"projection shapes {kp_shape}/{vp_shape}, expected {proj_shape}")

    dev = None
    for x in q_chunks + k_chunks + v_chunks:
        if isinstance(x, torch.Tensor) and x.is_cuda:
            dev = x.device
            break
    dev = dev or ops.default_device()
    b, z, c, a = expect
    kdim = cfg.proj_dim
    q, k, v = _stack(q_chunks, dev), _stack(k_chunks, dev), _stack(v_chunks, dev)
    e = ops.to_device(weights.key_proj, dev)  # (K, L) bf16
    f = ops.to_device(weights.value_proj, dev)
    # Partial projections of each rank's chunk with its own column block,
    # accumulated over ranks in fp32 (the ring-accumulate / all-reduce).
    k_low = torch.empty((b, z, kdim, a), dtype=torch.float32, device=dev)
    v_low = torch.empty_like(k_low)
    for d in range(n):
        cols = slice(d * c, (d + 1) * c)
        ops.matmul(e[:, cols], k[d], out=k_low, accumulate=d > 0)
        ops.matmul(f[:, cols], v[d], out=v_low, accumulate=d > 0)
    k_low16 = k_low.to(torch.bfloat16)
    v_low16 = v_low.to(torch.bfloat16)
    scale = 1.0 / math.sqrt(a)
    scores = ops.matmul(q, k_low16.transpose(-1, -2))  # [N][B][Z][c][K] fp32
    probs = ops.softmax_rows(scores, scale=scale, out_dtype=torch.bfloat16)  # NumericError on non-finite
    out = ops.matmul(probs, v_low16, out_dtype=torch.bfloat16)  # [N][B][Z][c][A]

    chunk, low, rows = (b, z, c, a), (b, z, kdim, a), (b, z, c, kdim)
    logs = []
    ledger = CommLedger(n)
    for d in range(n):
        # allocation shapes of rank d, in the order the reference logs them (:111-126)
        log = [chunk, low, low] + [low] * (n - 1) + [low] * (n - 1) + [rows, rows, chunk]
        logs.append(log)
        if n > 1:
            ledger.record_ring_send(d, 2 * (n - 1) * b * z * kdim * a)
    return SparseRingForward(outputs=[out[d] for d in range(n)], shape_logs=logs, ledger=ledger)


def full_length_dims(shape_logs, cfg: SparseAttentionConfig) -> list:
    """Every logged shape carrying a full-L dimension (ringseq/sparse_attention.py:136-149)."""
    seq_len = cfg.base.seq_len
    return [shape for log in shape_logs for shape in log if seq_len in shape]

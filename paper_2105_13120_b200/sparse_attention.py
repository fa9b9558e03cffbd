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
sqrt(A)) V' -- for A = 64 and K, c multiples of 8 ONE stream-mode launch
(rsa_fwd_factored_ex with key_chunk = K: scores in TMEM, probabilities in
registers and shared memory, neither in HBM), and its backward the two
stream kernels (rsa_bwd_kv_stream gives the cross-rank sums dK', dV' directly,
rsa_bwd_q_stream gives dQ); other shapes take the primitive kernels (fp32 scores,
rsa_softmax_rows).  With every rank resident on one GPU the sum is one fp32
accumulation over the ranks' partial GEMMs (every rank gets the same total;
the reference's totals differ only in addition grouping); across GPUs it is
one NCCL all-reduce of the concatenated [K'; V'] buffer
(``distributed.SpmdRing.linformer_forward``).

The ledger charges the reference's ring-accumulate convention:
2(N-1)*B*Z*K*A elements per rank (ringseq/cost_model.py:160-168).
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass

import numpy as np
import torch

from . import engine
from . import tensor_ops as ops
from ._native import BF16, F32, check, lib
from .cluster import CommLedger, resolve_executor
from .config import SparseAttentionConfig
from .errors import NumericError, ShapeError

__all__ = ["SparseRingForward", "SparseRingBackward", "split_projection_columns", "sparse_ring_attention_forward",
           "sparse_ring_attention_backward", "full_length_dims", "low_rank_attention"]


@dataclass
class SparseRingForward:
    """Per-rank (B, Z, L/N, A) outputs, per-rank allocation shape logs, ledger."""

    outputs: list
    shape_logs: list
    ledger: CommLedger


@dataclass
class SparseRingBackward:
    """Per-rank (B, Z, L/N, A) gradients of q/k/v, the (K, L) projection gradients, ledger."""

    grad_q: list
    grad_k: list
    grad_v: list
    grad_key_proj: torch.Tensor
    grad_value_proj: torch.Tensor
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


def _sequence_view(chunks):
    """The (1, B, Z, L, A) tensor the chunks are consecutive slices of along the sequence axis
    (chunk d = tokens [d*c, (d+1)*c) of one bf16 device tensor, the layout scatter_sequence
    produces), as a zero-copy view -- or None.  Every Linformer product is local to a query row
    or sums over all ranks' positions, so with every rank resident the whole sequence can run
    as one rank of L rows; the chunk list is only the reference's calling convention."""
    if not chunks or not all(isinstance(x, torch.Tensor) and x.is_cuda and x.dtype == torch.bfloat16 for x in chunks):
        return None
    c0 = chunks[0]
    if c0.dim() != 4 or c0.stride(-1) != 1:
        return None
    step = c0.shape[-2] * c0.stride(-2) * c0.element_size()
    base = c0.untyped_storage().data_ptr()
    for d, x in enumerate(chunks):
        if (x.shape != c0.shape or x.stride() != c0.stride() or x.untyped_storage().data_ptr() != base
                or x.data_ptr() != c0.data_ptr() + d * step):
            return None
    b, z, c, a = c0.shape
    return c0.as_strided((1, b, z, c * len(chunks), a), (0,) + tuple(c0.stride()))


def _device(chunks):
    for x in chunks:
        if isinstance(x, torch.Tensor) and x.is_cuda:
            return x.device
    return ops.default_device()


def _check_inputs(name_chunks, weights, cfg: SparseAttentionConfig):
    base = cfg.base
    n = base.num_devices
    expect = base.chunk_shape()
    out = []
    for name, chunks in name_chunks:
        chunks = list(chunks)
        if len(chunks) != n:
            raise ShapeError(f"{name}: got {len(chunks)} chunks for {n} devices")
        for i, c in enumerate(chunks):
            if _shape(c) != expect:
                raise ShapeError(f"{name}[{i}] has shape {_shape(c)}, expected {expect}")
        out.append(chunks)
    proj_shape = (cfg.proj_dim, base.seq_len)
    kp_shape, vp_shape = _shape(weights.key_proj), _shape(weights.value_proj)
    if kp_shape != proj_shape or vp_shape != proj_shape:
        raise ShapeError(f"projection shapes {kp_shape}/{vp_shape}, expected {proj_shape}")
    return out


def _project(q, k, v, e, f, kdim):
    """K' = sum_d E_d K_d, V' = sum_d F_d V_d as bf16 [B][Z][K][A].

    rsa_linformer_project: every head at once, four heads per 128 x 256 tensor-core tile (E_d
    staged once for four heads), the sum over the resident ranks as one contraction over L in
    ascending rank order -- the reference's ring-accumulate (:59-71) when every rank is
    resident -- split over the SMs with fp32 TMA reduce-add, then bf16.  Shapes it cannot tile
    (A != 64, c % 64, K % 128, B*Z % 4) take the generic path: one rsa_gemm launch per
    projection over every (rank, head) pair into fp32 per-rank partials, summed in ascending
    rank order by rsa_sum_ranks."""
    n, b, z, c, a = q.shape
    if (a == 64 and c % 64 == 0 and kdim % 128 == 0 and (b * z) % 4 == 0 and e.dtype == f.dtype == torch.bfloat16
            and e.stride(1) == f.stride(1) == 1 and e.stride(0) == f.stride(0)):
        dev = q.device
        acc = torch.empty((2, b, z, kdim, a), dtype=torch.float32, device=dev)
        low = torch.empty((2, b, z, kdim, a), dtype=torch.bfloat16, device=dev)
        g = engine._geom(n, b, z, c, a, n * c, 0, n)
        check(lib().rsa_linformer_project(ctypes.byref(g), kdim, e.data_ptr(), f.data_ptr(), e.stride(0),
                                          engine._view(k), engine._view(v), acc[0].data_ptr(), acc[1].data_ptr(),
                                          low[0].data_ptr(), low[1].data_ptr(),
                                          torch.cuda.current_stream(dev).cuda_stream), "rsa_linformer_project")
        return low[0], low[1]
    out = []
    for proj, x in ((e, k), (f, v)):
        blocks = proj.reshape(kdim, n, c).permute(1, 0, 2).unsqueeze(1)  # [N][1][K][c], row stride L
        part = ops.matmul(blocks, x.reshape(n, b * z, c, a))             # [N][B*Z][K][A] fp32
        low = torch.empty((b, z, kdim, a), dtype=torch.bfloat16, device=q.device)
        per_rank = b * z * kdim * a
        check(lib().rsa_sum_ranks(part.data_ptr(), F32, n, per_rank, per_rank, low.data_ptr(), BF16,
                                  torch.cuda.current_stream(q.device).cuda_stream), "rsa_sum_ranks")
        out.append(low)
    return out[0], out[1]


def _fused_ok(a: int, c: int, kdim: int) -> bool:
    return engine.stream_supported(1, 1, 1, c, a, kdim)


def _low_rank_stream(q, k_low16, v_low16):
    """softmax(Q K'^T / sqrt(A)) V' as ONE stream-mode launch (rsa_fwd_factored_ex with
    key_chunk = K, no panel): scores and probabilities never reach HBM.  Returns the
    engine.StreamForward, or None when a row needs the two-pass treatment (flag bit 1)."""
    res = engine.forward_stream(q, k_low16.unsqueeze(0), v_low16.unsqueeze(0))
    status = int(res.flag.item())
    if status & 1:
        raise NumericError("softmax_rows requires finite inputs")
    return None if status else res


def _low_rank_staged(q, k_low16, v_low16):
    """The same product through the primitive kernels (fp32 scores, rsa_softmax_rows, bf16 P):
    shapes the fused kernels cannot tile (A != 64, K or c not a multiple of 8) and flag-bit-1 rows."""
    a = q.shape[-1]
    scores = ops.matmul(q, k_low16.transpose(-1, -2))  # [N][B][Z][c][K] fp32
    probs = ops.softmax_rows(scores, scale=1.0 / math.sqrt(a), out_dtype=torch.bfloat16)  # NumericError
    return probs, ops.matmul(probs, v_low16, out_dtype=torch.bfloat16)


def low_rank_attention(q, k_low, v_low) -> torch.Tensor:
    """Local attention of [N][B][Z][c][A] queries against the projected (B, Z, K, A) keys and
    values (ringseq/sparse_attention.py:124-125); every row is local to its rank."""
    k_low16, v_low16 = k_low.to(torch.bfloat16), v_low.to(torch.bfloat16)
    if _fused_ok(q.shape[-1], q.shape[-2], k_low.shape[-2]):
        res = _low_rank_stream(q, k_low16, v_low16)
        if res is not None:
            return res.out
    return _low_rank_staged(q, k_low16, v_low16)[1]


def sparse_ring_attention_forward(q_chunks, k_chunks, v_chunks, weights, cfg: SparseAttentionConfig, *,
                                  executor: str | None = None, results: str | None = None) -> SparseRingForward:
    """Projected attention on sequence-partitioned (B, Z, L/N, A) chunks (ringseq/sparse_attention.py:74-133)."""
    resolve_executor(executor)
    base = cfg.base
    n = base.num_devices
    expect = base.chunk_shape()
    q_chunks, k_chunks, v_chunks = _check_inputs(
        (("q_chunks", q_chunks), ("k_chunks", k_chunks), ("v_chunks", v_chunks)), weights, cfg)

    dev = _device(q_chunks + k_chunks + v_chunks)
    b, z, c, a = expect
    kdim = cfg.proj_dim
    seq = [_sequence_view(x) for x in (q_chunks, k_chunks, v_chunks)]
    e = ops.to_device(weights.key_proj, dev)  # (K, L) bf16
    f = ops.to_device(weights.value_proj, dev)
    if all(x is not None for x in seq):  # zero-copy: the sequence as one resident rank of L rows
        q, k, v = seq
        k_low16, v_low16 = _project(q, k, v, e, f, kdim)
        whole = low_rank_attention(q, k_low16, v_low16)[0]  # (B, Z, L, A)
        out = [whole[:, :, d * c:(d + 1) * c] for d in range(n)]
    else:
        q, k, v = _stack(q_chunks, dev), _stack(k_chunks, dev), _stack(v_chunks, dev)
        k_low16, v_low16 = _project(q, k, v, e, f, kdim)
        out = low_rank_attention(q, k_low16, v_low16)  # [N][B][Z][c][A]

    chunk, low, rows = (b, z, c, a), (b, z, kdim, a), (b, z, c, kdim)
    logs = []
    ledger = CommLedger(n)
    for d in range(n):
        # allocation shapes of rank d, in the order the reference logs them (:111-126)
        log = [chunk, low, low] + [low] * (n - 1) + [low] * (n - 1) + [rows, rows, chunk]
        logs.append(log)
        if n > 1:
            ledger.record_ring_send(d, 2 * (n - 1) * b * z * kdim * a)
    from .ring_attention import _out_list, _results_mode

    return SparseRingForward(outputs=_out_list(out, n, _results_mode(results)), shape_logs=logs, ledger=ledger)


def sparse_ring_attention_backward(q_chunks, k_chunks, v_chunks, weights, cfg: SparseAttentionConfig,
                                   grad_chunks, *, executor: str | None = None) -> SparseRingBackward:
    """Gradients of ``sparse_ring_attention_forward`` (the reference
    ships the forward only, ringseq/sparse_attention.py:74-133).

    Chain rule through the forward, per rank d with its projection column blocks E_d, F_d:
    dV' = sum_d P_d^T dO_d and dK' = sum_d dS_d^T Q_d (the two cross-rank sums -- one
    all-reduce of [dK'; dV'] across GPUs, the same size as the forward's), then the local
    dQ_d = dS_d K', dK_d = E_d^T dK', dV_d = F_d^T dV', and the projection gradients
    dE[:, d-block] = sum_{b,z} dK' K_d^T, dF[:, d-block] = sum_{b,z} dV' V_d^T.
    dS = P (dO V'^T - rowsum) / sqrt(A) is rsa_softmax_bwd.  Every product is an
    sm_100a GEMM (tensor_ops.matmul).  The ledger charges the forward's ring-accumulate
    convention for the two gradient sums: 2(N-1)*B*Z*K*A elements per rank.
    """
    resolve_executor(executor)
    base = cfg.base
    n = base.num_devices
    q_chunks, k_chunks, v_chunks, grad_chunks = _check_inputs(
        (("q_chunks", q_chunks), ("k_chunks", k_chunks), ("v_chunks", v_chunks), ("grad_chunks", grad_chunks)),
        weights, cfg)
    dev = _device(q_chunks + k_chunks + v_chunks + grad_chunks)
    b, z, c, a = base.chunk_shape()
    kdim = cfg.proj_dim
    seq = [_sequence_view(x) for x in (q_chunks, k_chunks, v_chunks, grad_chunks)]
    n_run, c_run = n, c
    if all(x is not None for x in seq):  # zero-copy: the sequence as one resident rank of L rows
        q, k, v, g = seq
        n_run, c_run = 1, n * c
    else:
        q, k, v, g = (_stack(x, dev) for x in (q_chunks, k_chunks, v_chunks, grad_chunks))
    e = ops.to_device(weights.key_proj, dev)
    f = ops.to_device(weights.value_proj, dev)
    k_low16, v_low16 = _project(q, k, v, e, f, kdim)
    res = _low_rank_stream(q, k_low16, v_low16) if _fused_ok(a, c_run, kdim) else None
    if res is not None:
        # fused: P recomputed on chip; the kv kernel walks every rank's query rows, so its
        # fp32 dK' / dV' are already the cross-rank sums
        dq, d_klow, d_vlow = engine.backward_stream(q, k_low16.unsqueeze(0), v_low16.unsqueeze(0), g, res.out,
                                                    res.rowscale, res.rowmax, dkv_f32=True)
        d_klow, d_vlow = d_klow[0], d_vlow[0]
    else:
        probs, _ = _low_rank_staged(q, k_low16, v_low16)
        # cross-rank sums (fp32 over ranks in ascending order)
        d_vlow = torch.empty((b, z, kdim, a), dtype=torch.float32, device=dev)
        for d in range(n_run):
            ops.matmul(probs[d].transpose(-1, -2), g[d], out=d_vlow, accumulate=d > 0)
        dp = ops.matmul(g, v_low16.transpose(-1, -2))  # [N][B][Z][c][K] fp32
        ds = ops.softmax_backward(probs, dp, 1.0 / math.sqrt(a), out_dtype=torch.bfloat16)
        dq = ops.matmul(ds, k_low16, out_dtype=torch.bfloat16)
        d_klow = torch.empty_like(d_vlow)
        for d in range(n_run):
            ops.matmul(ds[d].transpose(-1, -2), q[d], out=d_klow, accumulate=d > 0)
    d_klow16, d_vlow16 = d_klow.to(torch.bfloat16), d_vlow.to(torch.bfloat16)
    dk = torch.empty((n_run, b, z, c_run, a), dtype=torch.bfloat16, device=dev)
    dv = torch.empty_like(dk)
    grad_e = torch.empty((kdim, base.seq_len), dtype=torch.float32, device=dev)
    grad_f = torch.empty_like(grad_e)
    if (a == 64 and c_run % 128 == 0 and kdim % 64 == 0 and (b * z) % 4 == 0 and e.stride(1) == f.stride(1) == 1
            and e.stride(0) == f.stride(0)):
        # dK_d = E_d^T dK', dV_d = F_d^T dV' for every rank and head in one launch
        g_ = engine._geom(n_run, b, z, c_run, a, n * c, 0, n_run)
        check(lib().rsa_linformer_proj_back(ctypes.byref(g_), kdim, e.data_ptr(), f.data_ptr(), e.stride(0),
                                            d_klow16.data_ptr(), d_vlow16.data_ptr(), engine._view(dk),
                                            engine._view(dv), torch.cuda.current_stream(dev).cuda_stream),
              "rsa_linformer_proj_back")
    else:
        for d in range(n_run):
            cols = slice(d * c_run, (d + 1) * c_run)
            ops.matmul(e[:, cols].transpose(0, 1), d_klow16, out=dk[d])
            ops.matmul(f[:, cols].transpose(0, 1), d_vlow16, out=dv[d])
    if a == 64 and c_run % 256 == 0 and kdim % 128 == 0:
        # dE / dF for every rank in one launch: each (Kp x 256-position) tile sums the heads'
        # dK'_h K_{d,h}^T with both operands read in place (csrc/linformer.cu)
        g_ = engine._geom(n_run, b, z, c_run, a, n * c, 0, n_run)
        check(lib().rsa_linformer_proj_grad(ctypes.byref(g_), kdim, d_klow16.data_ptr(), d_vlow16.data_ptr(),
                                            engine._view(k), engine._view(v), grad_e.data_ptr(), grad_f.data_ptr(),
                                            grad_e.stride(0), torch.cuda.current_stream(dev).cuda_stream),
              "rsa_linformer_proj_grad")
    else:
        # (K, B*Z*A) views of the low-rank gradients for the shared-projection gradients
        dk_flat = d_klow16.permute(2, 0, 1, 3).reshape(kdim, b * z * a)
        dv_flat = d_vlow16.permute(2, 0, 1, 3).reshape(kdim, b * z * a)
        for d in range(n_run):
            cols = slice(d * c_run, (d + 1) * c_run)
            ops.matmul(dk_flat, k[d].transpose(-1, -2).reshape(b * z * a, c_run), out=grad_e[:, cols])
            ops.matmul(dv_flat, v[d].transpose(-1, -2).reshape(b * z * a, c_run), out=grad_f[:, cols])
    ledger = CommLedger(n)
    if n > 1:
        for d in range(n):
            ledger.record_ring_send(d, 2 * (n - 1) * b * z * kdim * a)
    per_rank = (lambda t: [t[0][:, :, d * c:(d + 1) * c] for d in range(n)]) if n_run == 1 and n > 1 else (
        lambda t: [t[d] for d in range(n)])
    return SparseRingBackward(grad_q=per_rank(dq), grad_k=per_rank(dk), grad_v=per_rank(dv), grad_key_proj=grad_e,
                              grad_value_proj=grad_f, ledger=ledger)


def full_length_dims(shape_logs, cfg: SparseAttentionConfig) -> list:
    """Every logged shape carrying a full-L dimension (ringseq/sparse_attention.py:136-149)."""
    seq_len = cfg.base.seq_len
    return [shape for log in shape_logs for shape in log if seq_len in shape]

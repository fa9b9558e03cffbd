"""Device primitives of the RSA path: ``matmul`` and ``softmax_rows`` on sm_100a.

Counterparts of ringseq/tensor_ops.py:44-84 with the reference's names and
error behaviour (ShapeError on bad shapes, NumericError on non-finite
softmax input).  Arithmetic differs by design: operands are bf16, products
accumulate in fp32 on tcgen05 tensor cores (TMEM), softmax works in fp32.
The reference's fixed summation order is a property of its float64 NumPy
loop and is not reproduced; parity is gated by tolerances instead (see
DESIGN.md, "Numerics").

``split_heads`` / ``merge_heads`` (ringseq/tensor_ops.py:93-119) are pure
layout changes; the fused kernels consume strided views directly, so these
helpers are only used at the API surface.
"""

from __future__ import annotations

import numpy as np
import torch

from . import _native
from ._native import BF16, F32, check, lib
from .errors import NumericError, ShapeError

__all__ = [
    "to_device",
    "matmul",
    "softmax_rows",
    "softmax_backward",
    "rowdot",
    "rowdot_scale",
    "gelu",
    "gelu_backward",
    "panel_normalize",
    "split_heads",
    "merge_heads",
    "set_gemm_backend",
]

_DT = {torch.float32: F32, torch.bfloat16: BF16}


def _stream(t: torch.Tensor) -> int:
    return torch.cuda.current_stream(t.device).cuda_stream


def default_device() -> torch.device:
    if not torch.cuda.is_available():
        raise _native.NativeUnavailable("no CUDA device: the RSA kernels only run on an sm_100a GPU")
    return torch.device("cuda", torch.cuda.current_device())


def to_device(x, device=None, dtype=torch.bfloat16) -> torch.Tensor:
    """Move an array-like to ``device`` in ``dtype``.

    float64 NumPy input is rounded through float32, matching the oracle's
    ``bf16_round`` (f64 -> f32 -> bf16, nearest-even at each step).
    """
    if device is None:
        device = x.device if isinstance(x, torch.Tensor) and x.is_cuda else default_device()
    if isinstance(x, torch.Tensor):
        if x.dtype == torch.float64:
            x = x.to(torch.float32)
        # pinned host memory: asynchronous on the current stream (callers may overlap layers on streams)
        return x.to(device=device, dtype=dtype, non_blocking=x.device.type == "cpu" and x.is_pinned())
    arr = np.asarray(x)
    if arr.dtype != np.float32:
        arr = arr.astype(np.float32)
    return torch.from_numpy(np.ascontiguousarray(arr)).to(device=device).to(dtype)


def set_gemm_backend(name: str) -> None:
    """'auto' | 'tcgen05' | 'simt' -- test hook to pin one GEMM backend."""
    code = {"auto": 0, "tcgen05": 1, "simt": 2}[name]
    check(lib().rsa_gemm_set_backend(code), "rsa_gemm_set_backend")


def _matrix_layout(t: torch.Tensor):
    """(trans, ld) for the trailing 2-D block of t, or None if neither dim is unit-stride."""
    rows, cols = t.shape[-2], t.shape[-1]
    sr, sc = t.stride(-2), t.stride(-1)
    # A leading dimension of a single row/column is never dereferenced; pick
    # one the TMA path accepts (a multiple of 8 elements).
    if sc == 1 or cols == 1:
        return 0, (sr if rows > 1 else -(-cols // 8) * 8)
    if sr == 1 or rows == 1:
        return 1, (sc if cols > 1 else -(-rows // 8) * 8)
    return None


def _coalesce(lead, strides_list):
    """Merge adjacent leading dims that are contiguous for every operand."""
    dims = [(s, [st[i] for st in strides_list]) for i, s in enumerate(lead) if s != 1]
    merged = []
    for size, strs in dims:
        if merged:
            psize, pstrs = merged[-1]
            if all(ps == s * size for ps, s in zip(pstrs, strs)):
                merged[-1] = (psize * size, strs)
                continue
        merged.append((size, strs))
    return merged


def matmul(a, b, out_dtype=torch.float32, *, alpha: float = 1.0, out: torch.Tensor | None = None,
           accumulate: bool = False) -> torch.Tensor:
    """Batched matrix product over the trailing two axes, leading axes broadcast.

    ringseq/tensor_ops.py:44-72.  Operands are taken to bf16 on the GPU;
    the product accumulates in fp32.  Returns ``out_dtype`` (fp32 default).
    """
    a_t = a if isinstance(a, torch.Tensor) and a.is_cuda else None
    dev = a_t.device if a_t is not None else (b.device if isinstance(b, torch.Tensor) and b.is_cuda else None)
    a = to_device(a, dev) if not (isinstance(a, torch.Tensor) and a.is_cuda and a.dtype in _DT) else a
    b = to_device(b, a.device) if not (isinstance(b, torch.Tensor) and b.is_cuda and b.dtype in _DT) else b
    if a.dim() < 2 or b.dim() < 2:
        raise ShapeError(f"matmul needs operands with at least 2 dimensions, got {tuple(a.shape)} and {tuple(b.shape)}")
    if a.shape[-1] != b.shape[-2]:
        raise ShapeError(f"matmul inner dimensions disagree: {tuple(a.shape)} vs {tuple(b.shape)}")
    try:
        lead = tuple(torch.broadcast_shapes(a.shape[:-2], b.shape[:-2]))
    except RuntimeError as exc:
        raise ShapeError(f"matmul batch dimensions disagree: {tuple(a.shape)} vs {tuple(b.shape)}") from exc
    m, k = a.shape[-2], a.shape[-1]
    n = b.shape[-1]
    if out is None:
        out = torch.empty(lead + (m, n), dtype=out_dtype, device=a.device)
        if accumulate:
            raise ShapeError("accumulate=True needs an explicit out tensor")
    if out.dtype not in _DT or out.stride(-1) != 1 and n > 1:
        raise ShapeError("matmul out must be fp32/bf16 with a unit-stride last axis")
    if out.numel() == 0:
        return out
    ae = a.expand(lead + (m, k))
    be = b.expand(lead + (k, n))
    la = _matrix_layout(ae)
    if la is None:
        ae = ae.contiguous()
        la = _matrix_layout(ae)
    lb = _matrix_layout(be)
    if lb is None:
        be = be.contiguous()
        lb = _matrix_layout(be)
    ldc = out.stride(-2) if m > 1 else n
    nlead = len(lead)
    groups = _coalesce(lead, [ae.stride()[:nlead], be.stride()[:nlead], out.stride()[:nlead]])
    # At most two batch levels go to the kernel; outer ones loop here.
    unit = (1, [0, 0, 0])
    inner = ([unit, unit] + groups)[-2:]
    outer = groups[:-2]
    (nb1, s1), (nb2, s2) = inner
    L = lib()
    stream = _stream(a)
    asz, bsz, csz = ae.element_size(), be.element_size(), out.element_size()
    import itertools

    for idx in itertools.product(*[range(sz) for sz, _ in outer]):
        offs = [sum(i * strs[j] for i, (_, strs) in zip(idx, outer)) for j in range(3)]
        code = L.rsa_gemm(
            m, n, k,
            ae.data_ptr() + offs[0] * asz, _DT[ae.dtype], la[1], la[0], s1[0], s2[0],
            be.data_ptr() + offs[1] * bsz, _DT[be.dtype], lb[1], lb[0], s1[1], s2[1],
            out.data_ptr() + offs[2] * csz, _DT[out.dtype], ldc, s1[2], s2[2],
            nb1, nb2, float(alpha), int(accumulate), stream,
        )
        check(code, "rsa_gemm")
    return out


def softmax_rows(t, *, scale: float = 1.0, out_dtype=torch.float32, check_finite: bool = True,
                 out: torch.Tensor | None = None) -> torch.Tensor:
    """Row-stabilised softmax along the last axis (ringseq/tensor_ops.py:75-84).

    Computes softmax(scale * t).  Non-finite input raises NumericError after
    the kernel (one device->host flag read) unless ``check_finite`` is False.
    """
    if not (isinstance(t, torch.Tensor) and t.is_cuda and t.dtype in _DT):
        t = to_device(t, dtype=torch.float32)
    if t.dim() < 1 or t.shape[-1] < 1:
        raise ShapeError(f"softmax_rows needs a non-empty last axis, got shape {tuple(t.shape)}")
    cols = t.shape[-1]
    x = t if t.is_contiguous() else t.contiguous()
    rows = x.numel() // cols
    if out is None:
        out = torch.empty(t.shape, dtype=out_dtype, device=t.device)
    flag = torch.zeros(1, dtype=torch.int32, device=t.device)
    code = lib().rsa_softmax_rows(x.data_ptr(), _DT[x.dtype], rows, cols, cols, float(scale),
                                  out.data_ptr(), _DT[out.dtype], cols, flag.data_ptr(), _stream(x))
    check(code, "rsa_softmax_rows")
    if check_finite and int(flag.item()):
        raise NumericError("softmax_rows requires finite inputs")
    return out


def softmax_backward(p: torch.Tensor, dp: torch.Tensor, scale: float, out_dtype=torch.bfloat16,
                     out: torch.Tensor | None = None) -> torch.Tensor:
    """ds = p * (dp - rowsum(dp * p)) * scale (ringseq/ring_attention.py:187-190)."""
    if p.shape != dp.shape:
        raise ShapeError(f"softmax_backward shapes {tuple(p.shape)} vs {tuple(dp.shape)}")
    cols = p.shape[-1]
    p = p.contiguous()
    dp = dp.contiguous().to(torch.float32)
    rows = p.numel() // cols
    if out is None:
        out = torch.empty(p.shape, dtype=out_dtype, device=p.device)
    code = lib().rsa_softmax_bwd(p.data_ptr(), _DT[p.dtype], cols, dp.data_ptr(), cols, rows, cols, float(scale),
                                 out.data_ptr(), _DT[out.dtype], cols, _stream(p))
    check(code, "rsa_softmax_bwd")
    return out


def rowdot(a: torch.Tensor, b: torch.Tensor, out: torch.Tensor | None = None) -> torch.Tensor:
    """out[..., r] = sum_c a[..., r, c] * b[..., r, c] in fp32 (bf16 inputs)."""
    if a.shape != b.shape or a.dtype != torch.bfloat16 or b.dtype != torch.bfloat16:
        raise ShapeError("rowdot needs two bf16 tensors of the same shape")
    cols = a.shape[-1]
    a = a.contiguous()
    b = b.contiguous()
    rows = a.numel() // max(cols, 1)
    if out is None:
        out = torch.empty(a.shape[:-1], dtype=torch.float32, device=a.device)
    check(lib().rsa_rowdot(a.data_ptr(), cols, b.data_ptr(), cols, rows, cols, out.data_ptr(), _stream(a)), "rsa_rowdot")
    return out


def rowdot_scale(a: torch.Tensor, b: torch.Tensor, scale: torch.Tensor, out: torch.Tensor | None = None,
                 a_scaled: torch.Tensor | None = None):
    """(scale * rowsum(a * b), bf16(scale[..., None] * a)) for bf16 a, b and fp32 per-row scale."""
    if a.shape != b.shape or a.dtype != torch.bfloat16 or b.dtype != torch.bfloat16:
        raise ShapeError("rowdot_scale needs two bf16 tensors of the same shape")
    if scale.dtype != torch.float32 or scale.shape != a.shape[:-1]:
        raise ShapeError(f"rowdot_scale: scale must be fp32 of shape {tuple(a.shape[:-1])}")
    cols = a.shape[-1]
    a, b, scale = a.contiguous(), b.contiguous(), scale.contiguous()
    rows = a.numel() // max(cols, 1)
    if out is None:
        out = torch.empty(a.shape[:-1], dtype=torch.float32, device=a.device)
    if a_scaled is None:
        a_scaled = torch.empty_like(a)
    check(lib().rsa_rowdot_scale(a.data_ptr(), cols, b.data_ptr(), cols, scale.data_ptr(), rows, cols, out.data_ptr(),
                                 a_scaled.data_ptr(), cols, _stream(a)), "rsa_rowdot_scale")
    return out, a_scaled


def panel_normalize(panel: torch.Tensor, scale: torch.Tensor, out_dtype=torch.float32) -> torch.Tensor:
    """Probabilities from a factored panel: scale[..., None] * panel (bf16 panel, fp32 row scale)."""
    if panel.dtype != torch.bfloat16 or scale.dtype != torch.float32 or scale.shape != panel.shape[:-1]:
        raise ShapeError("panel_normalize needs a bf16 panel and an fp32 scale per row")
    cols = panel.shape[-1]
    panel, scale = panel.contiguous(), scale.contiguous()
    rows = panel.numel() // max(cols, 1)
    out = torch.empty(panel.shape, dtype=out_dtype, device=panel.device)
    check(lib().rsa_panel_normalize(panel.data_ptr(), cols, scale.data_ptr(), rows, cols, out.data_ptr(),
                                    _DT[out_dtype], cols, _stream(panel)), "rsa_panel_normalize")
    return out


def gelu(x: torch.Tensor, out_dtype=torch.bfloat16) -> torch.Tensor:
    """Exact GELU x * Phi(x) (ringseq/tensor_ops.py:87-90), fp32 arithmetic (rsa_gelu)."""
    if not (isinstance(x, torch.Tensor) and x.is_cuda and x.dtype in _DT):
        x = to_device(x, dtype=torch.float32)
    x = x.contiguous()
    y = torch.empty(x.shape, dtype=out_dtype, device=x.device)
    check(lib().rsa_gelu(x.data_ptr(), _DT[x.dtype], x.numel(), y.data_ptr(), _DT[out_dtype], _stream(x)),
          "rsa_gelu")
    return y


def gelu_backward(x: torch.Tensor, dy: torch.Tensor, out_dtype=torch.bfloat16) -> torch.Tensor:
    """dx = dy * (Phi(x) + x phi(x)) for y = gelu(x) (rsa_gelu_bwd)."""
    if x.shape != dy.shape:
        raise ShapeError(f"gelu_backward shapes {tuple(x.shape)} vs {tuple(dy.shape)}")
    x, dy = x.contiguous(), dy.contiguous()
    dx = torch.empty(x.shape, dtype=out_dtype, device=x.device)
    check(lib().rsa_gelu_bwd(x.data_ptr(), _DT[x.dtype], dy.data_ptr(), _DT[dy.dtype], x.numel(), dx.data_ptr(),
                             _DT[out_dtype], _stream(x)), "rsa_gelu_bwd")
    return dx


def split_heads(t, num_heads: int):
    """(..., S, Z*A) -> (..., Z, S, A), head h = channels [h*A, (h+1)*A) (ringseq/tensor_ops.py:93-110)."""
    if t.dim() < 2:
        raise ShapeError(f"split_heads needs at least 2 dimensions, got shape {tuple(t.shape)}")
    if num_heads < 1:
        raise ShapeError(f"split_heads needs a positive head count, got {num_heads}")
    ch = t.shape[-1]
    if ch % num_heads:
        raise ShapeError(f"split_heads: channel dimension {ch} not divisible by {num_heads} heads")
    x = t.reshape(t.shape[:-1] + (num_heads, ch // num_heads))
    return x.transpose(-3, -2).contiguous()


def merge_heads(t):
    """(..., Z, S, A) -> (..., S, Z*A), exact inverse of split_heads (ringseq/tensor_ops.py:113-119)."""
    if t.dim() < 3:
        raise ShapeError(f"merge_heads needs at least 3 dimensions, got shape {tuple(t.shape)}")
    x = t.transpose(-3, -2).contiguous()
    return x.reshape(x.shape[:-2] + (x.shape[-2] * x.shape[-1],))

"""Device orchestration of the RSA protocol on stacked chunk tensors.

Every tensor here is stacked over ring ranks: per-head chunks are
``[N][B][Z][c][A]`` and probability / dS panels ``[N][B][Z][c][L]`` (bf16).
Rank d's slice is exactly the chunk / panel the reference keeps on device d
(ringseq/ring_attention.py:43-60), so the list API in ``ring_attention.py``
returns views of these stacks.

Two device paths compute the same protocol:

* ``fused`` (A = 64, c % 8 == 0): the four tcgen05 kernels of
  csrc/fused.cu.  With all N ranks resident in one GPU's HBM a ring hop is a
  pointer rotation, so one launch per stage covers every (rank, origin)
  pair: the K-ring stage is rsa_fwd_stats, the V-ring stage
  rsa_fwd_probs_pv, and the backward's V ring / K ring are rsa_bwd_dkdv /
  rsa_bwd_dq.  dK/dV are reduced over ranks inside rsa_bwd_dkdv (the CTA
  for a key tile walks every rank's query rows), which is the all-reduce of
  ringseq/ring_attention.py:206-209 done in TMEM.
* ``staged``: the reference's own stage structure built from the primitive
  kernels -- per-origin score GEMMs into an fp32 panel, row softmax, per-
  origin PV GEMMs summed in ascending origin order; backward dP panel,
  softmax Jacobian, dQ / dK / dV GEMMs with the dK/dV partials summed over
  ranks in ascending order (ringseq/cluster.py:346-349).  Any shape.
"""

from __future__ import annotations

import ctypes
import math
import os
from typing import NamedTuple

import torch

from . import tensor_ops as ops
from ._native import BF16, F32, RsaFwdExt, RsaGeom, RsaView, check, lib
from .errors import ShapeError

__all__ = ["fused_supported", "forward", "backward", "Forward", "normalized_panel", "recompute_outputs", "NULL_VIEW",
           "KernelTimer", "StreamForward", "forward_stream", "backward_stream", "stream_backward_kernels", "stream_panel",
           "deterministic", "backward_kind",
           "stream_supported"]

NULL_VIEW = RsaView(None, 0, 0, 0, 0)


class KernelTimer:
    """Per-kernel CUDA-event timing on the launching stream (bench instrumentation).

    ``with timer("fwd_pv"): launch(...)`` records an event pair around the
    launch; ``totals()`` returns {name: (launches, total_ms)} after a sync.
    """

    def __init__(self, external: bool = False):
        self.events: dict[str, list] = {}
        self.enabled = True
        # external: events that keep their timestamps when recorded inside a CUDA-graph
        # capture (cudaEventRecordExternal), so a replayed step can be timed per kernel
        self.external = external

    def __call__(self, name: str):
        return _Span(self, name)

    def totals(self) -> dict:
        torch.cuda.synchronize()
        return {k: (len(v), sum(a.elapsed_time(b) for a, b in v)) for k, v in self.events.items()}

    def reset(self) -> None:
        self.events.clear()


class _Span:
    __slots__ = ("t", "name", "a")

    def __init__(self, t, name):
        self.t, self.name = t, name

    def __enter__(self):
        if self.t.enabled:
            self.a = torch.cuda.Event(enable_timing=True, external=self.t.external)
            self.a.record()

    def __exit__(self, *exc):
        if self.t.enabled:
            b = torch.cuda.Event(enable_timing=True, external=self.t.external)
            b.record()
            self.t.events.setdefault(self.name, []).append((self.a, b))


class _NoTimer:
    def __call__(self, name):
        return _NULL_SPAN


class _NullSpan:
    def __enter__(self):
        return None

    def __exit__(self, *exc):
        return False


_NULL_SPAN = _NullSpan()
_NO_TIMER = _NoTimer()


def _stream(t: torch.Tensor) -> int:
    return torch.cuda.current_stream(t.device).cuda_stream


def _view(t: torch.Tensor | None) -> RsaView:
    if t is None:
        return NULL_VIEW
    if t.dim() != 5 or t.stride(-1) != 1:
        raise ShapeError(f"expected a [rank][b][z][row][col] tensor with unit column stride, got {tuple(t.shape)}")
    return RsaView(t.data_ptr(), t.stride(0), t.stride(1), t.stride(2), t.stride(3))


def _geom(n_rank, b, z, c, a, seq, org_lo, n_org, key_chunk=0) -> RsaGeom:
    return RsaGeom(n_rank, b, z, c, a, seq, org_lo, n_org, 1.0 / math.sqrt(a), key_chunk)


def fused_supported(n: int, b: int, z: int, c: int, a: int) -> bool:
    g = _geom(n, b, z, c, a, n * c, 0, n)
    return bool(lib().rsa_fused_supported(ctypes.byref(g)))


def _pick(path: str, n, b, z, c, a) -> str:
    if path == "auto":
        return "fused" if fused_supported(n, b, z, c, a) else "staged"
    if path not in ("fused", "staged"):
        raise ValueError(f"unknown path {path!r}")
    if path == "fused" and not fused_supported(n, b, z, c, a):
        raise ShapeError(f"fused kernels cannot tile N={n} B={b} Z={z} c={c} A={a} (need A=64, c%8==0)")
    return path


# ----------------------------------------------------------------- forward

class Forward(NamedTuple):
    """Result of ``forward``: outputs and the saved probability panel.

    ``rowscale`` is None for a normalised panel (panel = P).  For a factored
    panel (rsa_fwd_factored) it is the fp32 [N][B][Z][c] row scale r with
    P = r * panel; ``backward`` and ``ring_attention.ProbPanels`` take either.
    """

    out: torch.Tensor
    panel: torch.Tensor
    rowscale: torch.Tensor | None
    flag: torch.Tensor


def forward(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, *, path: str = "auto",
            flag: torch.Tensor | None = None, out: torch.Tensor | None = None,
            panel: torch.Tensor | None = None, stats: torch.Tensor | None = None,
            rowscale: torch.Tensor | None = None, factored: bool = True, timer=None) -> Forward:
    """RSA forward on stacked [N][B][Z][c][A] bf16 chunks.

    Returns ``Forward(out, panel, rowscale, flag)``: outputs [N][B][Z][c][A]
    bf16, the panel [N][B][Z][c][L] bf16 (factored when ``rowscale`` is not
    None), and the status flag, a device int the kernels OR bits into (callers
    decide when to read it): bit 0 = a non-finite score, bit 1 = the factored
    kernel needs the two-pass fallback (``factored=False``) for this input.

    Fused path: ``factored`` (default) runs rsa_fwd_factored (one exp2 per
    panel element); ``factored=False`` the normalised rsa_fwd_resident, and a
    ``stats`` buffer the two-launch K-ring / V-ring form.
    """
    n, b, z, c, a = q.shape
    seq = n * c
    dev = q.device
    if flag is None:
        flag = torch.zeros(1, dtype=torch.int32, device=dev)
    if out is None:
        out = torch.empty((n, b, z, c, a), dtype=torch.bfloat16, device=dev)
    if panel is None:
        panel = torch.empty((n, b, z, c, seq), dtype=torch.bfloat16, device=dev)
    which = _pick(path, n, b, z, c, a)
    if which == "fused":
        tm = timer or _NO_TIMER
        L = lib()
        st = _stream(q)
        g = _geom(n, b, z, c, a, seq, 0, n)
        if stats is not None:  # two-launch form (K-ring stats, then V-ring probs/PV)
            with tm("fwd_stats"):
                check(L.rsa_fwd_stats(ctypes.byref(g), _view(q), _view(k), stats.data_ptr(), 0, flag.data_ptr(),
                                      st), "rsa_fwd_stats")
            with tm("fwd_probs_pv"):
                check(L.rsa_fwd_probs_pv(ctypes.byref(g), _view(q), _view(k), _view(v), stats.data_ptr(), 1,
                                         _view(panel), NULL_VIEW, 0, _view(out), st), "rsa_fwd_probs_pv")
            return Forward(out, panel, None, flag)
        if factored:
            if rowscale is None:
                rowscale = torch.empty((n, b, z, c), dtype=torch.float32, device=dev)
            with tm("fwd_factored"):
                check(L.rsa_fwd_factored(ctypes.byref(g), _view(q), _view(k), _view(v), _view(panel), _view(out),
                                         rowscale.data_ptr(), flag.data_ptr(), st), "rsa_fwd_factored")
            return Forward(out, panel, rowscale, flag)
        with tm("fwd_resident"):
            check(L.rsa_fwd_resident(ctypes.byref(g), _view(q), _view(k), _view(v), _view(panel), _view(out),
                                     flag.data_ptr(), st), "rsa_fwd_resident")
        return Forward(out, panel, None, flag)
    _forward_staged(q, k, v, out, panel, flag)
    return Forward(out, panel, None, flag)


def normalized_panel(panel: torch.Tensor, rowscale: torch.Tensor | None, dtype=torch.float32) -> torch.Tensor:
    """The reference's probs from a saved panel: rowscale * panel (or the panel itself when normalised)."""
    if rowscale is None:
        return panel if panel.dtype == dtype else panel.to(dtype)
    return ops.panel_normalize(panel, rowscale, out_dtype=dtype)


def _softmax_into(x: torch.Tensor, y: torch.Tensor, scale: float, flag: torch.Tensor) -> None:
    cols = x.shape[-1]
    rows = x.numel() // cols
    check(lib().rsa_softmax_rows(x.data_ptr(), F32, rows, cols, cols, float(scale), y.data_ptr(), BF16, cols,
                                 flag.data_ptr(), _stream(x)), "rsa_softmax_rows")


def _forward_staged(q, k, v, out, panel, flag) -> None:
    n, b, z, c, a = q.shape
    scale = 1.0 / math.sqrt(a)
    scores = torch.empty((b, z, c, n * c), dtype=torch.float32, device=q.device)
    acc = torch.empty((b, z, c, a), dtype=torch.float32, device=q.device)
    for d in range(n):
        # stage 1: score row blocks in ring arrival order (origin d, d-1, ...)
        for h in range(n):
            j = (d - h) % n
            ops.matmul(q[d], k[j].transpose(-1, -2), out=scores[..., j * c:(j + 1) * c])
        _softmax_into(scores, panel[d], scale, flag)
        # stage 2: O = sum_j P_j V_j in ascending origin order
        for j in range(n):
            ops.matmul(panel[d][..., j * c:(j + 1) * c], v[j], out=acc, accumulate=j > 0)
        out[d].copy_(acc)


# ---------------------------------------------------------------- backward

def recompute_outputs(panel: torch.Tensor, v: torch.Tensor) -> torch.Tensor:
    """O = P V from saved panels (used when the caller's panels carry no O)."""
    n, b, z, c, _ = panel.shape
    a = v.shape[-1]
    out = torch.empty((n, b, z, c, a), dtype=torch.bfloat16, device=panel.device)
    acc = torch.empty((b, z, c, a), dtype=torch.float32, device=panel.device)
    for d in range(n):
        for j in range(n):
            ops.matmul(panel[d][..., j * c:(j + 1) * c], v[j], out=acc, accumulate=j > 0)
        out[d].copy_(acc)
    return out


def backward_kind(n: int, b: int, z: int, c: int, a: int) -> str:
    """The panel backward ``backward(single_pass=None)`` runs for this geometry:
    "bwd_fused" (one CTA per head, one panel read) when it tiles the geometry and there are at
    least half as many heads as SMs; otherwise "bwd_panel_fused" (one CTA per key tile, one
    panel read at any length) when a head has more than 4 query tiles, and the fixed-order
    "bwd_dkdv_dq" pair for the small-batch short shapes (config 1: 44.9 against 45.3 us per
    graph-captured layer for the one-pass kernel with its dQ zero-fill and cast) or under
    RSA_B200_DETERMINISTIC=1."""
    if single_pass_default(n, b, z, c, a):
        return "bwd_fused"
    if not deterministic() and not single_pass_supported(n, b, z, c, a):
        return "bwd_panel_fused"
    return "bwd_dkdv_dq"


def single_pass_default(n: int, b: int, z: int, c: int, a: int) -> bool:
    """The backward ``backward(single_pass=None)`` runs: rsa_bwd_fused when it can tile the
    geometry and there are at least half as many heads as SMs, else rsa_bwd_panel_fused (or,
    with RSA_B200_DETERMINISTIC=1, rsa_bwd_dkdv + rsa_bwd_dq)."""
    return single_pass_supported(n, b, z, c, a) and 2 * b * z >= lib().rsa_num_sms()


def single_pass_supported(n: int, b: int, z: int, c: int, a: int) -> bool:
    """Does rsa_bwd_fused cover this geometry (a head's query rows in <= 4 tiles)?"""
    g = _geom(n, b, z, c, a, n * c, 0, n)
    return bool(lib().rsa_bwd_fused_supported(ctypes.byref(g)))


def backward(q, k, v, panel, grad, *, outputs: torch.Tensor | None = None, path: str = "auto",
             grads: tuple | None = None, dvec: torch.Tensor | None = None, rowscale: torch.Tensor | None = None,
             grad_scaled: torch.Tensor | None = None, timer=None, single_pass: bool | None = None,
             prologue: bool = True, dq_acc: torch.Tensor | None = None):
    """RSA backward on stacked chunks; returns (dq, dk, dv) as [N][B][Z][c][A] bf16.

    ``grads`` / ``dvec`` optionally supply preallocated output and D buffers
    (the bench reuses them across layers).  On the fused path,
    ``single_pass`` picks rsa_bwd_fused (one CTA per head, one panel read; default when the
    geometry allows and there are at least half as many heads as SMs); otherwise, for heads
    of more than 4 query tiles, rsa_bwd_panel_fused (one CTA per key tile, one panel read at
    any length, dQ partials added in L2 through ``dq_acc``), else (or with
    RSA_B200_DETERMINISTIC=1) the fixed-order rsa_bwd_dkdv + rsa_bwd_dq pair, which reads the
    panel twice (see ``backward_kind``).

    ``rowscale`` marks ``panel`` as factored (P = rowscale * panel, see
    ``forward``): rsa_rowdot_scale then forms D*r and dO*r (``grad_scaled``
    optionally preallocates the latter) and the same kernels consume the
    factored panel unchanged.  ``prologue=False`` skips that row pass: ``dvec`` (and
    ``grad_scaled`` for a factored panel) must already hold its results (bench.py times
    the two launches separately)."""
    n, b, z, c, a = q.shape
    seq = n * c
    dev = q.device
    if grads is None:
        dq = torch.empty((n, b, z, c, a), dtype=torch.bfloat16, device=dev)
        dk = torch.empty_like(dq)
        dv = torch.empty_like(dq)
    else:
        dq, dk, dv = grads
    which = _pick(path, n, b, z, c, a)
    if which == "fused":
        tm = timer or _NO_TIMER
        if outputs is None and prologue:
            outputs = recompute_outputs(normalized_panel(panel, rowscale, torch.bfloat16), v)
        if dvec is None:
            if not prologue:
                raise ValueError("prologue=False needs the precomputed dvec")
            dvec = torch.empty((n, b, z, c), dtype=torch.float32, device=dev)
        if not prologue:
            if rowscale is not None:
                if grad_scaled is None:
                    raise ValueError("prologue=False with a factored panel needs grad_scaled")
                grad = grad_scaled
        elif rowscale is None:
            with tm("rowdot"):
                ops.rowdot(grad, outputs, out=dvec)  # D = rowsum(dO * O) = rowsum(dP * P)
        else:  # factored panel: D*r and dO*r, so P (dP - D) = P~ (dO*r V^T - D*r) and P^T dO = P~^T (dO*r)
            with tm("rowdot"):
                dvec, grad = ops.rowdot_scale(grad, outputs, rowscale, out=dvec, a_scaled=grad_scaled)
        L = lib()
        st = _stream(q)
        g = _geom(n, b, z, c, a, seq, 0, n)
        if single_pass is None:
            # one CTA per head: with fewer heads than half the SMs the per-key-tile forms
            # (rsa_bwd_panel_fused, or the two-kernel pair) fill the machine better
            # (config 1, B4 Z12: 46.6 vs 48.4 us per graph-captured layer for the pair)
            single_pass = bool(L.rsa_bwd_fused_supported(ctypes.byref(g))) and 2 * b * z >= L.rsa_num_sms()
        if single_pass:
            with tm("bwd_fused"):
                check(L.rsa_bwd_fused(ctypes.byref(g), _view(q), _view(k), _view(v), _view(grad), _view(panel),
                                      dvec.data_ptr(), NULL_VIEW, 0, _view(dq), _view(dk), _view(dv), BF16, 0, st),
                      "rsa_bwd_fused")
            return dq, dk, dv
        if not deterministic() and not L.rsa_bwd_fused_supported(ctypes.byref(g)):
            dq_acc = _dq_accumulator(dq_acc, (n, b, z, c, a), dev)
            with tm("bwd_panel_fused"):
                check(L.rsa_bwd_panel_fused(ctypes.byref(g), _view(q), _view(k), _view(v), _view(grad), _view(panel),
                                            dvec.data_ptr(), _view(dk), _view(dv), BF16, 0, dq_acc.data_ptr(), 0,
                                            _view(dq), st), "rsa_bwd_panel_fused")
            return dq, dk, dv
        with tm("bwd_dkdv"):
            check(L.rsa_bwd_dkdv(ctypes.byref(g), _view(q), _view(v), _view(grad), _view(panel), dvec.data_ptr(),
                                 _view(dk), _view(dv), BF16, 0, st), "rsa_bwd_dkdv")
        with tm("bwd_dq"):
            check(L.rsa_bwd_dq(ctypes.byref(g), _view(grad), _view(k), _view(v), _view(panel), dvec.data_ptr(),
                               NULL_VIEW, 0, _view(dq), st), "rsa_bwd_dq")
        return dq, dk, dv
    if rowscale is not None:
        panel = normalized_panel(panel, rowscale, torch.bfloat16)
    _backward_staged(q, k, v, panel, grad, dq, dk, dv)
    return dq, dk, dv


def _backward_staged(q, k, v, panel, grad, dq, dk, dv) -> None:
    n, b, z, c, a = q.shape
    seq = n * c
    scale = 1.0 / math.sqrt(a)
    dev = q.device
    dp = torch.empty((b, z, c, seq), dtype=torch.float32, device=dev)
    ds = torch.empty((b, z, c, seq), dtype=torch.bfloat16, device=dev)
    acc = torch.empty((b, z, c, a), dtype=torch.float32, device=dev)
    dk_acc = torch.empty((n, b, z, c, a), dtype=torch.float32, device=dev)
    dv_acc = torch.empty_like(dk_acc)
    for d in range(n):
        # V ring: dP row blocks (ringseq/ring_attention.py:181-184)
        for h in range(n):
            j = (d - h) % n
            ops.matmul(grad[d], v[j].transpose(-1, -2), out=dp[..., j * c:(j + 1) * c])
        ops.softmax_backward(panel[d], dp, scale, out=ds)
        # K ring: dQ in ascending origin order (ringseq/ring_attention.py:193-196)
        for j in range(n):
            ops.matmul(ds[..., j * c:(j + 1) * c], k[j], out=acc, accumulate=j > 0)
        dq[d].copy_(acc)
        # full-length partials, summed over ranks in ascending order
        for j in range(n):
            blk = slice(j * c, (j + 1) * c)
            ops.matmul(ds[..., blk].transpose(-1, -2), q[d], out=dk_acc[j], accumulate=d > 0)
            ops.matmul(panel[d][..., blk].transpose(-1, -2), grad[d], out=dv_acc[j], accumulate=d > 0)
    dk.copy_(dk_acc)
    dv.copy_(dv_acc)


# ------------------------------------------------------------- stream mode

class StreamForward(NamedTuple):
    """Result of ``forward_stream``: outputs plus the two numbers per row the stream-mode
    backward needs -- ``rowscale`` r = 1 / sum_k P~ and ``rowmax`` m, the reference point of
    P~ = 2^(s * scale * log2(e) - m) -- instead of a (c x L) probability panel per row block."""

    out: torch.Tensor
    rowscale: torch.Tensor
    rowmax: torch.Tensor
    flag: torch.Tensor


def stream_supported(n: int, b: int, z: int, c: int, a: int, key_chunk: int = 0) -> bool:
    """Can the stream-mode kernels tile this geometry (A = 64, chunks of 8-row multiples)?"""
    return a == 64 and c % 8 == 0 and (key_chunk or c) % 8 == 0 and min(n, b, z, c) >= 1


def _fwd_ex(q, k, v, g, *, panel=None, rowmax=None, rowmax_in=None, rowmax_stride=1, exact=False, o_acc=None,
            l_acc=None, acc_in=False, final=True, out=None, rowscale=None, flag=None):
    ext = RsaFwdExt(_view(panel), None if rowmax is None else rowmax.data_ptr(),
                    None if rowmax_in is None else rowmax_in.data_ptr(), rowmax_stride, int(exact), _view(o_acc),
                    None if l_acc is None else l_acc.data_ptr(), int(acc_in), int(final))
    check(lib().rsa_fwd_factored_ex(ctypes.byref(g), _view(q), _view(k), _view(v), ctypes.byref(ext), _view(out),
                                    None if rowscale is None else rowscale.data_ptr(), flag.data_ptr(), _stream(q)),
          "rsa_fwd_factored_ex")


def forward_stream(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, *, flag: torch.Tensor | None = None,
                   out: torch.Tensor | None = None, rowscale: torch.Tensor | None = None,
                   rowmax: torch.Tensor | None = None, exact: bool = False) -> StreamForward:
    """Stream-mode RSA forward on stacked [N][B][Z][c][A] bf16 chunks (keys: [N][B][Z][ck][A]).

    One rsa_fwd_factored_ex launch with no panel: O, r and m survive, O(c) per row instead
    of O(L).  ``exact=True`` (the fallback for flag bit 1) first takes every row's true
    maximum with rsa_fwd_stats and runs the single pass on it.  The caller reads ``flag``.
    """
    n, b, z, c, a = q.shape
    ck = k.shape[3]
    dev = q.device
    if flag is None:
        flag = torch.zeros(1, dtype=torch.int32, device=dev)
    if out is None:
        out = torch.empty((n, b, z, c, a), dtype=torch.bfloat16, device=dev)
    if rowscale is None:
        rowscale = torch.empty((n, b, z, c), dtype=torch.float32, device=dev)
    if rowmax is None:
        rowmax = torch.empty((n, b, z, c), dtype=torch.float32, device=dev)
    norg = k.shape[0]
    g = _geom(n, b, z, c, a, norg * ck, 0, norg, 0 if ck == c else ck)
    if not exact:
        _fwd_ex(q, k, v, g, rowmax=rowmax, out=out, rowscale=rowscale, flag=flag)
        return StreamForward(out, rowscale, rowmax, flag)
    if ck != c:
        raise ShapeError("the exact (two-pass) stream forward needs key_chunk == chunk")
    stats = torch.empty((n, b, z, c, 2), dtype=torch.float32, device=dev)
    check(lib().rsa_fwd_stats(ctypes.byref(g), _view(q), _view(k), stats.data_ptr(), 0, flag.data_ptr(), _stream(q)),
          "rsa_fwd_stats")
    _fwd_ex(q, k, v, g, rowmax_in=stats, rowmax_stride=2, exact=True, out=out, rowscale=rowscale, flag=flag)
    rowmax.copy_(stats[..., 0])
    return StreamForward(out, rowscale, rowmax, flag)


def stream_panel(q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, rowmax: torch.Tensor, rowscale: torch.Tensor,
                 d: int, dtype=torch.float32) -> torch.Tensor:
    """Rank d's probability panel (B, Z, c, L) recomputed from a stream-mode forward's
    saved m and r: the factored kernel re-run with m given writes P~ bit for bit as the
    panel forward would have, then P = r * P~ (the reference's probs, materialised only
    when a caller looks at them)."""
    n, b, z, c, a = q.shape
    seq = k.shape[0] * k.shape[3]
    dev = q.device
    qd = q[d:d + 1]
    panel = torch.empty((1, b, z, c, seq), dtype=torch.bfloat16, device=dev)
    scratch_o = torch.empty((1, b, z, c, a), dtype=torch.bfloat16, device=dev)
    scratch_r = torch.empty((1, b, z, c), dtype=torch.float32, device=dev)
    flag = torch.zeros(1, dtype=torch.int32, device=dev)
    g = _geom(1, b, z, c, a, seq, 0, k.shape[0])
    _fwd_ex(qd, k, v, g, panel=panel, rowmax_in=rowmax[d:d + 1].contiguous(), exact=True, out=scratch_o,
            rowscale=scratch_r, flag=flag)
    return normalized_panel(panel[0], rowscale[d], dtype)


def _dq_accumulator(dq_acc: torch.Tensor | None, shape, device) -> torch.Tensor:
    """The one-pass backwards' fp32 dQ accumulator: contiguous [N][B][Z][c][A] fp32 (the kernel
    adds 16-column x 32-row boxes into it by TMA); allocated when not supplied."""
    if dq_acc is None:
        return torch.empty(shape, dtype=torch.float32, device=device)
    if dq_acc.dtype != torch.float32 or tuple(dq_acc.shape) != tuple(shape) or not dq_acc.is_contiguous():
        raise ShapeError(f"dq_acc must be a contiguous fp32 tensor of shape {tuple(shape)}, got "
                         f"{dq_acc.dtype} {tuple(dq_acc.shape)}")
    return dq_acc


def deterministic() -> bool:
    """RSA_B200_DETERMINISTIC=1 selects the stream backward's two-kernel form, whose sums are
    all taken in a fixed order (bitwise reproducible and bitwise equal to the panel mode);
    the default one-pass kernel adds dQ's key-tile partials in arrival order."""
    return os.environ.get("RSA_B200_DETERMINISTIC", "0") not in ("", "0")


def backward_stream(q, k, v, grad, out, rowscale, rowmax, *, grads: tuple | None = None,
                    dvec: torch.Tensor | None = None, grad_scaled: torch.Tensor | None = None,
                    dkv_f32: bool = False, timer=None, fused: bool | None = None, dq_acc: torch.Tensor | None = None):
    """Stream-mode RSA backward: (dq, dk, dv) from q, k, v, dO and the forward's O, r, m.

    rsa_rowdot_scale forms D*r and dO*r; then either rsa_bwd_stream_fused (default: one pass
    per key tile, dQ partials added in L2) or, with ``fused=False`` / RSA_B200_DETERMINISTIC=1,
    rsa_bwd_kv_stream (dK, dV) and rsa_bwd_q_stream (dQ).  Every kernel recomputes P~ on
    chip.  dk / dv are bf16 [N_org][B][Z][ck][A] (fp32 with ``dkv_f32``)."""
    n, b, z, c, a = q.shape
    norg, ck = k.shape[0], k.shape[3]
    dev = q.device
    tm = timer or _NO_TIMER
    if grads is None:
        dq = torch.empty((n, b, z, c, a), dtype=torch.bfloat16, device=dev)
        kdt = torch.float32 if dkv_f32 else torch.bfloat16
        dk = torch.empty((norg, b, z, ck, a), dtype=kdt, device=dev)
        dv = torch.empty_like(dk)
    else:
        dq, dk, dv = grads
    with tm("rowdot"):
        dvec, gsc = ops.rowdot_scale(grad, out, rowscale, out=dvec, a_scaled=grad_scaled)
    return stream_backward_kernels(q, k, v, gsc, rowmax, dvec, (dq, dk, dv), timer=timer, fused=fused, dq_acc=dq_acc)


def stream_backward_kernels(q, k, v, grad_scaled, rowmax, dvec, grads, timer=None, fused: bool | None = None,
                            dq_acc: torch.Tensor | None = None):
    """The stream-mode backward launches on prepared dO*r (``grad_scaled``) and D*r (``dvec``)
    into grads = (dq bf16, dk, dv bf16 or fp32).

    ``fused`` (default: not ``deterministic()``): rsa_bwd_stream_fused, one launch computing
    S, dP and the exp2 once, with ``dq_acc`` (fp32 [N][B][Z][c][A], allocated if None) as its
    dQ accumulator, then the bf16 cast of dQ.  Otherwise rsa_bwd_kv_stream then
    rsa_bwd_q_stream."""
    n, b, z, c, a = q.shape
    norg, ck = k.shape[0], k.shape[3]
    dq, dk, dv = grads
    tm = timer or _NO_TIMER
    g = _geom(n, b, z, c, a, norg * ck, 0, norg, 0 if ck == c else ck)
    L = lib()
    st = _stream(q)
    kdt = F32 if dk.dtype == torch.float32 else BF16
    if fused is None:
        fused = not deterministic()
    if fused:
        dq_acc = _dq_accumulator(dq_acc, (n, b, z, c, a), q.device)
        with tm("bwd_stream_fused"):
            check(L.rsa_bwd_stream_fused(ctypes.byref(g), _view(q), _view(k), _view(v), _view(grad_scaled),
                                         rowmax.data_ptr(), dvec.data_ptr(), _view(dk), _view(dv), kdt, 0,
                                         dq_acc.data_ptr(), 0, _view(dq), st), "rsa_bwd_stream_fused")
        return dq, dk, dv
    with tm("bwd_kv_stream"):
        check(L.rsa_bwd_kv_stream(ctypes.byref(g), _view(q), _view(k), _view(v), _view(grad_scaled),
                                  rowmax.data_ptr(), dvec.data_ptr(), _view(dk), _view(dv), kdt, 0, st),
              "rsa_bwd_kv_stream")
    with tm("bwd_q_stream"):
        check(L.rsa_bwd_q_stream(ctypes.byref(g), _view(q), _view(k), _view(v), _view(grad_scaled),
                                 rowmax.data_ptr(), dvec.data_ptr(), NULL_VIEW, 0, _view(dq), st), "rsa_bwd_q_stream")
    return dq, dk, dv

"""Ring Self-Attention (RSA) behind the reference API of ``ringseq.ring_attention``.

Drop-in counterparts of ringseq/ring_attention.py:124-241 with the same
names, positional/keyword signatures, result dataclasses and exceptions:

* ``ring_attention_forward(q_chunks, k_chunks, v_chunks, cfg, *, executor=None)``
  -> ``RingAttentionForward(outputs, probs, ledger)``
* ``ring_attention_backward(q_chunks, k_chunks, v_chunks, probs, grad_chunks, cfg, *, executor=None)``
  -> ``RingAttentionBackward(grad_q, grad_k, grad_v, ledger)``
* ``sequence_parallel_attention(x_chunks, weights, cfg, *, executor=None)``
  -> ``(results, ledger)``

Chunks may be NumPy arrays (any float dtype) or torch tensors; they are
moved to the GPU as bf16.  Results are CUDA tensors (bf16), one per ring
rank, in the reference's layout: outputs (B, Z, L/N, A), probability panels
(B, Z, L/N, L) whose column block j belongs to origin j.

The ring itself: when every rank's chunk sits in one GPU's HBM (this
single-controller API), a hop is a pointer rotation, and the kernels in
``engine`` read each origin's chunk in place.  The ledger charges exactly
what the reference's simulated ring charges (ringseq/cluster.py:130-135):
2(N-1)*C elements per rank forward; 2(N-1)*C ring plus two all-reduces of
N*C elements backward.  Multi-GPU rings (one process per GPU, NCCL) live in
``distributed.py`` and reuse the same kernels hop by hop.
"""

from __future__ import annotations

import os
from dataclasses import dataclass

import torch

from . import engine
from . import tensor_ops as ops
from .cluster import CommLedger, resolve_executor
from .config import AttentionConfig
from .errors import NumericError, ShapeError, StateError

__all__ = [
    "RingAttentionForward",
    "RingAttentionBackward",
    "ring_attention_forward",
    "ring_attention_backward",
    "sequence_parallel_attention",
    "sequence_parallel_attention_backward",
    "sequence_parallel_mlp",
    "sequence_parallel_mlp_backward",
    "ProbPanels",
    "StreamPanels",
    "check_forward",
]


@dataclass
class RingAttentionForward:
    """Per-rank outputs (B, Z, L/N, A), saved probability panels (B, Z, L/N, L), ledger."""

    outputs: list
    probs: list
    ledger: CommLedger


@dataclass
class RingAttentionBackward:
    """Per-rank gradient chunks for queries, keys and values, plus the ledger."""

    grad_q: list
    grad_k: list
    grad_v: list
    ledger: CommLedger


RESULTS_ENV_VAR = "RSA_B200_RESULTS"
RESULT_MODES = ("device", "numpy")


def _results_mode(results: str | None) -> str:
    """'device' (CUDA bf16 tensors, the default) or 'numpy' (float64 ndarrays, as the
    reference returns them): argument, then $RSA_B200_RESULTS, then 'device'."""
    mode = results or os.environ.get(RESULTS_ENV_VAR) or "device"
    if mode not in RESULT_MODES:
        raise ValueError(f"results must be one of {RESULT_MODES}, got {mode!r}")
    return mode


def _host(t):
    return t.double().cpu().numpy()


def _out_list(stacked, n, mode):
    return [_host(stacked[d]) if mode == "numpy" else stacked[d] for d in range(n)]


class ProbPanels(list):
    """The ``probs`` list returned by the forward: one (B, Z, c, L) panel per rank.

    Backed by one stacked [N][B][Z][c][L] bf16 panel plus, for the fused path,
    an fp32 row scale r (``engine.Forward``): the saved state is the factored
    panel P~ with P = r * P~.  Indexing or iterating materialises rank d's
    probabilities on demand (``engine.normalized_panel``, fp32; a bf16 view
    when the panel is already normalised) and caches them.  Passing the object
    back to ``ring_attention_backward`` (as the reference's callers do with
    ``fwd.probs``) hands the factored panel and the saved outputs straight to
    the kernels -- nothing is materialised or copied.  Any other list of
    panels works too, at the cost of one staging copy.
    """

    def __init__(self, stacked: torch.Tensor, outputs: torch.Tensor, rowscale: torch.Tensor | None = None,
                 inputs: dict | None = None):
        super().__init__([None] * stacked.shape[0])
        self.stacked = stacked
        self.outputs = outputs
        self.rowscale = rowscale
        self.panel_shape = tuple(stacked.shape[1:])
        # device copies of the forward's q / k / v chunks with the identities (object and
        # in-place version) of the caller's torch chunks: a backward called with the same,
        # unmodified tensors reuses them instead of uploading again
        self.inputs = inputs or []
        # a caller that replaces a panel (probs[d] = X) gets reference semantics: the
        # backward then uses the given panels, not the saved stack
        self.dirty = False
        self.as_numpy = False  # results="numpy": items materialise as float64 ndarrays
        self.pending = None  # a deferred status-flag check (RSA_B200_CHECK=deferred)

    def __setitem__(self, i, value):
        list.__setitem__(self, i, value)
        self.dirty = True

    def _get(self, d: int):
        item = list.__getitem__(self, d)
        if item is None:
            scale = None if self.rowscale is None else self.rowscale[d]
            item = engine.normalized_panel(self.stacked[d], scale, torch.float32 if scale is not None else
                                           self.stacked.dtype)
            if self.as_numpy:
                item = _host(item)
            list.__setitem__(self, d, item)
        return item

    def __getitem__(self, i):
        idx = range(len(self))[i]
        return [self._get(d) for d in idx] if isinstance(i, slice) else self._get(idx)

    def __iter__(self):
        for d in range(len(self)):
            yield self._get(d)


class StreamPanels(ProbPanels):
    """The ``probs`` list of a stream-mode forward (``mode="stream"``).

    No panel exists: the forward kept O and two fp32 numbers per query row (the
    reference point m and the row scale r of the factored panel P = r * 2^(s' - m)),
    O(B*Z*c) per rank instead of O(B*Z*c*L).  Indexing recomputes rank d's probabilities
    on the device (``engine.stream_panel``: the same products and exp2 as the panel
    forward, so the values are those ``mode="panel"`` would return) -- the reference's
    ``probs`` contract holds, but memory is only spent on the panels a caller looks at.
    Passing the object back to ``ring_attention_backward`` runs the stream-mode backward,
    which recomputes each probability tile on chip and never materialises a panel.
    """

    def __init__(self, q, k, v, outputs, rowscale, rowmax, inputs, panel_shape):
        list.__init__(self, [None] * q.shape[0])
        self.stacked = None
        self.q, self.k, self.v = q, k, v
        self.outputs, self.rowscale, self.rowmax = outputs, rowscale, rowmax
        self.panel_shape = tuple(panel_shape)
        self.inputs = inputs
        self.dirty = False
        self.as_numpy = False
        self.pending = None

    def _get(self, d: int):
        item = list.__getitem__(self, d)
        if item is None:
            item = engine.stream_panel(self.q, self.k, self.v, self.rowmax, self.rowscale, d)
            if self.as_numpy:
                item = _host(item)
            list.__setitem__(self, d, item)
        return item


def _panels(p: ProbPanels, rmode: str) -> ProbPanels:
    p.as_numpy = rmode == "numpy"
    return p


def _shape_of(x) -> tuple:
    return tuple(x.shape) if hasattr(x, "shape") else tuple(__import__("numpy").asarray(x).shape)


def _check_chunks(name: str, chunks, cfg: AttentionConfig, expect: tuple) -> list:
    """ringseq/ring_attention.py:106-117: count and shape of the per-rank chunks."""
    chunks = chunks if isinstance(chunks, list) else list(chunks)  # keep ProbPanels intact
    if len(chunks) != cfg.num_devices:
        raise ShapeError(f"{name}: got {len(chunks)} chunks for {cfg.num_devices} devices")
    if isinstance(chunks, ProbPanels) and not chunks.dirty:  # shape check without materialising the panels
        if chunks.panel_shape != expect:
            raise ShapeError(f"{name}[0] has shape {chunks.panel_shape}, expected {expect}")
        return chunks
    for i, c in enumerate(chunks):
        if _shape_of(c) != expect:
            raise ShapeError(f"{name}[{i}] has shape {_shape_of(c)}, expected {expect}")
    return chunks


def _device_of(*lists):
    for lst in lists:
        if isinstance(lst, ProbPanels):  # never materialise the panels just to find the device
            ref = lst.stacked if lst.stacked is not None else lst.outputs
            if ref.is_cuda:
                return ref.device
            continue
        for x in lst:
            if isinstance(x, torch.Tensor) and x.is_cuda:
                return x.device
    return ops.default_device()


def _stack(chunks: list, device) -> torch.Tensor:
    """Stack per-rank chunks into one contiguous bf16 [N][...] device tensor.

    bf16 torch chunks in pinned host memory are copied asynchronously on the
    current stream; a single device chunk that is already bf16 and contiguous
    is used in place (a view, no copy)."""
    if (isinstance(chunks, ProbPanels) and not chunks.dirty and chunks.stacked is not None
            and chunks.stacked.device == device):
        return chunks.stacked
    first = chunks[0]
    if (len(chunks) == 1 and isinstance(first, torch.Tensor) and first.device == device
            and first.dtype == torch.bfloat16 and first.is_contiguous()):
        return first.unsqueeze(0)
    out = torch.empty((len(chunks),) + _shape_of(first), dtype=torch.bfloat16, device=device)
    for d, c in enumerate(chunks):
        if isinstance(c, torch.Tensor) and c.dtype == torch.bfloat16:
            out[d].copy_(c, non_blocking=c.device.type == "cpu" and c.is_pinned())
        else:
            out[d].copy_(ops.to_device(c, device))
    return out


def _chunk_key(chunks):
    """Identity of a list of torch chunks (objects + in-place version counters), or None."""
    if not all(isinstance(c, torch.Tensor) for c in chunks):
        return None
    return tuple((c, c._version) for c in chunks)


def _same_tensor(k: torch.Tensor, ver: int, c) -> bool:
    """c is k, or a view of the same memory with the same layout, unmodified since
    (views share the version counter of their base, so an in-place write shows)."""
    if c is k:
        return c._version == ver
    return (isinstance(c, torch.Tensor) and c.device == k.device and c.dtype == k.dtype and c.shape == k.shape
            and c.stride() == k.stride() and c.data_ptr() == k.data_ptr() and c._version == ver)


def _same_chunks(key, chunks) -> bool:
    return key is not None and len(key) == len(chunks) and all(
        _same_tensor(k, ver, c) for (k, ver), c in zip(key, chunks))


def _chunk_elements(cfg: AttentionConfig) -> int:
    return cfg.batch_size * cfg.num_heads * cfg.chunk_len * cfg.head_size


CHECK_ENV_VAR = "RSA_B200_CHECK"


def _deferred_checks() -> bool:
    """$RSA_B200_CHECK=deferred: the forward does not wait for its status flag (a host sync
    per call); the flag travels to pinned host memory behind an event and is read by the
    backward that consumes the forward's panels (or by ``check_forward``).  Default "sync":
    the forward raises NumericError itself, as ringseq/tensor_ops.py:80-81 does."""
    mode = os.environ.get(CHECK_ENV_VAR, "sync")
    if mode not in ("sync", "deferred"):
        raise ValueError(f"${CHECK_ENV_VAR} must be 'sync' or 'deferred', got {mode!r}")
    return mode == "deferred"


class _PendingCheck:
    """A forward's status flag, copied to pinned host memory behind an event on its stream."""

    def __init__(self, flag: torch.Tensor):
        self.host = torch.empty(1, dtype=torch.int32, pin_memory=True)
        self.host.copy_(flag, non_blocking=True)
        self.event = torch.cuda.Event()
        self.event.record()

    def raise_if_bad(self) -> None:
        self.event.synchronize()  # waits for this forward only, not the whole device
        status = int(self.host[0])
        if status & 1:
            raise NumericError("softmax_rows requires finite inputs")
        if status & 2:
            raise NumericError("a row exceeded the single-pass panel's headroom in a forward with deferred checks; "
                               f"rerun it with ${CHECK_ENV_VAR}=sync")


def check_forward(fwd) -> None:
    """Raise the NumericError a forward with deferred checks found (no-op otherwise)."""
    pending = getattr(fwd.probs, "pending", None)
    if pending is not None:
        pending.raise_if_bad()


def _forward_checked(q, k, v, path: str) -> engine.Forward:
    """engine.forward plus the host-side status check.

    Flag bit 0: a non-finite score (NumericError, as ringseq/tensor_ops.py:80-81).
    Flag bit 1: the single-pass factored kernel found a row whose max lies more
    than 2^96 above its first key tile's max; the two-pass normalised kernel
    recomputes the whole launch (never seen for real attention logits).
    """
    res = engine.forward(q, k, v, path=path)
    if _deferred_checks():
        return res
    status = int(res.flag.item())
    if status == 2:
        res.flag.zero_()
        res = engine.forward(q, k, v, path=path, factored=False, flag=res.flag, out=res.out, panel=res.panel)
        status = int(res.flag.item())
    if status:
        raise NumericError("softmax_rows requires finite inputs")
    return res


def forward_ledger(cfg: AttentionConfig) -> CommLedger:
    """Keys then values circulate N-1 hops each (ringseq/ring_attention.py:124-130)."""
    n = cfg.num_devices
    ledger = CommLedger(n)
    if n > 1:
        for d in range(n):
            ledger.record_ring_send(d, 2 * (n - 1) * _chunk_elements(cfg))
    return ledger


def backward_ledger(cfg: AttentionConfig) -> CommLedger:
    """One V and one K circulation plus two all-reduces of (B, Z, L, A) partials
    (ringseq/ring_attention.py:150-156, 206-207)."""
    n = cfg.num_devices
    ledger = CommLedger(n)
    if n > 1:
        full = cfg.batch_size * cfg.num_heads * cfg.seq_len * cfg.head_size
        for d in range(n):
            ledger.record_ring_send(d, 2 * (n - 1) * _chunk_elements(cfg))
            ledger.record_allreduce(d, full)
            ledger.record_allreduce(d, full)
    return ledger


def _stream_checked(q, k, v) -> engine.StreamForward:
    """engine.forward_stream plus the status check (bit 0 NumericError; bit 1 reruns the
    launch on every row's true maximum, as _forward_checked does for the panel)."""
    res = engine.forward_stream(q, k, v)
    if _deferred_checks():
        return res
    status = int(res.flag.item())
    if status == 2:
        res.flag.zero_()
        res = engine.forward_stream(q, k, v, flag=res.flag, out=res.out, rowscale=res.rowscale, rowmax=res.rowmax,
                                    exact=True)
        status = int(res.flag.item())
    if status:
        raise NumericError("softmax_rows requires finite inputs")
    return res


MODES = ("panel", "stream")


def ring_attention_forward(q_chunks, k_chunks, v_chunks, cfg: AttentionConfig, *, executor: str | None = None,
                           path: str = "auto", mode: str = "panel", results: str | None = None) -> RingAttentionForward:
    """Distributed attention forward over per-rank (B, Z, L/N, A) chunks.

    ringseq/ring_attention.py:124-147.  ``path`` ('auto' | 'fused' | 'staged')
    selects the device implementation; both compute the same protocol.

    ``mode="panel"`` (default) saves the reference's probability panels (B, Z, L/N, L)
    per rank, so memory grows as L^2/N.  ``mode="stream"`` saves O plus two numbers per
    query row; ``probs`` is then a ``StreamPanels`` list that recomputes any rank's
    panel on access, and the backward recomputes probability tiles on chip -- memory
    grows as L/N, so the trainable length grows linearly with the rank count.

    ``results="numpy"`` (or $RSA_B200_RESULTS=numpy) returns float64 ndarrays, as the
    reference does; the default returns CUDA bf16 tensors (no host round trip).
    """
    rmode = _results_mode(results)
    if mode not in MODES:
        raise ValueError(f"unknown mode {mode!r}; expected one of {MODES}")
    resolve_executor(executor)
    shape = cfg.chunk_shape()
    q_chunks = _check_chunks("q_chunks", q_chunks, cfg, shape)
    k_chunks = _check_chunks("k_chunks", k_chunks, cfg, shape)
    v_chunks = _check_chunks("v_chunks", v_chunks, cfg, shape)
    dev = _device_of(q_chunks, k_chunks, v_chunks)
    q, k, v = (_stack(x, dev) for x in (q_chunks, k_chunks, v_chunks))
    saved = [(_chunk_key(c), t) for c, t in ((q_chunks, q), (k_chunks, k), (v_chunks, v))]
    if mode == "stream":
        if not engine.stream_supported(cfg.num_devices, cfg.batch_size, cfg.num_heads, cfg.chunk_len,
                                       cfg.head_size):
            raise ShapeError(f"stream mode needs head_size 64 and chunk_len % 8 == 0 (got {cfg.head_size}, "
                             f"{cfg.chunk_len})")
        res = _stream_checked(q, k, v)
        probs = StreamPanels(q, k, v, res.out, res.rowscale, res.rowmax, saved, cfg.panel_shape())
        probs.as_numpy = rmode == "numpy"
        probs.pending = _PendingCheck(res.flag) if _deferred_checks() else None
        return RingAttentionForward(outputs=_out_list(res.out, cfg.num_devices, rmode), probs=probs,
                                    ledger=forward_ledger(cfg))
    out, panel, rowscale, flag = _forward_checked(q, k, v, path)
    probs = _panels(ProbPanels(panel, out, rowscale, saved), rmode)
    probs.pending = _PendingCheck(flag) if _deferred_checks() else None
    return RingAttentionForward(
        outputs=_out_list(out, cfg.num_devices, rmode),
        probs=probs,
        ledger=forward_ledger(cfg),
    )


def ring_attention_backward(q_chunks, k_chunks, v_chunks, probs, grad_chunks, cfg: AttentionConfig, *,
                            executor: str | None = None, path: str = "auto",
                            results: str | None = None) -> RingAttentionBackward:
    """Gradients of ring_attention_forward w.r.t. the q/k/v chunks.

    ringseq/ring_attention.py:150-217.  ``probs`` are the panels saved by the
    forward (StateError when missing, ShapeError when mis-shaped).
    """
    resolve_executor(executor)
    rmode = _results_mode(results)
    shape = cfg.chunk_shape()
    q_chunks = _check_chunks("q_chunks", q_chunks, cfg, shape)
    k_chunks = _check_chunks("k_chunks", k_chunks, cfg, shape)
    v_chunks = _check_chunks("v_chunks", v_chunks, cfg, shape)
    grad_chunks = _check_chunks("grad_chunks", grad_chunks, cfg, shape)
    if probs is None:
        raise StateError("ring_attention_backward needs the probability panels saved by ring_attention_forward")
    probs = _check_chunks("probs", probs, cfg, cfg.panel_shape())
    if getattr(probs, "pending", None) is not None:  # the forward's deferred status check
        probs.pending.raise_if_bad()
    dev = _device_of(q_chunks, k_chunks, v_chunks, grad_chunks, probs)
    saved = probs.inputs if isinstance(probs, ProbPanels) else []

    def stack_or_saved(chunks, i):
        if i < len(saved):
            key, t = saved[i]
            if t.device == dev and _same_chunks(key, chunks):
                return t, True
            if key is None and t.device == dev:  # NumPy chunks: identity unknown, compare values
                up = _stack(chunks, dev)
                return (t, True) if torch.equal(up, t) else (up, False)
        return _stack(chunks, dev), False

    (q, q_saved), (k, k_saved), (v, v_saved) = (stack_or_saved(x, i)
                                                 for i, x in enumerate((q_chunks, k_chunks, v_chunks)))
    g = _stack(grad_chunks, dev)
    n = cfg.num_devices
    if isinstance(probs, StreamPanels) and not probs.dirty and q_saved and k_saved and v_saved:
        # the forward's own state: recompute probability tiles on chip, no panel anywhere
        dq, dk, dv = engine.backward_stream(q, k, v, g, probs.outputs, probs.rowscale, probs.rowmax)
        return RingAttentionBackward(grad_q=_out_list(dq, n, rmode), grad_k=_out_list(dk, n, rmode),
                                     grad_v=_out_list(dv, n, rmode), ledger=backward_ledger(cfg))
    panel = _stack(probs, dev)
    own = isinstance(probs, ProbPanels) and panel is probs.stacked
    # the forward's O = P V is reused for D = rowsum(dP * P) = rowsum(dO * O) only when the
    # caller passes the forward's own, unmodified panels AND values; otherwise D follows the
    # given arguments (O recomputed from them), as the reference computes it
    outputs = probs.outputs if own and v_saved else None
    rowscale = probs.rowscale if own else None
    if outputs is not None and (outputs.shape != q.shape or outputs.device != dev):
        outputs = None
    dq, dk, dv = engine.backward(q, k, v, panel, g, outputs=outputs, rowscale=rowscale, path=path)
    return RingAttentionBackward(
        grad_q=_out_list(dq, n, rmode),
        grad_k=_out_list(dk, n, rmode),
        grad_v=_out_list(dv, n, rmode),
        ledger=backward_ledger(cfg),
    )


def _layer_weights(weights, cfg: AttentionConfig, dev):
    h, za = cfg.hidden_size, cfg.num_heads * cfg.head_size
    for name, expect_w in (("wq", (h, za)), ("wk", (h, za)), ("wv", (h, za)), ("wo", (za, h))):
        if _shape_of(getattr(weights, name)) != expect_w:
            raise ShapeError(f"{name} has shape {_shape_of(getattr(weights, name))}, expected {expect_w}")
    return [ops.to_device(getattr(weights, n), dev) for n in ("wq", "wk", "wv", "wo")]


def _split_heads(y, n, b, c, z, a):
    """[N][B][c][Z*A] -> [N][B][Z][c][A] (split_heads per rank, ringseq/tensor_ops.py:93-110)."""
    return y.view(n, b, c, z, a).permute(0, 1, 3, 2, 4).contiguous()


def _merge_heads(t):
    """[N][B][Z][c][A] -> [N][B][c][Z*A] (merge_heads per rank, ringseq/tensor_ops.py:113-119)."""
    n, b, z, c, a = t.shape
    return t.permute(0, 1, 3, 2, 4).reshape(n, b, c, z * a)


def _layer_forward(x, ws, cfg: AttentionConfig, path: str):
    n, b, c, z, a = cfg.num_devices, cfg.batch_size, cfg.chunk_len, cfg.num_heads, cfg.head_size
    q, k, v = (_split_heads(ops.matmul(x, w, out_dtype=torch.bfloat16), n, b, c, z, a) for w in ws[:3])
    return q, k, v, _forward_checked(q, k, v, path)


def sequence_parallel_attention(x_chunks, weights, cfg: AttentionConfig, *, executor: str | None = None,
                                path: str = "auto", results: str | None = None):
    """Multi-head attention layer on sequence-partitioned (B, L/N, H) inputs.

    ringseq/ring_attention.py:220-241: replicated projections are local
    GEMMs, only the attention stages ring.  Returns (per-rank outputs, ledger).
    """
    resolve_executor(executor)
    expect = (cfg.batch_size, cfg.chunk_len, cfg.hidden_size)
    x_chunks = _check_chunks("x_chunks", x_chunks, cfg, expect)
    dev = _device_of(x_chunks)
    ws = _layer_weights(weights, cfg, dev)
    x = _stack(x_chunks, dev)  # [N][B][c][H]
    _, _, _, res = _layer_forward(x, ws, cfg, path)
    y = ops.matmul(_merge_heads(res.out), ws[3])
    return _out_list(y, cfg.num_devices, _results_mode(results)), forward_ledger(cfg)


def sequence_parallel_attention_backward(x_chunks, weights, cfg: AttentionConfig, grad_chunks, *,
                                         executor: str | None = None, path: str = "auto"):
    """Gradients of ``sequence_parallel_attention`` w.r.t. its inputs and weights.

    The reference ships only the layer's forward (ringseq/ring_attention.py:220-241);
    this follows its dense oracle ``multi_head_backward`` (ringseq/reference.py:133-174)
    with the attention stages replaced by the ring backward.  Returns
    ``(grad_x chunks (B, L/N, H) bf16, AttentionWeights(grad_wq, grad_wk, grad_wv,
    grad_wo) fp32, ledger)``.  Weight gradients are sums over every rank's rows;
    on N devices that is one all-reduce of the four replicated matrices, which the
    ledger charges with the reference's all-reduce convention
    (ringseq/cluster.py:320-359) on top of the ring backward's traffic.
    """
    from .weights import AttentionWeights

    resolve_executor(executor)
    expect = (cfg.batch_size, cfg.chunk_len, cfg.hidden_size)
    x_chunks = _check_chunks("x_chunks", x_chunks, cfg, expect)
    grad_chunks = _check_chunks("grad_chunks", grad_chunks, cfg, expect)
    dev = _device_of(x_chunks, grad_chunks)
    ws = _layer_weights(weights, cfg, dev)
    wq, wk, wv, wo = ws
    n, b, c, z, a, h = (cfg.num_devices, cfg.batch_size, cfg.chunk_len, cfg.num_heads, cfg.head_size,
                        cfg.hidden_size)
    za = z * a
    x = _stack(x_chunks, dev)     # [N][B][c][H]
    g = _stack(grad_chunks, dev)  # [N][B][c][H]
    q, k, v, res = _layer_forward(x, ws, cfg, path)
    # output projection (ringseq/reference.py:155-160): rows of every rank folded together
    o2 = _merge_heads(res.out).reshape(-1, za)
    g2 = g.reshape(-1, h)
    grad_wo = ops.matmul(o2.transpose(0, 1), g2)
    grad_o = _split_heads(ops.matmul(g, wo.transpose(0, 1), out_dtype=torch.bfloat16), n, b, c, z, a)
    dq, dk, dv = engine.backward(q, k, v, res.panel, grad_o, outputs=res.out, rowscale=res.rowscale, path=path)
    # input projections (ringseq/reference.py:162-173)
    x2 = x.reshape(-1, h)
    gq2, gk2, gv2 = (_merge_heads(t).reshape(-1, za) for t in (dq, dk, dv))
    grad_wq, grad_wk, grad_wv = (ops.matmul(x2.transpose(0, 1), t) for t in (gq2, gk2, gv2))
    gx = ops.matmul(gq2, wq.transpose(0, 1))
    ops.matmul(gk2, wk.transpose(0, 1), out=gx, accumulate=True)
    ops.matmul(gv2, wv.transpose(0, 1), out=gx, accumulate=True)
    gx = gx.to(torch.bfloat16).view(n, b, c, h)
    ledger = backward_ledger(cfg)
    if n > 1:
        for d in range(n):
            ledger.record_allreduce(d, 2 * h * za + za * h + h * za)  # wq, wk, wv, wo gradients
    return [gx[d] for d in range(n)], AttentionWeights(grad_wq, grad_wk, grad_wv, grad_wo), ledger


def _mlp_weights(weights, h: int, dev):
    up_s, down_s = _shape_of(weights.up), _shape_of(weights.down)
    if len(up_s) != 2 or up_s[0] != h or down_s != (up_s[1], h):
        raise ShapeError(f"mlp weights {up_s} / {down_s} do not match input feature size {h}")
    return ops.to_device(weights.up, dev), ops.to_device(weights.down, dev)


def _chunks_of_rows(x_chunks):
    x_chunks = x_chunks if isinstance(x_chunks, list) else list(x_chunks)
    if not x_chunks:
        raise ShapeError("x_chunks: need at least one chunk")
    shape = _shape_of(x_chunks[0])
    for i, c in enumerate(x_chunks):
        if _shape_of(c) != shape:
            raise ShapeError(f"x_chunks[{i}] has shape {_shape_of(c)}, expected {shape}")
    return x_chunks, shape


def sequence_parallel_mlp(x_chunks, weights, *, executor: str | None = None):
    """Feed-forward block on sequence-partitioned inputs (ringseq/ring_attention.py:244-256).

    gelu(x @ up) @ down per rank (ringseq/reference.py:177-185); token rows never
    interact, so nothing is communicated and the ledger stays at zero.  The GEMMs are
    rsa_gemm (tcgen05), the activation rsa_gelu (exact erf form).  Returns
    (per-rank outputs (B, L/N, H) bf16, ledger).
    """
    resolve_executor(executor)
    x_chunks, shape = _chunks_of_rows(x_chunks)
    dev = _device_of(x_chunks)
    up, down = _mlp_weights(weights, shape[-1], dev)
    x = _stack(x_chunks, dev)
    a = ops.gelu(ops.matmul(x, up), out_dtype=torch.bfloat16)
    y = ops.matmul(a, down, out_dtype=torch.bfloat16)
    return [y[d] for d in range(len(x_chunks))], CommLedger(len(x_chunks))


def sequence_parallel_mlp_backward(x_chunks, weights, grad_chunks, *, executor: str | None = None):
    """Gradients of ``sequence_parallel_mlp`` (the reference ships the forward only).

    Chain rule through gelu(x @ up) @ down with the pre-activation recomputed:
    grad_down = a^T dy, dh = (dy down^T) * gelu'(h), grad_up = x^T dh, grad_x = dh up^T.
    Weight gradients sum every rank's rows (one all-reduce of the replicated weights on N
    devices, charged with the reference's all-reduce convention, ringseq/cluster.py:320-359).
    Returns (grad_x chunks bf16, MlpWeights(grad_up, grad_down) fp32, ledger).
    """
    from .weights import MlpWeights

    resolve_executor(executor)
    x_chunks, shape = _chunks_of_rows(x_chunks)
    grad_chunks, gshape = _chunks_of_rows(grad_chunks)
    if gshape != shape or len(grad_chunks) != len(x_chunks):
        raise ShapeError(f"grad_chunks shape {gshape} x {len(grad_chunks)} does not match x_chunks {shape}")
    n, h = len(x_chunks), shape[-1]
    dev = _device_of(x_chunks, grad_chunks)
    up, down = _mlp_weights(weights, h, dev)
    inner = up.shape[1]
    x = _stack(x_chunks, dev)
    g = _stack(grad_chunks, dev)
    hpre = ops.matmul(x, up)  # fp32 pre-activation
    a = ops.gelu(hpre, out_dtype=torch.bfloat16)
    grad_down = ops.matmul(a.reshape(-1, inner).transpose(0, 1), g.reshape(-1, h))
    da = ops.matmul(g, down.transpose(0, 1))  # fp32
    dh = ops.gelu_backward(hpre, da, out_dtype=torch.bfloat16)
    grad_up = ops.matmul(x.reshape(-1, h).transpose(0, 1), dh.reshape(-1, inner))
    gx = ops.matmul(dh, up.transpose(0, 1), out_dtype=torch.bfloat16)
    ledger = CommLedger(n)
    if n > 1:
        for d in range(n):
            ledger.record_allreduce(d, 2 * h * inner)
    return [gx[d] for d in range(n)], MlpWeights(grad_up, grad_down), ledger

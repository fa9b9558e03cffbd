"""RSA across real ranks: one process per GPU, rings over torch.distributed (NCCL).

This is the multi-GPU form of ringseq/ring_attention.py:124-217.  Rank d
holds only its own (B, Z, c, A) chunks; keys and values travel d -> d+1 by
NCCL send/recv (``batch_isend_irecv``), exactly the reference's ring
(ringseq/ring_attention.py:67-79, ringseq/cluster.py:293-318), and the
per-hop arithmetic runs in the same sm_100a kernels the single-GPU path
uses, launched with ``n_org = 1`` for the origin that just arrived.

Schedule per rank (h = hop, origin j = (d - h) mod N):

  forward   K ring: hop h+1 is posted before hop h's rsa_fwd_stats runs, so
            the transfer overlaps the kernel; received chunks land directly
            in a per-origin slot (no copies).  V ring: rsa_fwd_probs_pv per
            hop -- it needs K_j again, taken from the slots filled by the K
            ring (the reference discards them; keeping them costs L*A per
            head and no extra communication).
  backward  V ring: rsa_bwd_dkdv per hop writes this rank's dK/dV
            contribution for origin j into full-length fp32 partials and the
            dS panel block j.  K ring: rsa_bwd_dq accumulates dQ.  The two
            partials are then summed across ranks: ``reduce_scatter`` by
            default (each rank receives only its own rows -- half the bytes
            of the reference's all-reduce + slice), ``all_reduce`` in
            ``mode="paper"``.

The ledger charges what the reference charges (element counts, all-reduce
convention); ``wire_bytes`` records the bytes actually sent.

The per-hop kernels are injected (``HopKernels``) so the schedule can be
tested on CPU with the gloo backend (tests/test_distributed_gloo.py) using a
test-only implementation; the product path always uses ``CudaHopKernels``.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field

import torch
import torch.distributed as dist

from .cluster import CommLedger

__all__ = ["SpmdRing", "PeerRing", "CudaHopKernels", "RingContext", "bench_main"]


def _acc_dtype(t: torch.Tensor) -> torch.dtype:
    """Cross-hop accumulators: fp32 for bf16 chunks, else the chunk dtype."""
    return torch.float32 if t.dtype == torch.bfloat16 else t.dtype


class CudaHopKernels:
    """Per-hop launches of the fused kernels (librsa_b200.so)."""

    def __init__(self):
        from . import engine
        from ._native import BF16, RsaGeom, check, lib

        self.engine, self.BF16, self.RsaGeom, self.check, self.lib = engine, BF16, RsaGeom, check, lib

    def _g(self, q, seq, origin):
        _, b, z, c, a = q.shape
        return self.RsaGeom(1, b, z, c, a, seq, origin, 1, 1.0 / math.sqrt(a))

    def _st(self, t):
        return torch.cuda.current_stream(t.device).cuda_stream

    def new_stats(self, q, n):
        _, b, z, c, _ = q.shape
        return torch.empty((n * b * z * c * 2,), dtype=torch.float32, device=q.device)

    def stats(self, q, k_j, origin, seq, stats, flag):
        g = self._g(q, seq, origin)
        v = self.engine._view
        self.check(self.lib().rsa_fwd_stats(ctypes.byref(g), v(q), v(k_j), stats.data_ptr(), origin,
                                            flag.data_ptr(), self._st(q)), "rsa_fwd_stats")

    def probs_pv(self, q, k_j, v_j, origin, seq, stats, n_slots, panel, o_acc, accumulate, o_out):
        g = self._g(q, seq, origin)
        v = self.engine._view
        self.check(self.lib().rsa_fwd_probs_pv(ctypes.byref(g), v(q), v(k_j), v(v_j), stats.data_ptr(), n_slots,
                                               v(panel), v(o_acc), int(accumulate), v(o_out), self._st(q)),
                   "rsa_fwd_probs_pv")

    def rowdot(self, grad, out):
        from . import tensor_ops

        return tensor_ops.rowdot(grad, out)

    def dkdv(self, q, v_j, grad, panel, dvec, origin, seq, dk_j, dv_j):
        g = self._g(q, seq, origin)
        v = self.engine._view
        self.check(self.lib().rsa_bwd_dkdv(ctypes.byref(g), v(q), v(v_j), v(grad), v(panel), dvec.data_ptr(),
                                           v(dk_j), v(dv_j), 0, 0, self._st(q)), "rsa_bwd_dkdv")

    def project_pair(self, e_cols, k, f_cols, v):
        """[E_d K_d ; F_d V_d] as one fp32 [2][B][Z][K][A] buffer (tcgen05 GEMMs)."""
        from . import tensor_ops

        b, z, _, a = k.shape
        out = torch.empty((2, b, z, e_cols.shape[0], a), dtype=torch.float32, device=k.device)
        tensor_ops.matmul(e_cols, k, out=out[0])
        tensor_ops.matmul(f_cols, v, out=out[1])
        return out

    def low_rank_attention(self, q, k_low, v_low):
        """softmax(Q K'^T / sqrt(A)) V' with rows fully local."""
        from . import tensor_ops

        scores = tensor_ops.matmul(q, k_low.to(torch.bfloat16).transpose(-1, -2))
        probs = tensor_ops.softmax_rows(scores, scale=1.0 / math.sqrt(q.shape[-1]), out_dtype=torch.bfloat16)
        return tensor_ops.matmul(probs, v_low.to(torch.bfloat16), out_dtype=torch.bfloat16)

    def dq(self, grad, k_j, v_j, panel, dvec, origin, seq, dq_acc, accumulate, dq_out):
        g = self._g(grad, seq, origin)
        v = self.engine._view
        self.check(self.lib().rsa_bwd_dq(ctypes.byref(g), v(grad), v(k_j), v(v_j), v(panel), dvec.data_ptr(),
                                         v(dq_acc), int(accumulate), v(dq_out), self._st(grad)), "rsa_bwd_dq")


@dataclass
class RingContext:
    """What the forward keeps for the backward (the reference keeps only probs)."""

    q: torch.Tensor
    k_slots: torch.Tensor
    panel: torch.Tensor
    out: torch.Tensor
    v_local: torch.Tensor
    extra: dict = field(default_factory=dict)


class SpmdRing:
    """One rank's view of the RSA ring over a torch.distributed process group."""

    def __init__(self, group=None, kernels=None, mode: str = "reduce_scatter", overlap: bool = True,
                 transport: str = "device"):
        """``transport="host"`` stages every hop and reduction through host memory, for
        process groups whose backend cannot move device tensors point to point (gloo);
        the default sends the device buffers themselves (NCCL over NVLink)."""
        if mode not in ("reduce_scatter", "paper"):
            raise ValueError(f"unknown mode {mode!r}")
        if transport not in ("device", "host"):
            raise ValueError(f"unknown transport {transport!r}")
        self.host_staged = transport == "host"
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.kernels = CudaHopKernels() if kernels is None else kernels  # False: communication only
        self.mode = mode
        self.overlap = overlap
        self.ledger = CommLedger(self.world)

    # ---- communication -------------------------------------------------

    def _post(self, send: torch.Tensor, recv: torch.Tensor):
        """Post one ring hop (send to rank+1, receive from rank-1); returns works."""
        n = self.world
        nxt = dist.get_global_rank(self.group, (self.rank + 1) % n) if self.group else (self.rank + 1) % n
        prv = dist.get_global_rank(self.group, (self.rank - 1) % n) if self.group else (self.rank - 1) % n
        self.ledger.record_ring_send(self.rank, send.numel(), send.numel() * send.element_size())
        if self.host_staged and send.is_cuda:
            s_h, r_h = send.cpu(), torch.empty(recv.shape, dtype=recv.dtype)
            ops = [dist.P2POp(dist.isend, s_h, nxt, self.group), dist.P2POp(dist.irecv, r_h, prv, self.group)]
            return (dist.batch_isend_irecv(ops), recv, r_h, s_h)
        ops = [dist.P2POp(dist.isend, send, nxt, self.group), dist.P2POp(dist.irecv, recv, prv, self.group)]
        return (dist.batch_isend_irecv(ops), None, None, None)

    @staticmethod
    def _wait(pending):
        if not pending:
            return
        works, recv, r_h, _ = pending
        for w in works:
            w.wait()
        if recv is not None:
            recv.copy_(r_h)

    def _circulate(self, slots: torch.Tensor, on_arrival):
        """Run the ring over per-origin ``slots`` ([N][...]); slot d must hold
        the local chunk.  ``on_arrival(h, j)`` runs once slot j is valid."""
        n, d = self.world, self.rank
        pending = self._post(slots[d], slots[(d - 1) % n]) if n > 1 and self.overlap else None
        for h in range(n):
            j = (d - h) % n
            if h > 0:
                if not self.overlap:
                    pending = self._post(slots[(j + 1) % n], slots[j])
                self._wait(pending)
                pending = None
                if self.overlap and h + 1 < n:
                    pending = self._post(slots[j], slots[(j - 1) % n])
            on_arrival(h, j)
        self._wait(pending)

    # ---- protocol --------------------------------------------------------

    def forward(self, q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, flag: torch.Tensor | None = None):
        """q/k/v: this rank's [1][B][Z][c][A] chunks.  Returns (out, ctx)."""
        kern = self.kernels
        n, d = self.world, self.rank
        _, b, z, c, a = q.shape
        seq = n * c
        dev = q.device
        if flag is None:
            flag = torch.zeros(1, dtype=torch.int32, device=dev)
        k_slots = torch.empty((n, b, z, c, a), dtype=k.dtype, device=dev)
        k_slots[d].copy_(k[0])
        stats = kern.new_stats(q, n)
        self._circulate(k_slots, lambda h, j: kern.stats(q, k_slots[j:j + 1], j, seq, stats, flag))
        v_slots = torch.empty((n, b, z, c, a), dtype=v.dtype, device=dev)
        v_slots[d].copy_(v[0])
        panel = torch.empty((1, b, z, c, seq), dtype=q.dtype, device=dev)
        o_acc = torch.empty((1, b, z, c, a), dtype=_acc_dtype(q), device=dev)
        out = torch.empty((1, b, z, c, a), dtype=q.dtype, device=dev)

        def pv(h, j):
            kern.probs_pv(q, k_slots[j:j + 1], v_slots[j:j + 1], j, seq, stats, n, panel, o_acc, h > 0,
                          out if h == n - 1 else None)

        self._circulate(v_slots, pv)
        return out, RingContext(q=q, k_slots=k_slots, panel=panel, out=out, v_local=v, extra={"flag": flag})

    def backward(self, ctx: RingContext, grad: torch.Tensor):
        """grad: this rank's [1][B][Z][c][A] dO.  Returns (dq, dk, dv) chunks."""
        kern = self.kernels
        n, d = self.world, self.rank
        _, b, z, c, a = grad.shape
        seq = n * c
        dev = grad.device
        dvec = kern.rowdot(grad, ctx.out)
        dk_part = torch.empty((n, b, z, c, a), dtype=_acc_dtype(grad), device=dev)
        dv_part = torch.empty_like(dk_part)
        v_slots = torch.empty((n, b, z, c, a), dtype=ctx.v_local.dtype, device=dev)
        v_slots[d].copy_(ctx.v_local[0])
        self._circulate(v_slots, lambda h, j: kern.dkdv(ctx.q, v_slots[j:j + 1], grad, ctx.panel, dvec, j, seq,
                                                        dk_part[j:j + 1], dv_part[j:j + 1]))
        # K ring (the reference re-circulates keys: ringseq/ring_attention.py:192-196).  dS for origin j is
        # recomputed from P, dO V_j^T and D with V_j from the V ring's slots, so no dS panel is kept.
        k_slots = torch.empty_like(ctx.k_slots)
        k_slots[d].copy_(ctx.k_slots[d])
        dq_acc = torch.empty((1, b, z, c, a), dtype=_acc_dtype(grad), device=dev)
        dq = torch.empty((1, b, z, c, a), dtype=grad.dtype, device=dev)
        self._circulate(k_slots, lambda h, j: kern.dq(grad, k_slots[j:j + 1], v_slots[j:j + 1], ctx.panel, dvec, j,
                                                      seq, dq_acc, h > 0, dq if h == n - 1 else None))
        dk = self._reduce(dk_part)
        dv = self._reduce(dv_part)
        return dq, dk.to(grad.dtype), dv.to(grad.dtype)

    def linformer_forward(self, q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, e_cols: torch.Tensor,
                          f_cols: torch.Tensor) -> torch.Tensor:
        """Sequence-sharded Linformer forward (ringseq/sparse_attention.py:74-133).

        q/k/v: this rank's [1][B][Z][c][A] chunks; e_cols/f_cols: this rank's
        (K, c) column blocks of the projections.  The two partial projections
        are summed across ranks with ONE all-reduce of the concatenated
        [K'; V'] buffer (the reference spells it as 2(N-1) ring hops; the
        ledger charges that convention, wire_bytes the all-reduce).
        """
        kern = self.kernels
        n, d = self.world, self.rank
        _, b, z, c, a = q.shape
        kdim = e_cols.shape[0]
        low = kern.project_pair(e_cols, k[0], f_cols, v[0])  # [2][B][Z][K][A] accumulator dtype
        self.ledger.record_ring_send(d, 2 * (n - 1) * b * z * kdim * a)
        if n > 1 and self.host_staged and low.is_cuda:
            host = low.cpu()
            dist.all_reduce(host, group=self.group)
            low.copy_(host)
        elif n > 1:
            dist.all_reduce(low, group=self.group)
            self.ledger.devices[d].wire_bytes += 2 * low.numel() * low.element_size() * (n - 1) // n
        return kern.low_rank_attention(q, low[0], low[1])

    def _reduce(self, part: torch.Tensor) -> torch.Tensor:
        """Sum full-length partials over ranks; return this rank's [1][...] rows."""
        n, d = self.world, self.rank
        self.ledger.record_allreduce(d, part.numel())
        if n == 1:
            return part[d:d + 1]
        use_rs = self.mode == "reduce_scatter" and dist.get_backend(self.group) == "nccl"
        if use_rs:
            out = torch.empty_like(part[0:1])
            dist.reduce_scatter_tensor(out, part, group=self.group)
            self.ledger.devices[d].wire_bytes += part.numel() * part.element_size() * (n - 1) // n
            return out
        if self.host_staged and part.is_cuda:
            host = part.cpu()
            dist.all_reduce(host, group=self.group)
            part.copy_(host)
        else:
            dist.all_reduce(part, group=self.group)
        self.ledger.devices[d].wire_bytes += 2 * part.numel() * part.element_size() * (n - 1) // n
        return part[d:d + 1].clone()


class _CudaBuffer:
    """A raw device allocation seen by torch through ``__cuda_array_interface__``
    (int16 words; viewed as bf16).  The tensor does not own the memory."""

    def __init__(self, ptr: int, shape: tuple):
        self.__cuda_array_interface__ = {"shape": tuple(shape), "typestr": "<i2", "data": (ptr, False),
                                         "version": 3, "strides": None}


class _PeerSlot:
    """One registered K/V buffer: this rank's [2][B][Z][c][A] chunk pair (``rsa_ipc_alloc``)
    and every peer's, mapped with ``rsa_ipc_open`` -- the device pointers a peer kernel
    reads over NVLink."""

    def __init__(self, ptr: int, peer_ptrs: list, local: torch.Tensor, peers: list):
        self.ptr, self.peer_ptrs, self.local, self.peers = ptr, peer_ptrs, local, peers


class PeerRing:
    """Ring-free RSA across the ranks of one NVLink/NVSwitch box.

    Every rank stages its K/V chunk in a registered buffer that all ranks have opened
    through CUDA IPC; one ``rsa_fwd_factored_peer`` launch then reads every origin's
    K/V tiles in place -- TMA loads from the owner's HBM over NVLink inside the kernel's
    pipeline, overlapped with the tensor-core work -- instead of N-1 ring hops with one
    kernel launch each.  The backward is one ``rsa_bwd_fused_peer`` launch (dQ complete,
    fp32 dK/dV partials for every origin) and a reduce-scatter of the partials, as in
    ``SpmdRing``.  The panel is the factored one.  The ledger
    charges the reference's ring convention (ringseq/ring_attention.py:124-217) for the
    same K/V bytes.

    ``forward`` does not read its status flag back; call ``PeerRing.check(ctx)`` (one device
    sync) before trusting a layer's outputs.  This is the correctness-first form: staging
    is fenced by host barriers (buffer free on every rank, then staged on every rank).  Cross-process CUDA IPC events would
    replace them.  The buffers are plain cudaMalloc allocations exported with
    cudaIpcGetMemHandle (``rsa_ipc_*``), outside torch's allocator, so their lifetime is
    exactly ``close()``.
    """

    def __init__(self, group=None, mode: str = "reduce_scatter", transport: str = "device"):
        self.ring = SpmdRing(group, mode=mode, transport=transport, kernels=False)
        self.group, self.rank, self.world = group, self.ring.rank, self.ring.world
        self.ledger = self.ring.ledger
        self._free: dict = {}
        self._all: list = []

    def _barrier(self):
        torch.cuda.synchronize()
        dist.barrier(group=self.group)

    def _slot(self, shape, dtype, dev) -> _PeerSlot:
        from ._native import check, lib

        if dtype != torch.bfloat16:
            raise ValueError(f"PeerRing stages bf16 K/V, got {dtype}")
        key = (tuple(shape), dtype)
        pool = self._free.setdefault(key, [])
        if pool:
            return pool.pop()
        full = (2,) + tuple(shape)
        nbytes = 2 * math.prod(full)
        ptr, handle = ctypes.c_void_p(), ctypes.create_string_buffer(64)
        check(lib().rsa_ipc_alloc(nbytes, ctypes.byref(ptr), handle), "rsa_ipc_alloc")
        handles = [None] * self.world
        dist.all_gather_object(handles, handle.raw, group=self.group)
        ptrs, tensors = [], []
        for j, h in enumerate(handles):
            if j == self.rank:
                p = ptr.value
            else:
                pj = ctypes.c_void_p()
                check(lib().rsa_ipc_open(ctypes.create_string_buffer(h, 64), ctypes.byref(pj)), "rsa_ipc_open")
                p = pj.value
            ptrs.append(p)
            tensors.append(torch.as_tensor(_CudaBuffer(p, full), device=dev).view(torch.bfloat16))
        slot = _PeerSlot(ptr.value, ptrs, tensors[self.rank], tensors)
        self._all.append(slot)
        return slot

    def close(self):
        """Unmap every peer's buffer, then free this rank's own -- in that order on every
        rank, so no process frees memory a peer still maps or reads.  Call it before
        ``destroy_process_group``; the ring is unusable afterwards."""
        from ._native import check, lib

        self._barrier()  # every rank's kernels on the shared buffers have finished
        for s in self._all:
            s.local, s.peers = None, []
            for j, p in enumerate(s.peer_ptrs):
                if j != self.rank:
                    check(lib().rsa_ipc_close(ctypes.c_void_p(p)), "rsa_ipc_close")
        self._barrier()  # every mapping is closed
        for s in self._all:
            check(lib().rsa_ipc_free(ctypes.c_void_p(s.ptr)), "rsa_ipc_free")
        self._all, self._free = [], {}

    def _views(self, slot: _PeerSlot, which: int):
        from .engine import _view

        views = (self.ring_view_type * self.world)()
        for j, t in enumerate(slot.peers):
            views[j] = _view(t[which].unsqueeze(0))
        return views

    @property
    def ring_view_type(self):
        from ._native import RsaView

        return RsaView

    def forward(self, q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, flag: torch.Tensor | None = None):
        """q/k/v: this rank's [1][B][Z][c][A] bf16 chunks.  Returns (out, ctx)."""
        from . import engine
        from ._native import check, lib

        n, d = self.world, self.rank
        _, b, z, c, a = q.shape
        seq = n * c
        dev = q.device
        if flag is None:
            flag = torch.zeros(1, dtype=torch.int32, device=dev)
        slot = self._slot((b, z, c, a), k.dtype, dev)
        self._barrier()  # no rank still reads this buffer (a released slot of an earlier layer)
        slot.local[0].copy_(k[0])
        slot.local[1].copy_(v[0])
        self._barrier()  # every origin is staged
        panel = torch.empty((1, b, z, c, seq), dtype=torch.bfloat16, device=dev)
        out = torch.empty((1, b, z, c, a), dtype=torch.bfloat16, device=dev)
        rowscale = torch.empty((1, b, z, c), dtype=torch.float32, device=dev)
        g = engine._geom(1, b, z, c, a, seq, 0, n)
        check(lib().rsa_fwd_factored_peer(ctypes.byref(g), engine._view(q), self._views(slot, 0), self._views(slot, 1),
                                          engine._view(panel), engine._view(out), rowscale.data_ptr(),
                                          flag.data_ptr(), torch.cuda.current_stream(dev).cuda_stream),
              "rsa_fwd_factored_peer")
        elements = b * z * c * a
        self.ledger.record_ring_send(d, 2 * (n - 1) * elements, 2 * (n - 1) * elements * q.element_size())
        return out, RingContext(q=q, k_slots=None, panel=panel, out=out, v_local=v,
                                extra={"flag": flag, "rowscale": rowscale, "slot": slot})

    @staticmethod
    def check(ctx: RingContext) -> None:
        """Host read of the forward's status flag (a device sync).  Bit 0: a non-finite score
        (``NumericError``, as ringseq/tensor_ops.py:80-81).  Bit 1: a row whose scores exceed
        the single-pass panel's headroom above its first key tile's max.
        The resident engine reruns those layers two-pass; this ring has no two-pass peer
        kernel, so it raises and ``SpmdRing`` is the path for such inputs."""
        from .errors import NumericError

        status = int(ctx.extra["flag"].item())
        if status & 1:
            raise NumericError("softmax_rows requires finite inputs")
        if status & 2:
            raise NumericError("score range exceeds the single-pass panel's headroom; use SpmdRing")

    def backward(self, ctx: RingContext, grad: torch.Tensor):
        """grad: this rank's [1][B][Z][c][A] dO.  Returns (dq, dk, dv) chunks."""
        from . import engine
        from . import tensor_ops as ops
        from ._native import check, lib

        from .errors import StateError

        n, d = self.world, self.rank
        _, b, z, c, a = grad.shape
        seq = n * c
        dev = grad.device
        if "slot" not in ctx.extra:
            raise StateError("PeerRing.backward: this context's K/V slot was already released by a backward")
        self.check(ctx)  # the forward's status flag, read at this first synchronising use
        slot = ctx.extra.pop("slot")  # released exactly once: a second backward must not re-pool it
        dvec, grad_r = ops.rowdot_scale(grad, ctx.out, ctx.extra["rowscale"])  # D*r and dO*r (factored panel)
        dq = torch.empty((1, b, z, c, a), dtype=torch.bfloat16, device=dev)
        dk_part = torch.empty((n, b, z, c, a), dtype=torch.float32, device=dev)
        dv_part = torch.empty_like(dk_part)
        g = engine._geom(1, b, z, c, a, seq, 0, n)
        if not lib().rsa_bwd_fused_supported(ctypes.byref(g)):
            raise ValueError(f"PeerRing backward needs <= 4 query tiles per rank (c = {c})")
        check(lib().rsa_bwd_fused_peer(ctypes.byref(g), engine._view(ctx.q), self._views(slot, 0),
                                       self._views(slot, 1), engine._view(grad_r), engine._view(ctx.panel),
                                       dvec.data_ptr(), engine._view(dq), engine._view(dk_part),
                                       engine._view(dv_part), torch.cuda.current_stream(dev).cuda_stream),
              "rsa_bwd_fused_peer")
        self.ledger.record_ring_send(d, 2 * (n - 1) * b * z * c * a, 2 * (n - 1) * b * z * c * a * 2)
        dk = self.ring._reduce(dk_part)
        dv = self.ring._reduce(dv_part)
        self._free.setdefault((tuple(slot.local.shape[1:]), slot.local.dtype), []).append(slot)
        return dq, dk.to(grad.dtype), dv.to(grad.dtype)


# ------------------------------------------------------------------ bench

def bench_main(args, metric, unit, config, clock_sampler=None, peaks=None):
    """Multi-GPU arm of bench.py (launched under torchrun, one rank per GPU).

    Each rank holds B = batch * N sequences' c = L / N chunk (the paper's weak-scaling
    batch rule) and runs the 12-layer stack through ``SpmdRing``: K/V rings and dK/dV
    reduce-scatters over NCCL.  ``value`` is the whole job's tokens/s with the step time
    taken as the max over ranks; ``e2e`` repeats the step with every rank's chunks
    uploaded from pinned host memory and its outputs copied back.  RSA_BENCH_BACKEND=gloo
    runs the same code with host-staged transfers (several ranks on one GPU; test only).
    """
    import json
    import os

    backend = os.environ.get("RSA_BENCH_BACKEND", "nccl")
    local = int(os.environ.get("LOCAL_RANK", "0")) % max(1, torch.cuda.device_count())
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if backend == "nccl":
        dist.init_process_group("nccl", device_id=dev)
    else:
        dist.init_process_group(backend)
    n, rank = dist.get_world_size(), dist.get_rank()
    B, Z, L, A, LAYERS = args.batch * n, args.heads, args.seq, args.head_size, args.layers
    if L % n:
        raise SystemExit(f"seq {L} not divisible by {n} ranks")
    c = L // n
    ring = SpmdRing(transport="device" if backend == "nccl" else "host")
    gen = torch.Generator(device=dev).manual_seed(1000 + rank)

    def rnd():
        return torch.randn((1, B, Z, c, A), generator=gen, device=dev).to(torch.bfloat16)

    layers = [dict(q=rnd(), k=rnd(), v=rnd(), g=rnd()) for _ in range(LAYERS)]
    flag = torch.zeros(1, dtype=torch.int32, device=dev)

    def step():
        ctxs = []
        for ly in layers:
            _, ctx = ring.forward(ly["q"], ly["k"], ly["v"], flag)
            ctxs.append(ctx)
        for ly, ctx in zip(reversed(layers), reversed(ctxs)):
            ring.backward(ctx, ly["g"])

    def timed(fn, steps):
        torch.cuda.synchronize()
        dist.barrier()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(steps):
            fn()
        e1.record()
        torch.cuda.synchronize()
        dist.barrier()
        t = torch.tensor([e0.elapsed_time(e1) / steps], device=dev)
        if backend != "nccl":
            t = t.cpu()
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    for _ in range(args.warmup):
        step()
    if clock_sampler is not None:
        with clock_sampler(local) as clk:
            ms = timed(step, args.steps)
        clocks = clk.result()
    else:
        ms, clocks = timed(step, args.steps), None

    # end to end: this rank's q, k, v, dO chunks from pinned host memory, O and dQ/dK/dV back;
    # step s + 1's uploads run on a copy stream into the other buffer set while step s
    # computes and copies down (the same pipelining as bench.py's single-GPU e2e)
    hg = torch.Generator().manual_seed(2000 + rank)
    host = [[torch.randn((1, B, Z, c, A), generator=hg).to(torch.bfloat16).pin_memory() for _ in range(4)]
            for _ in range(LAYERS)]
    outs = [[torch.empty((1, B, Z, c, A), dtype=torch.bfloat16).pin_memory() for _ in range(4)]
            for _ in range(LAYERS)]
    copy = torch.cuda.Stream(dev)
    cur = torch.cuda.current_stream(dev)
    bufs = [[[torch.empty((1, B, Z, c, A), dtype=torch.bfloat16, device=dev) for _ in range(4)]
             for _ in range(LAYERS)] for _ in range(2)]
    up, free = [None, None], [None, None]

    def upload(si):
        with torch.cuda.stream(copy):
            if free[si] is not None:
                copy.wait_event(free[si])
            for hb, db in zip(host, bufs[si]):
                for dst, src in zip(db, hb):
                    dst.copy_(src, non_blocking=True)
            up[si] = torch.cuda.Event()
            up[si].record(copy)

    def e2e_step(si, prefetch):
        cur.wait_event(up[si])
        ctxs = []
        for (q, k, v, _), o in zip(bufs[si], outs):
            out, ctx = ring.forward(q, k, v, flag)
            o[0].copy_(out, non_blocking=True)
            ctxs.append(ctx)
        if prefetch:
            upload(1 - si)
        for i in reversed(range(LAYERS)):
            dq, dk, dv = ring.backward(ctxs[i], bufs[si][i][3])
            for j, t in enumerate((dq, dk, dv)):
                outs[i][j + 1].copy_(t, non_blocking=True)
        free[si] = torch.cuda.Event()
        free[si].record(cur)

    upload(0)
    e2e_step(0, False)
    e2e_steps = max(1, getattr(args, "e2e_steps", 8))
    state = {"i": 0}

    def timed_e2e():
        i = state["i"]
        if i == 0:
            upload(0)
        e2e_step(i % 2, i + 1 < e2e_steps)
        state["i"] = i + 1

    e2e_ms = timed(timed_e2e, e2e_steps)
    chunk_bytes = B * Z * c * A * 2

    if int(flag.item()):
        raise RuntimeError("non-finite scores in the benchmark inputs")
    if rank == 0:
        value = B * L / (ms / 1e3)
        # whole-step roofline per GPU: algorithmic HBM bytes of the fused path (panel written
        # once and read once, per-kernel chunk traffic) over the step time
        p_e, c_e = B * Z * c * L, B * Z * c * A
        step_bytes = LAYERS * ((2 * p_e + 8 * c_e) + (6 * c_e + 8 * B * Z * c) + (2 * p_e + 14 * c_e))
        hbm = (peaks or {}).get("hbm_gbs", 6650.0)
        achieved = step_bytes / (ms / 1e3) / 1e9
        print(json.dumps({
            "metric": metric, "value": value, "unit": unit, "n_gpus": n, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic N(0,1) bf16 inputs, per-layer q/k/v/dO", "config": config,
            "clocks": clocks,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                         "kernel": "whole step per GPU (ring hops overlapped with the kernels)", "traffic": None},
            "gpu_launches": (LAYERS * (2 * n + 2 * n + 1)) * args.steps,
            "e2e": {"value": B * L / (e2e_ms / 1e3), "unit": unit, "ms_per_step": e2e_ms,
                    "h2d_bytes_per_step": LAYERS * 4 * chunk_bytes, "d2h_bytes_per_step": LAYERS * 4 * chunk_bytes,
                    "path": "SpmdRing.forward/backward per rank, pinned host chunks in, O/dQ/dK/dV out"},
            "comm": {"mode": ring.mode, "backend": backend, "wire_bytes_per_rank_per_step":
                     ring.ledger.devices[rank].wire_bytes // max(1, args.steps + args.warmup + e2e_steps + 1)},
        }), flush=True)
    dist.destroy_process_group()

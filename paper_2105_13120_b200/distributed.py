"""RSA across real ranks: one process per GPU, rings over torch.distributed (NCCL).

This is the multi-GPU form of ringseq/ring_attention.py:124-217.  Rank d holds only its
own (B, Z, c, A) chunks; keys and values travel d -> d+1 by NCCL send/recv
(``batch_isend_irecv``), exactly the reference's ring direction and schedule
(ringseq/ring_attention.py:67-79, ringseq/cluster.py:293-318): at hop h rank d holds
origin j = (d - h) mod N.  Each hop runs ONE sm_100a kernel launch on the origin that
just arrived while the next hop is in flight.

Forward (both modes): K and V of an origin travel together (one ring of the pair --
the reference's K ring and V ring carry the same bytes in two circulations).  Per hop,
rsa_fwd_factored_ex runs the single-pass factored forward on origin j: hop 0 takes each
row's reference point from its first key tile, later hops reuse it, and the running
O~ = sum P~ V and l = sum P~ stay in fp32 buffers until the last hop normalises.  So
neither the K-ring statistics pass nor the recomputation of S of the two-pass form is
needed.  A row whose later scores exceed the reference point by > 2^96 (never for real
logits) sets flag bit 1 and the layer is recomputed two-pass on every row's true max.

Backward, ``attn="panel"`` (the reference's saved probability panel): the forward keeps
every origin's K and V (the slots the ring filled; O(L) per rank, small next to the
O(c * L) panel), so the backward needs NO ring: one launch over all resident origins
(rsa_bwd_fused when c <= 512, else rsa_bwd_panel_fused, or rsa_bwd_dkdv + rsa_bwd_dq with
RSA_B200_DETERMINISTIC=1) writes fp32 dK/dV partials for every origin, summed across ranks by ``reduce_scatter`` (default; half the bytes of
the reference's all-reduce + slice) or ``all_reduce`` (``mode="paper"``,
ringseq/ring_attention.py:206-209).

Backward, ``attn="stream"`` (no panel, O(c) state per rank, so the trainable length
grows linearly with N): the K/V pair circulates again, and the fp32 dK/dV accumulator of
each origin travels with it -- every rank adds its queries' contribution
(rsa_bwd_kv_stream, accumulate) and passes it on, and a final hop brings the complete sum
home -- while dQ accumulates locally (rsa_bwd_q_stream).  No full-length partial exists
anywhere; the sums run in a fixed ring order (deterministic).

The ledger charges what the reference charges (element counts, all-reduce convention);
``wire_bytes`` records the bytes actually sent.  The per-hop kernels are injected
(``HopKernels``) so the schedule can be tested on CPU with the gloo backend
(tests/test_distributed_gloo.py) using a test-only implementation; the product path always
uses ``CudaHopKernels``.
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
    """Per-hop launches of the sm_100a kernels (librsa_b200.so)."""

    def __init__(self):
        from . import engine
        from ._native import BF16, F32, RsaGeom, check, lib

        self.engine, self.BF16, self.F32, self.RsaGeom, self.check, self.lib = engine, BF16, F32, RsaGeom, check, lib

    def _g(self, q, seq, origin, n_org=1):
        _, b, z, c, a = q.shape
        return self.RsaGeom(1, b, z, c, a, seq, origin, n_org, 1.0 / math.sqrt(a))

    def _st(self, t):
        return torch.cuda.current_stream(t.device).cuda_stream

    def new_state(self, q):
        """fp32 running O~ and l, reference points m, row scale r, bf16 output, status flag."""
        _, b, z, c, a = q.shape
        dev = q.device
        rows = (1, b, z, c)
        return {"o_acc": torch.empty((1, b, z, c, a), dtype=torch.float32, device=dev),
                "l_acc": torch.empty(rows, dtype=torch.float32, device=dev),
                "rowmax": torch.empty(rows, dtype=torch.float32, device=dev),
                "rowscale": torch.empty(rows, dtype=torch.float32, device=dev),
                "out": torch.empty((1, b, z, c, a), dtype=q.dtype, device=dev),
                "flag": torch.zeros(1, dtype=torch.int32, device=dev)}

    def hop_forward(self, q, k_j, v_j, origin, seq, st, first, last, panel, exact=False):
        """Origin j's keys into the running factored forward (rsa_fwd_factored_ex)."""
        g = self._g(q, seq, origin)
        given = exact or not first
        self.engine._fwd_ex(q, k_j, v_j, g, panel=panel, rowmax=None if given else st["rowmax"],
                            rowmax_in=st["rowmax"] if given else None, exact=exact, o_acc=st["o_acc"],
                            l_acc=st["l_acc"], acc_in=not first, final=last, out=st["out"] if last else None,
                            rowscale=st["rowscale"] if last else None, flag=st["flag"])

    def row_max(self, q, k_slots, seq):
        """Every row's true max over all origins (scaled base 2), for the two-pass fallback."""
        n = k_slots.shape[0]
        _, b, z, c, _ = q.shape
        stats = torch.empty((n, 1, b, z, c, 2), dtype=torch.float32, device=q.device)
        flag = torch.zeros(1, dtype=torch.int32, device=q.device)
        for j in range(n):
            self.check(self.lib().rsa_fwd_stats(ctypes.byref(self._g(q, seq, j)), self.engine._view(q),
                                                self.engine._view(k_slots[j:j + 1]), stats[j].data_ptr(), 0,
                                                flag.data_ptr(), self._st(q)), "rsa_fwd_stats")
        return stats[..., 0].amax(0)

    def rowdot_scale(self, grad, out, rowscale):
        from . import tensor_ops

        return tensor_ops.rowdot_scale(grad, out, rowscale)

    def bwd_resident(self, q, k_slots, v_slots, grad_r, panel, dvec, seq, dq, dk_part, dv_part):
        """One launch over every resident origin: dQ (bf16) and fp32 dK/dV partials per origin."""
        n = k_slots.shape[0]
        g = self._g(q, seq, 0, n)
        V = self.engine._view
        L = self.lib()
        if L.rsa_bwd_fused_supported(ctypes.byref(g)):
            self.check(L.rsa_bwd_fused(ctypes.byref(g), V(q), V(k_slots), V(v_slots), V(grad_r), V(panel),
                                       dvec.data_ptr(), self.engine.NULL_VIEW, 0, V(dq), V(dk_part), V(dv_part),
                                       self.F32, 0, self._st(q)), "rsa_bwd_fused")
            return
        if not self.engine.deterministic():  # one panel read at any length (rsa_bwd_panel_fused)
            dq_acc = torch.empty(dq.shape, dtype=torch.float32, device=dq.device)
            self.check(L.rsa_bwd_panel_fused(ctypes.byref(g), V(q), V(k_slots), V(v_slots), V(grad_r), V(panel),
                                             dvec.data_ptr(), V(dk_part), V(dv_part), self.F32, 0, dq_acc.data_ptr(),
                                             0, V(dq), self._st(q)), "rsa_bwd_panel_fused")
            return
        self.check(L.rsa_bwd_dkdv(ctypes.byref(g), V(q), V(v_slots), V(grad_r), V(panel), dvec.data_ptr(),
                                  V(dk_part), V(dv_part), self.F32, 0, self._st(q)), "rsa_bwd_dkdv")
        self.check(L.rsa_bwd_dq(ctypes.byref(g), V(grad_r), V(k_slots), V(v_slots), V(panel), dvec.data_ptr(),
                                self.engine.NULL_VIEW, 0, V(dq), self._st(q)), "rsa_bwd_dq")

    def kv_stream_hop(self, q, k_j, v_j, grad_r, rowmax, dvec, seq, origin, dk_acc, dv_acc, accumulate):
        g = self._g(q, seq, origin)
        V = self.engine._view
        self.check(self.lib().rsa_bwd_kv_stream(ctypes.byref(g), V(q), V(k_j), V(v_j), V(grad_r), rowmax.data_ptr(),
                                                dvec.data_ptr(), V(dk_acc), V(dv_acc), self.F32, int(accumulate),
                                                self._st(q)), "rsa_bwd_kv_stream")

    def q_stream_hop(self, q, k_j, v_j, grad_r, rowmax, dvec, seq, origin, dq_acc, accumulate, dq_out):
        g = self._g(q, seq, origin)
        V = self.engine._view
        self.check(self.lib().rsa_bwd_q_stream(ctypes.byref(g), V(q), V(k_j), V(v_j), V(grad_r), rowmax.data_ptr(),
                                               dvec.data_ptr(), V(dq_acc), int(accumulate), V(dq_out), self._st(q)),
                   "rsa_bwd_q_stream")

    def fused_stream_hop(self, q, k_j, v_j, grad_r, rowmax, dvec, seq, origin, dk_acc, dv_acc, dq_acc, accumulate,
                         dq_out):
        """kv_stream_hop + q_stream_hop in one launch (rsa_bwd_stream_fused): fp32 dK/dV of
        origin j (accumulating), dQ partials added into the fp32 dq_acc (zeroed on the first
        hop), bf16 dq_out on the last."""
        g = self._g(q, seq, origin)
        V = self.engine._view
        self.check(self.lib().rsa_bwd_stream_fused(ctypes.byref(g), V(q), V(k_j), V(v_j), V(grad_r),
                                                   rowmax.data_ptr(), dvec.data_ptr(), V(dk_acc), V(dv_acc), self.F32,
                                                   int(accumulate), dq_acc.data_ptr(), int(accumulate), V(dq_out),
                                                   self._st(q)), "rsa_bwd_stream_fused")

    def project_pair(self, e_cols, k, f_cols, v):
        """[E_d K_d ; F_d V_d] as one fp32 [2][B][Z][K][A] buffer: rsa_linformer_project (four
        heads per tensor-core tile, this rank's c positions) when it tiles the shapes, else
        two rsa_gemm launches."""
        from . import tensor_ops

        b, z, c, a = k.shape
        kdim = e_cols.shape[0]
        out = torch.empty((2, b, z, kdim, a), dtype=torch.float32, device=k.device)
        if (a == 64 and c % 64 == 0 and kdim % 128 == 0 and (b * z) % 4 == 0 and e_cols.dtype == f_cols.dtype ==
                torch.bfloat16 and e_cols.stride(1) == f_cols.stride(1) == 1 and e_cols.stride(0) == f_cols.stride(0)):
            g = self.engine._geom(1, b, z, c, a, c, 0, 1)
            V = self.engine._view
            self.check(self.lib().rsa_linformer_project(ctypes.byref(g), kdim, e_cols.data_ptr(), f_cols.data_ptr(),
                                                        e_cols.stride(0), V(k.unsqueeze(0)), V(v.unsqueeze(0)),
                                                        out[0].data_ptr(), out[1].data_ptr(), None, None,
                                                        self._st(k)), "rsa_linformer_project")
            return out
        tensor_ops.matmul(e_cols, k, out=out[0])
        tensor_ops.matmul(f_cols, v, out=out[1])
        return out

    def low_rank_attention(self, q, k_low, v_low):
        """softmax(Q K'^T / sqrt(A)) V' with rows fully local: the stream-mode forward with
        key_chunk = K (no score or probability panel in HBM)."""
        from . import sparse_attention

        return sparse_attention.low_rank_attention(q, k_low, v_low)


@dataclass
class RingContext:
    """What the forward keeps for the backward (the reference keeps only probs)."""

    q: torch.Tensor
    k_slots: torch.Tensor | None
    panel: torch.Tensor | None
    out: torch.Tensor
    v_local: torch.Tensor
    extra: dict = field(default_factory=dict)


class SpmdRing:
    """One rank's view of the RSA ring over a torch.distributed process group."""

    def __init__(self, group=None, kernels=None, mode: str = "reduce_scatter", overlap: bool = True,
                 transport: str = "device", attn: str = "panel", sync_checks: bool = True):
        """``transport="host"`` stages every hop and reduction through host memory, for
        process groups whose backend cannot move device tensors point to point (gloo);
        the default sends the device buffers themselves (NCCL over NVLink).  ``attn`` is
        "panel" (the reference's saved panel; K/V cached, ring-free backward) or "stream"
        (O(c) state; the backward re-circulates K/V with travelling dK/dV sums)."""
        if mode not in ("reduce_scatter", "paper"):
            raise ValueError(f"unknown mode {mode!r}")
        if transport not in ("device", "host"):
            raise ValueError(f"unknown transport {transport!r}")
        if attn not in ("panel", "stream"):
            raise ValueError(f"unknown attn {attn!r}")
        self.host_staged = transport == "host"
        # sync_checks=False: no host read of the status flag per layer (a device sync); the
        # caller reads every context's flag once (``check_flags``), e.g. at the end of a step
        self.sync_checks = sync_checks
        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.kernels = CudaHopKernels() if kernels is None else kernels  # False: communication only
        self.mode = mode
        self.attn = attn
        self.overlap = overlap
        self.ledger = CommLedger(self.world)

    # ---- communication -------------------------------------------------

    def _peer(self, off: int) -> int:
        r = (self.rank + off) % self.world
        return dist.get_global_rank(self.group, r) if self.group else r

    def _post(self, pairs, charge: bool = True):
        """Post one ring hop for every (send, recv) pair: send to rank+1, receive from
        rank-1, all in one group.  Returns the pending handle for ``_wait``."""
        nxt, prv = self._peer(1), self._peer(-1)
        nbytes = sum(s.numel() * s.element_size() for s, _ in pairs)
        if charge:
            self.ledger.record_ring_send(self.rank, sum(s.numel() for s, _ in pairs), nbytes)
        else:
            self.ledger.devices[self.rank].wire_bytes += nbytes
        if self.host_staged and pairs[0][0].is_cuda:
            staged = [(s.cpu(), torch.empty(r.shape, dtype=r.dtype)) for s, r in pairs]
            ops = []
            for s_h, r_h in staged:
                ops += [dist.P2POp(dist.isend, s_h, nxt, self.group), dist.P2POp(dist.irecv, r_h, prv, self.group)]
            return (dist.batch_isend_irecv(ops), [(r, r_h) for (_, r), (_, r_h) in zip(pairs, staged)], staged)
        ops = []
        for s_, r_ in pairs:
            ops += [dist.P2POp(dist.isend, s_, nxt, self.group), dist.P2POp(dist.irecv, r_, prv, self.group)]
        return (dist.batch_isend_irecv(ops), None, None)

    @staticmethod
    def _wait(pending):
        if not pending:
            return
        works, copies, _ = pending
        for w in works:
            w.wait()
        for r, r_h in copies or ():
            r.copy_(r_h)

    def _circulate(self, slots, on_arrival):
        """Ring over per-origin slot tensors (each [N][...], slot d holding the local chunk)
        that travel together; ``on_arrival(h, j)`` runs once slot j of every tensor is valid."""
        n, d = self.world, self.rank
        hop = lambda src, dst: [(t[src], t[dst]) for t in slots]  # noqa: E731
        pending = self._post(hop(d, (d - 1) % n)) if n > 1 and self.overlap else None
        for h in range(n):
            j = (d - h) % n
            if h > 0:
                if not self.overlap:
                    pending = self._post(hop((j + 1) % n, j))
                self._wait(pending)
                pending = None
                if self.overlap and h + 1 < n:
                    pending = self._post(hop(j, (j - 1) % n))
            on_arrival(h, j)
        self._wait(pending)

    # ---- protocol --------------------------------------------------------

    def _forward_ring(self, q, k_slots, v_slots, st, panel):
        """Panel mode: the K/V pair circulates into per-origin slots (kept for the backward)."""
        n = self.world
        seq = n * q.shape[3]
        kern = self.kernels
        self._circulate([k_slots, v_slots], lambda h, j: kern.hop_forward(
            q, k_slots[j:j + 1], v_slots[j:j + 1], j, seq, st, h == 0, h == n - 1, panel))

    def _forward_ring_stream(self, q, k, v, st):
        """Stream mode: the K/V pair circulates through two buffers (O(c) per rank)."""
        n, d = self.world, self.rank
        _, b, z, c, a = q.shape
        seq = n * c
        kv = torch.empty((2, 2, 1, b, z, c, a), dtype=k.dtype, device=q.device)  # [buffer][k | v]
        kv[0, 0].copy_(k)
        kv[0, 1].copy_(v)
        for h in range(n):
            j = (d - h) % n
            cur, nxt = h % 2, (h + 1) % 2
            pend = self._post([(kv[cur], kv[nxt])]) if h + 1 < n else None
            self.kernels.hop_forward(q, kv[cur, 0], kv[cur, 1], j, seq, st, h == 0, h == n - 1, None)
            self._wait(pend)

    def forward(self, q: torch.Tensor, k: torch.Tensor, v: torch.Tensor, flag: torch.Tensor | None = None,
                check: bool | None = None):
        """q/k/v: this rank's [1][B][Z][c][A] chunks.  Returns (out, ctx).

        ``check`` reads the status flag (one host sync): bit 0 raises NumericError
        (ringseq/tensor_ops.py:80-81), bit 1 recomputes the layer on every row's true max.
        With ``check=False`` the caller reads ``ctx.extra["flag"]`` later (the backward
        checks it at its first synchronising use)."""
        kern = self.kernels
        n, d = self.world, self.rank
        _, b, z, c, a = q.shape
        seq = n * c
        dev = q.device
        st = kern.new_state(q)
        if flag is not None:
            st["flag"] = flag
        if self.attn == "panel":
            k_slots = torch.empty((n, b, z, c, a), dtype=k.dtype, device=dev)
            v_slots = torch.empty((n, b, z, c, a), dtype=v.dtype, device=dev)
            k_slots[d].copy_(k[0])
            v_slots[d].copy_(v[0])
            panel = torch.empty((1, b, z, c, seq), dtype=q.dtype, device=dev)
            self._forward_ring(q, k_slots, v_slots, st, panel)
            ctx = RingContext(q=q, k_slots=k_slots, panel=panel, out=st["out"], v_local=v,
                              extra={"flag": st["flag"], "state": st, "checked": False, "v_slots": v_slots})
        else:
            k_slots = v_slots = None
            self._forward_ring_stream(q, k, v, st)
            ctx = RingContext(q=q, k_slots=None, panel=None, out=st["out"], v_local=v,
                              extra={"flag": st["flag"], "state": st, "checked": False, "k_local": k})
        if self.sync_checks if check is None else check:
            self._check(ctx, k_slots, v_slots)
        return st["out"], ctx

    @staticmethod
    def check_flags(contexts) -> None:
        """One host read of every unchecked context's status flag (``sync_checks=False``):
        NumericError on a non-finite score or a row beyond the single-pass headroom (which
        the checked path recomputes)."""
        from .errors import NumericError

        for ctx in contexts:
            status = int(ctx.extra["flag"].item())
            if status & 1:
                raise NumericError("softmax_rows requires finite inputs")
            if status & 2:
                raise NumericError("a row exceeded the single-pass headroom in an unchecked forward; rerun with "
                                   "sync_checks=True")

    def _check(self, ctx, k_slots=None, v_slots=None):
        from .errors import NumericError

        if ctx.extra.get("checked"):
            return
        st = ctx.extra["state"]
        status = int(st["flag"].item())
        if status & 2 and not status & 1:  # recompute on the true row maxima
            n, d = self.world, self.rank
            q = ctx.q
            seq = n * q.shape[3]
            if k_slots is None:  # stream mode keeps no slots: circulate once more
                _, b, z, c, a = q.shape
                k_slots = torch.empty((n, b, z, c, a), dtype=q.dtype, device=q.device)
                v_slots = torch.empty_like(k_slots)
                k_slots[d].copy_(ctx.extra["k_local"][0])
                v_slots[d].copy_(ctx.v_local[0])
                self._circulate([k_slots, v_slots], lambda h, j: None)
            st["flag"].zero_()
            st["rowmax"].copy_(self.kernels.row_max(q, k_slots, seq))
            for h in range(n):  # every origin is resident now: the exact pass needs no communication
                j = (d - h) % n
                self.kernels.hop_forward(q, k_slots[j:j + 1], v_slots[j:j + 1], j, seq, st, h == 0, h == n - 1,
                                         ctx.panel, exact=True)
            status = int(st["flag"].item())
        if status:
            raise NumericError("softmax_rows requires finite inputs")
        ctx.extra["checked"] = True

    def backward(self, ctx: RingContext, grad: torch.Tensor):
        """grad: this rank's [1][B][Z][c][A] dO.  Returns (dq, dk, dv) chunks."""
        if self.sync_checks:
            self._check(ctx, ctx.k_slots, ctx.extra.get("v_slots"))
        if self.attn == "panel":
            return self._backward_panel(ctx, grad)
        return self._backward_stream(ctx, grad)

    def _backward_panel(self, ctx, grad):
        kern = self.kernels
        n = self.world
        _, b, z, c, a = grad.shape
        seq = n * c
        dev = grad.device
        st = ctx.extra["state"]
        dvec, grad_r = kern.rowdot_scale(grad, st["out"], st["rowscale"])  # D*r and dO*r (factored panel)
        dq = torch.empty((1, b, z, c, a), dtype=grad.dtype, device=dev)
        dk_part = torch.empty((n, b, z, c, a), dtype=_acc_dtype(grad), device=dev)
        dv_part = torch.empty_like(dk_part)
        kern.bwd_resident(ctx.q, ctx.k_slots, ctx.extra["v_slots"], grad_r, ctx.panel, dvec, seq, dq, dk_part, dv_part)
        # the reference's backward V ring and K ring (ringseq/ring_attention.py:180-196) are charged
        # although the slots cached by the forward make them free here
        elements = b * z * c * a
        self.ledger.record_ring_send(self.rank, 2 * (n - 1) * elements, 0)
        dk = self._reduce(dk_part)
        dv = self._reduce(dv_part)
        return dq, dk.to(grad.dtype), dv.to(grad.dtype)

    def _backward_stream(self, ctx, grad):
        kern = self.kernels
        n, d = self.world, self.rank
        _, b, z, c, a = grad.shape
        seq = n * c
        dev = grad.device
        st = ctx.extra["state"]
        dvec, grad_r = kern.rowdot_scale(grad, st["out"], st["rowscale"])
        # two K/V slots and two dK/dV accumulators travel the ring (O(c) per rank)
        kv = torch.empty((2, 2, 1, b, z, c, a), dtype=grad.dtype, device=dev)     # [buf][k|v]
        acc = torch.empty((2, 2, 1, b, z, c, a), dtype=_acc_dtype(grad), device=dev)  # [buf][dk|dv]
        kv[0, 0].copy_(ctx.extra["k_local"])
        kv[0, 1].copy_(ctx.v_local)
        fused = hasattr(kern, "fused_stream_hop") and not kern.engine.deterministic()
        dq_acc = torch.empty((1, b, z, c, a), dtype=torch.float32 if fused else _acc_dtype(grad), device=dev)
        dq = torch.empty((1, b, z, c, a), dtype=grad.dtype, device=dev)
        for h in range(n):
            j = (d - h) % n
            cur, nxt = h % 2, (h + 1) % 2
            pend_kv = self._post([(kv[cur], kv[nxt])]) if h + 1 < n and n > 1 else None
            if fused:
                kern.fused_stream_hop(ctx.q, kv[cur, 0], kv[cur, 1], grad_r, st["rowmax"], dvec, seq, j, acc[cur, 0],
                                      acc[cur, 1], dq_acc, h > 0, dq if h == n - 1 else None)
            else:
                kern.kv_stream_hop(ctx.q, kv[cur, 0], kv[cur, 1], grad_r, st["rowmax"], dvec, seq, j, acc[cur, 0],
                                   acc[cur, 1], h > 0)
                kern.q_stream_hop(ctx.q, kv[cur, 0], kv[cur, 1], grad_r, st["rowmax"], dvec, seq, j, dq_acc, h > 0,
                                  dq if h == n - 1 else None)
            # origin j's dK/dV sum moves on with it; after the last hop it arrives home complete
            pend_acc = self._post([(acc[cur], acc[nxt])], charge=False) if n > 1 else None
            self._wait(pend_kv)
            self._wait(pend_acc)
        done = acc[n % 2]
        # the reference's backward also all-reduces two full-length (N*C element) partials
        elements = b * z * c * a
        self.ledger.record_allreduce(d, n * elements)
        self.ledger.record_allreduce(d, n * elements)
        return dq, done[0].to(grad.dtype), done[1].to(grad.dtype)

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
        self.ledger.record_ring_send(d, 2 * (n - 1) * b * z * kdim * a, 0)
        if n > 1 and self.host_staged and low.is_cuda:
            host = low.cpu()
            dist.all_reduce(host, group=self.group)
            low.copy_(host)
        elif n > 1:
            dist.all_reduce(low, group=self.group)
        if n > 1:
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
    batch rule, as the N = 1 arm) and runs the 12-layer stack through ``SpmdRing``: the K/V
    pair ring with one single-pass factored launch per hop, and (panel mode) one backward
    launch over the cached K/V plus the dK/dV reduce-scatter over NCCL.  ``value`` is the
    whole job's tokens/s with the step time taken as the max over ranks; ``e2e`` repeats the
    step with every rank's chunks uploaded from pinned host memory and its outputs copied
    back; ``link`` is the bytes each rank actually sent per step over the step time against
    NVLink 5's 900 GB/s per direction.  RSA_BENCH_BACKEND=gloo runs the same code with
    host-staged transfers (several ranks on one GPU; test only).
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
    attn = getattr(args, "attn", "panel")
    ring = SpmdRing(transport="device" if backend == "nccl" else "host", attn=attn, sync_checks=False)
    gen = torch.Generator(device=dev).manual_seed(1000 + rank)

    def rnd():
        return torch.randn((1, B, Z, c, A), generator=gen, device=dev).to(torch.bfloat16)

    layers = [dict(q=rnd(), k=rnd(), v=rnd(), g=rnd()) for _ in range(LAYERS)]
    last_ctx = []

    def step():
        ctxs = []
        for ly in layers:
            _, ctx = ring.forward(ly["q"], ly["k"], ly["v"])
            ctxs.append(ctx)
        for ly, ctx in zip(reversed(layers), reversed(ctxs)):
            ring.backward(ctx, ly["g"])
        last_ctx[:] = ctxs

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
    SpmdRing.check_flags(last_ctx)
    wire0 = ring.ledger.devices[rank].wire_bytes
    if clock_sampler is not None:
        with clock_sampler(local) as clk:
            ms = timed(step, args.steps)
        clocks = clk.result()
    else:
        ms, clocks = timed(step, args.steps), None
    SpmdRing.check_flags(last_ctx)
    wire_step = (ring.ledger.devices[rank].wire_bytes - wire0) / max(1, args.steps)

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
            out, ctx = ring.forward(q, k, v)
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
        last_ctx[:] = ctxs

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
    SpmdRing.check_flags(last_ctx)
    chunk_bytes = B * Z * c * A * 2

    if rank == 0:
        value = B * L / (ms / 1e3)
        hbm = (peaks or {}).get("hbm_gbs", 6650.0)
        # whole step per GPU against SURVEY.md 8(d): 4*P_e + 16*C_e HBM bytes per layer
        p_e, c_e = B * Z * c * L, B * Z * c * A
        step_bytes = LAYERS * (4 * p_e + 16 * c_e)
        achieved = step_bytes / (ms / 1e3) / 1e9
        t_hbm = step_bytes / (hbm * 1e9)
        t_link = wire_step / 900e9
        # per layer: n forward hops, rowdot, then one (c <= 512) or two backward launches (panel)
        # or one fused launch per hop plus dQ's bf16 cast (stream)
        launches = LAYERS * ((n + 1 + (1 if c <= 512 else 2)) if attn == "panel" else (2 * n + 2))
        print(json.dumps({
            "metric": metric, "value": value, "unit": unit, "n_gpus": n, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
            "data": "synthetic N(0,1) bf16 inputs, per-layer q/k/v/dO", "config": dict(config, attn=attn),
            "clocks": clocks,
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm, "unit": "GB/s", "frac": achieved / hbm,
                         "kernel": "whole step per GPU (ring hops overlapped with the kernels)", "traffic": None,
                         "step": {"bytes": step_bytes, "frac": achieved / hbm}},
            "link": {"wire_bytes_per_step": wire_step, "achieved_GBps": wire_step / (ms / 1e3) / 1e9,
                     "peak_GBps": 900.0, "frac": wire_step / (ms / 1e3) / 900e9,
                     "weak_scaling_ceiling": {"overlapped": t_hbm / max(t_hbm, t_link),
                                              "serial": t_hbm / (t_hbm + t_link)},
                     "note": "bytes this rank sent (ledger wire_bytes) per step; the ceiling is the HBM-roofline "
                             "step time over max(HBM, link) time at 900 GB/s per direction"},
            "gpu_launches": launches * args.steps,
            "e2e": {"value": B * L / (e2e_ms / 1e3), "unit": unit, "ms_per_step": e2e_ms,
                    "h2d_bytes_per_step": LAYERS * 4 * chunk_bytes, "d2h_bytes_per_step": LAYERS * 4 * chunk_bytes,
                    "path": "SpmdRing.forward/backward per rank, pinned host chunks in, O/dQ/dK/dV out"},
            "comm": {"mode": ring.mode, "backend": backend, "attn": attn},
        }), flush=True)
    dist.destroy_process_group()

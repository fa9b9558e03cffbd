"""World-size-2/3 CPU tests of the SPMD ring schedule (paper_2105_13120_b200.distributed).

The product path launches sm_100a kernels per hop; here the same
``SpmdRing`` schedule runs over the gloo backend with a TEST-ONLY float64
implementation of the four per-hop kernels (``CpuHopKernels`` below), so the
ring bookkeeping -- who sends what to whom, which origin arrives at which
hop, the stats slots, the panel column blocks, the cross-hop accumulation
and the dK/dV reduction -- is checked against the oracle without a GPU.
"""

from __future__ import annotations

import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import ringseq_np as orc


class CpuHopKernels:
    """float64 restatement of the per-hop kernel contracts (test double).

    Same factored convention as the device kernels: the panel block of origin j holds
    P~ = exp(s - m) with m the row's reference point (taken at hop 0, reused later), the
    running O~ = sum P~ V and l = sum P~ finish as O = O~ / l and r = 1 / l."""

    def new_state(self, q):
        _, b, z, c, a = q.shape
        rows = (1, b, z, c)
        return {"o_acc": torch.zeros((1, b, z, c, a), dtype=torch.float64),
                "l_acc": torch.zeros(rows, dtype=torch.float64), "rowmax": torch.zeros(rows, dtype=torch.float64),
                "rowscale": torch.zeros(rows, dtype=torch.float64),
                "out": torch.zeros((1, b, z, c, a), dtype=torch.float64), "flag": torch.zeros(1, dtype=torch.int32)}

    @staticmethod
    def _s(q, k_j):
        return q[0] @ k_j[0].transpose(-1, -2) / math.sqrt(q.shape[-1])

    def hop_forward(self, q, k_j, v_j, origin, seq, st, first, last, panel, exact=False):
        s = self._s(q, k_j)
        if first and not exact:
            st["rowmax"][0] = s.max(-1).values
        pt = torch.exp(s - st["rowmax"][0][..., None])
        c = q.shape[-2]
        if panel is not None:
            panel[0][..., origin * c:(origin + 1) * c] = pt
        o, lsum = pt @ v_j[0], pt.sum(-1)
        if not first:
            o, lsum = o + st["o_acc"][0], lsum + st["l_acc"][0]
        if last:
            st["out"][0] = o / lsum[..., None]
            st["rowscale"][0] = 1.0 / lsum
        else:
            st["o_acc"][0], st["l_acc"][0] = o, lsum

    def rowdot_scale(self, grad, out, rowscale):
        return rowscale * (grad * out).sum(-1), grad * rowscale[..., None]

    def _ds(self, pt, grad_r, v_j, dvec):
        dp = grad_r[0] @ v_j[0].transpose(-1, -2)
        return pt * (dp - dvec[0][..., None]) / math.sqrt(grad_r.shape[-1])

    def bwd_resident(self, q, k_slots, v_slots, grad_r, panel, dvec, seq, dq, dk_part, dv_part):
        c = q.shape[-2]
        dq.zero_()
        for j in range(k_slots.shape[0]):
            pt = panel[0][..., j * c:(j + 1) * c]
            ds = self._ds(pt, grad_r, v_slots[j:j + 1], dvec)
            dq[0] += ds @ k_slots[j]
            dk_part[j] = ds.transpose(-1, -2) @ q[0]
            dv_part[j] = pt.transpose(-1, -2) @ grad_r[0]

    def kv_stream_hop(self, q, k_j, v_j, grad_r, rowmax, dvec, seq, origin, dk_acc, dv_acc, accumulate):
        pt = torch.exp(self._s(q, k_j) - rowmax[0][..., None])
        ds = self._ds(pt, grad_r, v_j, dvec)
        dk, dv = ds.transpose(-1, -2) @ q[0], pt.transpose(-1, -2) @ grad_r[0]
        dk_acc[0] = dk_acc[0] + dk if accumulate else dk
        dv_acc[0] = dv_acc[0] + dv if accumulate else dv

    def q_stream_hop(self, q, k_j, v_j, grad_r, rowmax, dvec, seq, origin, dq_acc, accumulate, dq_out):
        pt = torch.exp(self._s(q, k_j) - rowmax[0][..., None])
        t = self._ds(pt, grad_r, v_j, dvec) @ k_j[0]
        dq_acc[0] = dq_acc[0] + t if accumulate else t
        if dq_out is not None:
            dq_out.copy_(dq_acc)


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, shape, seed, mode, overlap, attn, results):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2105_13120_b200.distributed import SpmdRing

        b, z, seq, a = shape
        rng = orc.make_rng(seed)
        q, k, v, g = (rng.standard_normal((b, z, seq, a)) for _ in range(4))
        ch = lambda x: torch.from_numpy(orc.chunks_of(x, world)[rank][None].copy())  # noqa: E731
        ring = SpmdRing(kernels=CpuHopKernels(), mode=mode, overlap=overlap, attn=attn)
        out, ctx = ring.forward(ch(q), ch(k), ch(v))
        dq, dk, dv = ring.backward(ctx, ch(g))
        st = ctx.extra["state"]
        panel = None if ctx.panel is None else (ctx.panel[0] * st["rowscale"][0][..., None]).numpy()
        results[rank] = {
            "out": out[0].numpy(), "panel": panel,
            "dq": dq[0].numpy(), "dk": dk[0].numpy(), "dv": dv[0].numpy(),
            "ring": ring.ledger.devices[rank].ring_p2p_elements,
            "ar": ring.ledger.devices[rank].allreduce_elements,
            "wire": ring.ledger.devices[rank].wire_bytes,
        }
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,mode,overlap,attn", [(2, "reduce_scatter", True, "panel"), (3, "paper", False, "panel"),
                                                     (2, "paper", True, "panel"), (2, "reduce_scatter", True, "stream"),
                                                     (3, "paper", True, "stream"), (4, "reduce_scatter", True, "stream")])
def test_spmd_ring_matches_oracle(world, mode, overlap, attn):
    """The ring schedule (K/V pair ring with single-pass factored hops; panel mode: cached
    slots and a ring-free backward with reduced partials; stream mode: re-circulated K/V
    with travelling dK/dV sums) against the oracle, ledgers in the reference convention."""
    shape = (1, 2, 6 * world, 4)
    seed = 17 + world
    mgr = mp.get_context("spawn").Manager()
    results = mgr.dict()
    mp.start_processes(_worker, args=(world, _free_port(), shape, seed, mode, overlap, attn, results), nprocs=world,
                       join=True, start_method="spawn")
    b, z, seq, a = shape
    rng = orc.make_rng(seed)
    q, k, v, g = (rng.standard_normal((b, z, seq, a)) for _ in range(4))
    ch = lambda x: orc.chunks_of(x, world)  # noqa: E731
    outs, probs, ring_f = orc.ring_forward(ch(q), ch(k), ch(v), exact=False)
    dq, dk, dv, (ring_b, ar_b) = orc.ring_backward(ch(q), ch(k), ch(v), probs, ch(g), exact=False)
    for d in range(world):
        r = results[d]
        assert np.max(np.abs(r["out"] - outs[d])) <= 1e-12
        if attn == "panel":
            assert np.max(np.abs(r["panel"] - probs[d])) <= 1e-12
        else:
            assert r["panel"] is None
        assert np.max(np.abs(r["dq"] - dq[d])) <= 1e-12
        assert np.max(np.abs(r["dk"] - dk[d])) <= 1e-12
        assert np.max(np.abs(r["dv"] - dv[d])) <= 1e-12
        # forward K+V rings, backward V+K rings: 4(N-1) chunks; two all-reduces
        assert r["ring"] == ring_f + ring_b
        assert r["ar"] == ar_b
        # the bytes on the wire are the cost report's plan (float64 here: 8-byte elements);
        # gloo has no reduce-scatter, so both panel modes all-reduce the partials
        from paper_2105_13120_b200 import AttentionConfig
        from paper_2105_13120_b200.cost_report import wire_bytes

        cfg = AttentionConfig(batch_size=b, seq_len=seq, hidden_size=z * a, num_heads=z, head_size=a,
                              num_devices=world)
        plan = "stream" if attn == "stream" else "panel_paper"
        want = wire_bytes(cfg, plan, kv_bytes=8, grad_bytes=8)
        assert r["wire"] == want["forward"] + want["backward"]


class CpuLinformerKernels(CpuHopKernels):
    def project_pair(self, e_cols, k, f_cols, v):
        return torch.stack([e_cols @ k, f_cols @ v])

    def low_rank_attention(self, q, k_low, v_low):
        s = q @ k_low.transpose(-1, -2) / math.sqrt(q.shape[-1])
        return torch.softmax(s, -1) @ v_low


def _lin_worker(rank, world, port, shape, seed, results):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2105_13120_b200.distributed import SpmdRing

        b, z, seq, a, kp = shape
        rng = orc.make_rng(seed)
        q, k, v = (rng.standard_normal((b, z, seq, a)) for _ in range(3))
        e, f = rng.standard_normal((kp, seq)), rng.standard_normal((kp, seq))
        ch = lambda x: torch.from_numpy(orc.chunks_of(x, world)[rank][None].copy())  # noqa: E731
        c = seq // world
        ring = SpmdRing(kernels=CpuLinformerKernels())
        out = ring.linformer_forward(ch(q), ch(k), ch(v), torch.from_numpy(e[:, rank * c:(rank + 1) * c].copy()),
                                     torch.from_numpy(f[:, rank * c:(rank + 1) * c].copy()))
        results[rank] = {"out": out[0].numpy(), "ring": ring.ledger.devices[rank].ring_p2p_elements}
    finally:
        dist.destroy_process_group()


def test_spmd_linformer_matches_oracle():
    world, shape, seed = 2, (2, 3, 40, 5, 7), 51
    mgr = mp.get_context("spawn").Manager()
    results = mgr.dict()
    mp.start_processes(_lin_worker, args=(world, _free_port(), shape, seed, results), nprocs=world, join=True,
                       start_method="spawn")
    b, z, seq, a, kp = shape
    rng = orc.make_rng(seed)
    q, k, v = (rng.standard_normal((b, z, seq, a)) for _ in range(3))
    e, f = rng.standard_normal((kp, seq)), rng.standard_normal((kp, seq))
    ch = lambda x: orc.chunks_of(x, world)  # noqa: E731
    outs, ring = orc.sparse_ring_forward(ch(q), ch(k), ch(v), e, f, exact=False)
    for d in range(world):
        assert np.max(np.abs(results[d]["out"] - outs[d])) <= 1e-12
        assert results[d]["ring"] == ring

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
    """float64 restatement of the per-hop kernel contracts (test double)."""

    def new_stats(self, q, n):
        _, b, z, c, _ = q.shape
        return torch.empty((n, b, z, c, 2), dtype=torch.float64)

    def stats(self, q, k_j, origin, seq, stats, flag):
        s = q[0] @ k_j[0].transpose(-1, -2) / math.sqrt(q.shape[-1])
        m = s.max(-1).values
        stats[origin, ..., 0] = m
        stats[origin, ..., 1] = torch.exp(s - m[..., None]).sum(-1)

    def probs_pv(self, q, k_j, v_j, origin, seq, stats, n_slots, panel, o_acc, accumulate, o_out):
        m_all = stats[:n_slots, ..., 0]
        mx = m_all.max(0).values
        lsum = (stats[:n_slots, ..., 1] * torch.exp(m_all - mx)).sum(0)
        s = q[0] @ k_j[0].transpose(-1, -2) / math.sqrt(q.shape[-1])
        p = torch.exp(s - mx[..., None]) / lsum[..., None]
        c = q.shape[-2]
        panel[0][..., origin * c:(origin + 1) * c] = p
        o = p @ v_j[0]
        o_acc[0] = o_acc[0] + o if accumulate else o
        if o_out is not None:
            o_out.copy_(o_acc)

    def rowdot(self, grad, out):
        return (grad * out).sum(-1)

    @staticmethod
    def _ds(grad, v_j, panel, dvec, origin):
        c = v_j.shape[-2]
        p = panel[0][..., origin * c:(origin + 1) * c]
        dp = grad[0] @ v_j[0].transpose(-1, -2)
        return p, p * (dp - dvec[0][..., None]) / math.sqrt(grad.shape[-1])

    def dkdv(self, q, v_j, grad, panel, dvec, origin, seq, dk_j, dv_j):
        p, dsb = self._ds(grad, v_j, panel, dvec, origin)
        dk_j[0] = dsb.transpose(-1, -2) @ q[0]
        dv_j[0] = p.transpose(-1, -2) @ grad[0]

    def dq(self, grad, k_j, v_j, panel, dvec, origin, seq, dq_acc, accumulate, dq_out):
        _, dsb = self._ds(grad, v_j, panel, dvec, origin)
        t = dsb @ k_j[0]
        dq_acc[0] = dq_acc[0] + t if accumulate else t
        if dq_out is not None:
            dq_out.copy_(dq_acc)


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, shape, seed, mode, overlap, results):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2105_13120_b200.distributed import SpmdRing

        b, z, seq, a = shape
        rng = orc.make_rng(seed)
        q, k, v, g = (rng.standard_normal((b, z, seq, a)) for _ in range(4))
        ch = lambda x: torch.from_numpy(orc.chunks_of(x, world)[rank][None].copy())  # noqa: E731
        ring = SpmdRing(kernels=CpuHopKernels(), mode=mode, overlap=overlap)
        out, ctx = ring.forward(ch(q), ch(k), ch(v))
        dq, dk, dv = ring.backward(ctx, ch(g))
        results[rank] = {
            "out": out[0].numpy(), "panel": ctx.panel[0].numpy(),
            "dq": dq[0].numpy(), "dk": dk[0].numpy(), "dv": dv[0].numpy(),
            "ring": ring.ledger.devices[rank].ring_p2p_elements,
            "ar": ring.ledger.devices[rank].allreduce_elements,
        }
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,mode,overlap", [(2, "reduce_scatter", True), (3, "paper", False), (2, "paper", True)])
def test_spmd_ring_matches_oracle(world, mode, overlap):
    shape = (1, 2, 6 * world, 4)
    seed = 17 + world
    mgr = mp.get_context("spawn").Manager()
    results = mgr.dict()
    mp.start_processes(_worker, args=(world, _free_port(), shape, seed, mode, overlap, results), nprocs=world,
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
        assert np.max(np.abs(r["panel"] - probs[d])) <= 1e-12
        assert np.max(np.abs(r["dq"] - dq[d])) <= 1e-12
        assert np.max(np.abs(r["dk"] - dk[d])) <= 1e-12
        assert np.max(np.abs(r["dv"] - dv[d])) <= 1e-12
        # forward K+V rings, backward V+K rings: 4(N-1) chunks; two all-reduces
        assert r["ring"] == ring_f + ring_b
        assert r["ar"] == ar_b


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

"""The SPMD ring (distributed.SpmdRing) with its real sm_100a per-hop kernels.

Two or three processes share cuda:0 and talk over gloo with host-staged hops
(``transport="host"``), so the CUDA hop kernels -- rsa_fwd_stats / rsa_fwd_probs_pv per
arriving origin, rsa_bwd_dkdv / rsa_bwd_dq per hop with fp32 cross-hop accumulation, the
dK/dV partial all-reduce, and the Linformer projection all-reduce -- run exactly as on N
GPUs, against the float64 oracle (tests/test_distributed_gloo.py checks the same schedule
with a float64 double of the kernels).  Tolerances as in test_gpu_rsa.py.
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

pytestmark = pytest.mark.gpu


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _inputs(b, z, seq, a, seed):
    rng = orc.make_rng(seed)
    return [orc.bf16_round(rng.standard_normal((b, z, seq, a))) for _ in range(4)]


def _worker(rank, world, port, shape, seed, mode, attn, results, backend="gloo"):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    if backend == "nccl":  # one GPU per rank: the real NCCL device transport
        torch.cuda.set_device(rank)
        dev = torch.device("cuda", rank)
        dist.init_process_group("nccl", rank=rank, world_size=world, device_id=dev)
    else:  # ranks share cuda:0, hops staged through host memory over gloo
        torch.cuda.set_device(0)
        dev = torch.device("cuda", 0)
        dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys

        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        from paper_2105_13120_b200 import engine
        from paper_2105_13120_b200.distributed import SpmdRing

        b, z, seq, a = shape
        q, k, v, g = _inputs(b, z, seq, a, seed)
        ch = lambda x: torch.from_numpy(orc.chunks_of(x, world)[rank][None].copy()).to(dev, torch.bfloat16)  # noqa
        ring = SpmdRing(mode=mode, transport="host" if backend == "gloo" else "device", attn=attn)
        out, ctx = ring.forward(ch(q), ch(k), ch(v))
        dq, dk, dv = ring.backward(ctx, ch(g))
        # Linformer: this rank's column blocks of E / F
        kp = 32
        rng = orc.make_rng(seed + 5)
        e = orc.bf16_round(rng.standard_normal((kp, seq)) / math.sqrt(seq))
        f = orc.bf16_round(rng.standard_normal((kp, seq)) / math.sqrt(seq))
        c = seq // world
        cols = lambda m: torch.from_numpy(m[:, rank * c:(rank + 1) * c].copy()).to(dev, torch.bfloat16)  # noqa
        lin = ring.linformer_forward(ch(q), ch(k), ch(v), cols(e), cols(f))
        torch.cuda.synchronize()
        f64 = lambda t: t.float().cpu().numpy().astype(np.float64)  # noqa: E731
        st = ctx.extra["state"]
        panel = None if ctx.panel is None else f64(engine.normalized_panel(ctx.panel[0], st["rowscale"][0]))
        results[rank] = {"out": f64(out[0]), "panel": panel, "dq": f64(dq[0]), "dk": f64(dk[0]),
                         "dv": f64(dv[0]), "lin": f64(lin[0] if lin.dim() == 5 else lin),
                         "ring": ring.ledger.devices[rank].ring_p2p_elements,
                         "wire": ring.ledger.devices[rank].wire_bytes,
                         "flag": int(ctx.extra["flag"].item())}
    finally:
        dist.destroy_process_group()


def _rel(x, y):
    return np.linalg.norm(x - y) / np.linalg.norm(y)


SPMD_CASES = [(2, "reduce_scatter", "panel", (1, 2, 256, 64)), (3, "paper", "panel", (1, 2, 384, 64)),
              (2, "paper", "panel", (2, 1, 400, 64)), (2, "reduce_scatter", "panel", (1, 2, 2048, 64)),
              (2, "reduce_scatter", "stream", (1, 2, 256, 64)), (3, "paper", "stream", (2, 1, 384, 64)),
              (2, "paper", "stream", (1, 2, 2048, 64))]


def _check_spmd(world, mode, attn, shape, seed, results, backend="gloo"):
    from paper_2105_13120_b200 import AttentionConfig
    from paper_2105_13120_b200.cost_report import wire_bytes

    b, z, seq, a = shape
    q, k, v, g = _inputs(b, z, seq, a, seed)
    ch = lambda x: orc.chunks_of(x, world)  # noqa: E731
    outs, probs, _ = orc.ring_forward(ch(q), ch(k), ch(v), exact=False)
    dq, dk, dv, _ = orc.ring_backward(ch(q), ch(k), ch(v), probs, ch(g), exact=False)
    rng = orc.make_rng(seed + 5)
    e = orc.bf16_round(rng.standard_normal((32, seq)) / math.sqrt(seq))
    f = orc.bf16_round(rng.standard_normal((32, seq)) / math.sqrt(seq))
    lin, _ = orc.sparse_ring_forward(ch(q), ch(k), ch(v), e, f, exact=False)
    for d in range(world):
        r = results[d]
        assert r["flag"] == 0
        assert _rel(r["out"], outs[d]) <= 1e-2
        if attn == "panel":
            assert np.max(np.abs(r["panel"] - probs[d])) <= 4e-3
        for name, want in (("dq", dq[d]), ("dk", dk[d]), ("dv", dv[d]), ("lin", lin[d])):
            assert _rel(r[name], want) <= 1e-2, (d, name, _rel(r[name], want))
        assert r["ring"] == 4 * (world - 1) * b * z * (seq // world) * a + 2 * (world - 1) * b * z * 32 * a
        # bytes on the wire = the cost report's plan + the Linformer's fp32 [K'; V'] all-reduce
        cfg = AttentionConfig(batch_size=b, seq_len=seq, hidden_size=z * a, num_heads=z, head_size=a,
                              num_devices=world)
        plan = "stream" if attn == "stream" else (
            "panel" if backend == "nccl" and mode == "reduce_scatter" else "panel_paper")
        want = wire_bytes(cfg, plan)
        lin_bytes = 2 * (2 * b * z * 32 * a * 4) * (world - 1) // world
        assert r["wire"] == want["forward"] + want["backward"] + lin_bytes, (r["wire"], want, lin_bytes)


@pytest.mark.parametrize("world,mode,attn,shape", SPMD_CASES)
def test_spmd_ring_cuda_kernels_match_oracle(world, mode, attn, shape):
    """SpmdRing with its real kernels: the K/V pair ring with one rsa_fwd_factored_ex per hop;
    panel mode's ring-free backward over the cached slots (rsa_bwd_fused for c <= 512, else
    rsa_bwd_panel_fused) with reduced partials; stream mode's re-circulated K/V with
    travelling dK/dV sums (rsa_bwd_stream_fused per hop: fp32 dK/dV accumulated across hops,
    dQ partials added into one fp32 accumulator over all hops)."""
    seed = 40 + world
    mgr = mp.get_context("spawn").Manager()
    results = mgr.dict()
    mp.start_processes(_worker, args=(world, _free_port(), shape, seed, mode, attn, results), nprocs=world, join=True,
                       start_method="spawn")
    _check_spmd(world, mode, attn, shape, seed, results)


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs 2 GPUs for the NCCL device transport")
@pytest.mark.parametrize("mode,attn", [("reduce_scatter", "panel"), ("paper", "panel"), ("reduce_scatter", "stream")])
def test_spmd_ring_nccl_two_gpus(mode, attn):
    """The product transport: NCCL send/recv of device buffers between two GPUs, the NCCL
    reduce-scatter / all-reduce of the dK/dV partials, and the Linformer all-reduce."""
    world, shape, seed = 2, (1, 2, 512, 64), 90
    mgr = mp.get_context("spawn").Manager()
    results = mgr.dict()
    mp.start_processes(_worker, args=(world, _free_port(), shape, seed, mode, attn, results, "nccl"), nprocs=world,
                       join=True, start_method="spawn")
    _check_spmd(world, mode, attn, shape, seed, results, backend="nccl")


def _peer_worker(rank, world, port, shape, seed, results):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys

        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        from paper_2105_13120_b200 import engine
        from paper_2105_13120_b200.distributed import PeerRing

        torch.cuda.set_device(0)
        dev = torch.device("cuda", 0)
        b, z, seq, a = shape
        q, k, v, g = _inputs(b, z, seq, a, seed)
        ch = lambda x: torch.from_numpy(orc.chunks_of(x, world)[rank][None].copy()).to(dev, torch.bfloat16)  # noqa
        ring = PeerRing(transport="host")
        outs = []
        for layer in range(2):  # two layers in flight: two registered slots, then reuse
            out, ctx = ring.forward(ch(q), ch(k), ch(v))
            outs.append((out, ctx))
        dq, dk, dv = ring.backward(outs[1][1], ch(g))
        dq0, dk0, dv0 = ring.backward(outs[0][1], ch(g))
        out, ctx = ring.forward(ch(q), ch(k), ch(v))  # reuses a released slot
        PeerRing.check(ctx)
        torch.cuda.synchronize()
        f64 = lambda t: t.float().cpu().numpy().astype(np.float64)  # noqa: E731
        probs = engine.normalized_panel(ctx.panel[0], ctx.extra["rowscale"][0])
        results[rank] = {"out": f64(out[0]), "probs": f64(probs), "dq": f64(dq[0]), "dk": f64(dk[0]),
                         "dv": f64(dv[0]), "same": bool(torch.equal(dq, dq0) and torch.equal(dk, dk0)
                                                        and torch.equal(dv, dv0)),
                         "flag": int(ctx.extra["flag"].item()), "ring": ring.ledger.devices[rank].ring_p2p_elements}
        ring.backward(ctx, ch(g))  # hand the last slot back, then unmap everything before teardown
        ring.close()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,shape", [(2, (1, 2, 256, 64)), (3, (2, 2, 384, 64)), (4, (1, 3, 512, 64)),
                                         (2, (2, 2, 400, 64))])  # c = 200: ragged tiles
def test_peer_ring_matches_oracle(world, shape):
    """PeerRing: one fwd_factored_peer / bwd_fused_peer launch per rank reading every origin's
    K/V through CUDA IPC (here: processes sharing one B200), against the oracle."""
    seed = 60 + world
    mgr = mp.get_context("spawn").Manager()
    results = mgr.dict()
    mp.start_processes(_peer_worker, args=(world, _free_port(), shape, seed, results), nprocs=world, join=True,
                       start_method="spawn")
    b, z, seq, a = shape
    q, k, v, g = _inputs(b, z, seq, a, seed)
    ch = lambda x: orc.chunks_of(x, world)  # noqa: E731
    outs, probs, _ = orc.ring_forward(ch(q), ch(k), ch(v), exact=False)
    dq, dk, dv, _ = orc.ring_backward(ch(q), ch(k), ch(v), probs, ch(g), exact=False)
    for d in range(world):
        r = results[d]
        assert r["flag"] == 0 and r["same"]
        assert _rel(r["out"], outs[d]) <= 1e-2
        assert np.max(np.abs(r["probs"] - probs[d])) <= 4e-3
        for name, want in (("dq", dq[d]), ("dk", dk[d]), ("dv", dv[d])):
            assert _rel(r[name], want) <= 1e-2, (d, name, _rel(r[name], want))
        c = seq // world
        assert r["ring"] == 3 * 2 * (world - 1) * b * z * c * a + 2 * 2 * (world - 1) * b * z * c * a


def test_bench_multi_rank_arm_runs_under_torchrun():
    """bench.py's N > 1 arm (distributed.bench_main) end to end under torchrun with 2 ranks on
    this one GPU (gloo, host-staged hops: the only multi-rank transport one GPU supports):
    one JSON line from rank 0 with the contract's keys, the step time the max over ranks."""
    import json
    import subprocess
    import sys

    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, RSA_BENCH_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py", "--gpus", "2",
           "--steps", "1", "--warmup", "1", "--layers", "2", "--batch", "4", "--e2e-steps", "1"]
    r = subprocess.run(cmd, cwd=root, env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "weak" and d["value"] > 0
    assert d["config"]["global_batch"] == 8 and d["config"]["ring_ranks"] == 2
    for key in ("clocks", "roofline", "e2e", "gpu_launches"):
        assert key in d
    assert d["e2e"]["h2d_bytes_per_step"] == 2 * 4 * (8 * 12 * 256 * 64 * 2)

"""CPU tests of the host-side mirror: config validation, ledger convention,
sharding, executor resolution (ringseq/config.py, ringseq/cluster.py)."""

from __future__ import annotations

from fractions import Fraction

import numpy as np
import pytest
import torch

import paper_2105_13120_b200 as pkg
from paper_2105_13120_b200.cluster import CommLedger, RingTopology, resolve_executor


def test_config_validation_matches_reference():
    cfg = pkg.AttentionConfig(batch_size=2, seq_len=512, hidden_size=768, num_heads=12, head_size=64, num_devices=4)
    assert cfg.chunk_len == 128
    assert cfg.chunk_shape() == (2, 12, 128, 64) and cfg.panel_shape() == (2, 12, 128, 512)
    with pytest.raises(pkg.ConfigError, match="hidden_size"):
        pkg.AttentionConfig(batch_size=1, seq_len=8, hidden_size=10, num_heads=2, head_size=4)
    with pytest.raises(pkg.ConfigError, match="not divisible"):
        pkg.AttentionConfig(batch_size=1, seq_len=10, hidden_size=8, num_heads=2, head_size=4, num_devices=4)
    for bad in (0, -1, 1.5, "2"):
        with pytest.raises(pkg.ConfigError, match="positive integer"):
            pkg.AttentionConfig(batch_size=bad, seq_len=8, hidden_size=8, num_heads=2, head_size=4)
    with pytest.raises(pkg.ConfigError):
        pkg.SparseAttentionConfig(base=cfg, proj_dim=0)
    assert issubclass(pkg.ShapeError, ValueError) and issubclass(pkg.DeadlockError, pkg.ProtocolError)
    assert issubclass(pkg.StateError, RuntimeError) and issubclass(pkg.NumericError, ValueError)


def test_ring_topology_and_origins():
    topo = RingTopology(4)
    assert [topo.next_device(i) for i in range(4)] == [1, 2, 3, 0]
    assert [topo.prev_device(i) for i in range(4)] == [3, 0, 1, 2]
    # hop h on device d delivers origin (d - h) mod N (ringseq/ring_attention.py:67-79)
    assert [topo.origin_at_hop(1, h) for h in range(4)] == [1, 0, 3, 2]


def test_ledger_convention_and_json():
    led = CommLedger(3)
    led.record_ring_send(0, 10)
    led.record_allreduce(0, 9)  # 2*9*(3-1)/3 = 12
    led.record_allreduce(1, 1)  # 4/3, kept exact
    assert led.devices[0].total_elements() == 22
    assert led.devices[1].allreduce_elements == Fraction(4, 3)
    obj = led.as_json_obj()
    assert obj[1]["allreduce_elements"] == "4/3" and obj[0]["total_bytes"] == 176
    other = CommLedger(3)
    other.record_ring_send(0, 10, wire_bytes=999)  # wire bytes are not part of equality
    other.record_allreduce(0, 9)
    other.record_allreduce(1, 1)
    assert led == other
    assert led.merge(other).devices[0].ring_p2p_elements == 20


def test_scatter_gather_roundtrip_numpy_and_torch():
    x = np.arange(2 * 3 * 8 * 4, dtype=np.float64).reshape(2, 3, 8, 4)
    shards = pkg.scatter_sequence(x, 4)
    assert [s.chunk.shape for s in shards] == [(2, 3, 2, 4)] * 4
    assert np.array_equal(pkg.gather_sequence(shards), x)
    assert np.array_equal(pkg.gather_sequence(list(reversed(shards))), x)
    t = torch.arange(24.0).reshape(2, 12, 1)
    assert torch.equal(pkg.gather_sequence(pkg.scatter_sequence(t, 3)), t)
    with pytest.raises(pkg.ConfigError):
        pkg.scatter_sequence(x, 3)
    with pytest.raises(pkg.ShapeError):
        pkg.gather_sequence([])
    with pytest.raises(pkg.ShapeError):
        pkg.gather_sequence(shards[1:])


def test_executor_resolution(monkeypatch):
    monkeypatch.delenv("RINGSEQ_EXECUTOR", raising=False)
    assert resolve_executor() == "sequential"
    monkeypatch.setenv("RINGSEQ_EXECUTOR", "concurrent")
    assert resolve_executor() == "concurrent"
    assert resolve_executor("sequential") == "sequential"
    with pytest.raises(pkg.ConfigError):
        resolve_executor("threads")


def test_cost_report_reconciles_model_and_ledgers():
    """The reference's communication model (ringseq/cost_model.py:122-159, restated in
    cost_report) equals the ledgers the API charges, element for element, including the
    BERT-base points of tests/test_acceptance.py:183-204 (B2 Z12 L512 A64 N4)."""
    from fractions import Fraction

    from paper_2105_13120_b200 import AttentionConfig, SparseAttentionConfig
    from paper_2105_13120_b200.cost_report import comm_volume, reconcile, sparse_comm_volume, wire_bytes

    for b, z, seq, a, n in [(2, 12, 512, 64, 4), (1, 2, 8, 4, 4), (4, 12, 512, 64, 8), (3, 2, 12, 4, 3)]:
        cfg = AttentionConfig(batch_size=b, seq_len=seq, hidden_size=z * a, num_heads=z, head_size=a, num_devices=n)
        rep = reconcile(cfg)
        assert rep["ledger_matches_model"], rep
    cfg = AttentionConfig(batch_size=2, seq_len=512, hidden_size=768, num_heads=12, head_size=64, num_devices=4)
    assert comm_volume(cfg, "forward") == 1179648 and comm_volume(cfg, "backward") == 3538944
    assert comm_volume(cfg) == 4718592
    sp = SparseAttentionConfig(base=AttentionConfig(batch_size=2, seq_len=40, hidden_size=15, num_heads=3,
                                                    head_size=5, num_devices=4), proj_dim=7)
    assert sparse_comm_volume(sp) == Fraction(3 * 2 * 2 * 3 * 7 * 5)
    # the plans: panel mode sends less than the paper's plan, stream mode more than panel mode
    w = {p: sum(wire_bytes(cfg, p).values()) for p in ("paper", "panel", "stream")}
    assert w["panel"] < w["paper"] and w["panel"] < w["stream"]
    rep = reconcile(cfg, measured=wire_bytes(cfg, "panel"), plan="panel")
    assert rep["measured"]["matches_plan"]


def test_dq_accumulator_validation():
    """The one-pass backwards' fp32 dQ accumulator: supplied buffers must match the launch."""
    import torch

    from paper_2105_13120_b200 import engine
    from paper_2105_13120_b200.errors import ShapeError

    shape = (1, 2, 3, 128, 64)
    acc = torch.empty(shape, dtype=torch.float32)
    assert engine._dq_accumulator(acc, shape, acc.device) is acc
    assert engine._dq_accumulator(None, shape, acc.device).shape == shape
    for bad in (torch.empty(shape, dtype=torch.bfloat16), torch.empty((1, 2, 3, 64, 64)),
                torch.empty((1, 2, 3, 64, 128)).transpose(-1, -2)):
        with pytest.raises(ShapeError):
            engine._dq_accumulator(bad, shape, acc.device)

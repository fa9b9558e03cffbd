"""Drop-in fidelity: the reference's own protocol idioms, run against this package with
``results="numpy"`` (the reference's return types) and stated bf16 tolerances.

Restates the behaviours pinned by the reference's tests/test_ring_attention.py (forward
against single-device attention for N in {1, 2, 4}, probability panels as softmax rows,
exact ledgers, executor independence, chunk errors, backward against the oracle, the
StateError for missing panels) exactly as a ``ringseq`` caller writes them: float64 NumPy
chunks in, float64 ndarrays out, ``gather_sequence`` on the outputs, ``fwd.probs`` passed
back to the backward.  Inputs are NOT pre-rounded here (as in the reference tests), so
the gates include bf16 input rounding: max |diff| <= 3e-2 for outputs and gradients
(values are O(1)), <= 1e-2 for probabilities; ledgers exact.
"""

from __future__ import annotations

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

from oracle import ringseq_np as orc

pytestmark = pytest.mark.gpu

TOL = 3e-2
PTOL = 1e-2


@pytest.fixture(autouse=True)
def numpy_results(monkeypatch):
    monkeypatch.setenv("RSA_B200_RESULTS", "numpy")


def _api():
    import paper_2105_13120_b200 as pkg
    from paper_2105_13120_b200 import ring_attention as ra

    return pkg, ra


def _cfg(pkg, b, z, seq, a, n):
    return pkg.AttentionConfig(batch_size=b, seq_len=seq, hidden_size=z * a, num_heads=z, head_size=a, num_devices=n)


def _qkv(cfg, seed):
    rng = orc.make_rng(seed)
    shape = (cfg.batch_size, cfg.num_heads, cfg.seq_len, cfg.head_size)
    return rng.standard_normal(shape), rng.standard_normal(shape), rng.standard_normal(shape)


def _fwd(ra, cfg, seed, executor=None):
    q, k, v = _qkv(cfg, seed)
    n = cfg.num_devices
    fwd = ra.ring_attention_forward(orc.chunks_of(q, n), orc.chunks_of(k, n), orc.chunks_of(v, n), cfg,
                                    executor=executor)
    return q, k, v, fwd


@pytest.mark.parametrize("shape", [(2, 2, 16, 4), (2, 2, 256, 64), (1, 3, 512, 64)])
@pytest.mark.parametrize("n", [1, 2, 4])
def test_forward_matches_single_device_attention(shape, n):
    pkg, ra = _api()
    cfg = _cfg(pkg, *shape, n)
    q, k, v, fwd = _fwd(ra, cfg, seed=100 + n)
    assert all(isinstance(o, np.ndarray) and o.dtype == np.float64 for o in fwd.outputs)
    got = pkg.gather_sequence(fwd.outputs)
    assert isinstance(got, np.ndarray)
    assert np.max(np.abs(got - orc.attention_forward(q, k, v, exact=False))) <= TOL


def test_probability_panels_are_softmax_rows():
    pkg, ra = _api()
    cfg = _cfg(pkg, 1, 2, 384, 64, 3)
    q, k, v, fwd = _fwd(ra, cfg, seed=3)
    want = orc.softmax_rows(orc.matmul(q, np.swapaxes(k, -1, -2), exact=False) / np.sqrt(cfg.head_size))
    for d in range(3):
        lo, hi = d * cfg.chunk_len, (d + 1) * cfg.chunk_len
        p = fwd.probs[d]
        assert isinstance(p, np.ndarray) and p.shape == want[..., lo:hi, :].shape
        assert np.max(np.abs(p - want[..., lo:hi, :])) <= PTOL
        assert np.max(np.abs(p.sum(-1) - 1.0)) <= 1e-2


def test_forward_ledger_is_exact():
    pkg, ra = _api()
    cfg = _cfg(pkg, 1, 2, 8, 4, 4)
    _, _, _, fwd = _fwd(ra, cfg, seed=1)
    per_device = 2 * (cfg.num_devices - 1) * cfg.batch_size * cfg.num_heads * cfg.chunk_len * cfg.head_size
    for traffic in fwd.ledger.devices:
        assert traffic.ring_p2p_elements == per_device == 96
        assert traffic.allreduce_elements == 0


def test_executors_agree_bitwise():
    pkg, ra = _api()
    cfg = _cfg(pkg, 2, 1, 256, 64, 4)
    _, _, _, seq = _fwd(ra, cfg, seed=5, executor="sequential")
    _, _, _, con = _fwd(ra, cfg, seed=5, executor="concurrent")
    for a, b in zip(seq.outputs, con.outputs):
        assert np.array_equal(a, b)
    assert seq.ledger == con.ledger


def test_chunk_errors():
    pkg, ra = _api()
    cfg = _cfg(pkg, 1, 1, 8, 2, 4)
    q, _, _ = _qkv(cfg, 0)
    halves = orc.chunks_of(q, 2)
    with pytest.raises(pkg.ShapeError, match="chunks"):
        ra.ring_attention_forward(halves, halves, halves, cfg)
    cfg2 = _cfg(pkg, 1, 1, 8, 2, 2)
    good = orc.chunks_of(np.zeros((1, 1, 8, 2)), 2)
    bad = orc.chunks_of(np.zeros((1, 1, 8, 3)), 2)
    with pytest.raises(pkg.ShapeError, match="expected"):
        ra.ring_attention_forward(good, bad, good, cfg2)


@pytest.mark.parametrize("n", [1, 2, 4])
def test_backward_matches_oracle_and_ledger(n):
    pkg, ra = _api()
    cfg = _cfg(pkg, 2, 2, 256, 64, n)
    q, k, v, fwd = _fwd(ra, cfg, seed=40 + n)
    g = orc.make_rng(99).standard_normal(q.shape)
    ch = lambda x: orc.chunks_of(x, n)  # noqa: E731
    bwd = ra.ring_attention_backward(ch(q), ch(k), ch(v), fwd.probs, ch(g), cfg)
    want = orc.attention_backward(q, k, v, g, exact=False)
    for got, ref in zip((bwd.grad_q, bwd.grad_k, bwd.grad_v), want):
        assert all(isinstance(x, np.ndarray) for x in got)
        assert np.max(np.abs(pkg.gather_sequence(got) - ref)) <= TOL
    c_el = cfg.batch_size * cfg.num_heads * cfg.chunk_len * cfg.head_size
    for t in bwd.ledger.devices:
        assert t.ring_p2p_elements == 2 * (n - 1) * c_el
        assert float(t.allreduce_elements) == (4 * (n - 1) * c_el if n > 1 else 0)


def test_backward_without_panels_raises_state_error():
    pkg, ra = _api()
    cfg = _cfg(pkg, 1, 1, 8, 2, 2)
    q, k, v = _qkv(cfg, 0)
    ch = lambda x: orc.chunks_of(x, 2)  # noqa: E731
    with pytest.raises(pkg.StateError):
        ra.ring_attention_backward(ch(q), ch(k), ch(v), None, ch(q), cfg)


@settings(max_examples=10, deadline=None)
@given(st.sampled_from([1, 2, 4]), st.integers(1, 2), st.integers(1, 2), st.integers(0, 2**32 - 1))
def test_property_matches_reference(n, b, z, seed):
    pkg, ra = _api()
    cfg = _cfg(pkg, b, z, 8, 2, n)
    q, k, v, fwd = _fwd(ra, cfg, seed=seed)
    got = pkg.gather_sequence(fwd.outputs)
    assert np.max(np.abs(got - orc.attention_forward(q, k, v, exact=False))) <= TOL


def test_stream_mode_keeps_the_numpy_contract():
    pkg, ra = _api()
    cfg = _cfg(pkg, 1, 2, 512, 64, 2)
    q, k, v = _qkv(cfg, 8)
    ch = lambda x: orc.chunks_of(x, 2)  # noqa: E731
    fwd = ra.ring_attention_forward(ch(q), ch(k), ch(v), cfg, mode="stream")
    assert isinstance(fwd.probs[1], np.ndarray)
    g = orc.make_rng(9).standard_normal(q.shape)
    bwd = ra.ring_attention_backward(ch(q), ch(k), ch(v), fwd.probs, ch(g), cfg)
    want = orc.attention_backward(q, k, v, g, exact=False)
    assert np.max(np.abs(pkg.gather_sequence(bwd.grad_q) - want[0])) <= TOL

"""GPU parity of the sequence-sharded Linformer forward (sparse_ring_attention_forward).

Against the reference goldens (bf16-rounded inputs, tests/golden) and the
oracle (oracle/ringseq_np.py::sparse_ring_forward), with the reference's
structural checks: identity projection == dense ring attention
(tests/test_sparse_ring.py:80-94), exact ledger 2(N-1)BZKA (:96-103), the
no-full-length shape audit (:130-150) and the projection/shape errors.
Tolerances as in test_gpu_rsa.py.
"""

from __future__ import annotations

import math

import numpy as np
import pytest
import torch

from conftest import golden_cases
from oracle import ringseq_np as orc

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sp():
    import paper_2105_13120_b200 as pkg
    from paper_2105_13120_b200 import sparse_attention

    return pkg, sparse_attention


def _cfg(pkg, b, z, seq, a, kp, n):
    base = pkg.AttentionConfig(batch_size=b, seq_len=seq, hidden_size=z * a, num_heads=z, head_size=a, num_devices=n)
    return pkg.SparseAttentionConfig(base=base, proj_dim=kp)


def _np(t):
    return t.float().cpu().numpy().astype(np.float64)


def _gate(got, want, rel_tol=1e-2):
    rel = np.linalg.norm(got - want) / np.linalg.norm(want)
    assert rel <= rel_tol, rel
    assert np.max(np.abs(got - want)) <= 2e-2 * max(1.0, np.abs(want).max())


def _draw(b, z, seq, a, kp, seed):
    rng = orc.make_rng(seed)
    q, k, v = (orc.bf16_round(rng.standard_normal((b, z, seq, a))) for _ in range(3))
    s = 1.0 / math.sqrt(seq)
    e = orc.bf16_round(rng.standard_normal((kp, seq)) * s)
    f = orc.bf16_round(rng.standard_normal((kp, seq)) * s)
    return q, k, v, e, f


def test_matches_reference_golden(sp, golden):
    pkg, spm = sp
    for case, want in golden_cases(golden, "sparse_mid").items():
        b, z, seq, a, kp, n, seed = (int(t) for t in case.split("_"))
        q, k, v, e, f = _draw(b, z, seq, a, kp, seed)
        cfg = _cfg(pkg, b, z, seq, a, kp, n)
        ch = lambda x: orc.chunks_of(x, n)  # noqa: E731
        fwd = spm.sparse_ring_attention_forward(ch(q), ch(k), ch(v), pkg.SparseWeights(e, f), cfg)
        _gate(_np(pkg.gather_sequence(fwd.outputs)), want["out"])
        assert [t.ring_p2p_elements for t in fwd.ledger.devices] == list(want["ledger_ring"])


@pytest.mark.parametrize("shape", [(2, 12, 1024, 64, 256, 4), (1, 2, 16, 2, 4, 2), (2, 3, 40, 5, 7, 4),
                                   (1, 2, 2048, 64, 128, 8)])
def test_matches_oracle(sp, shape):
    pkg, spm = sp
    b, z, seq, a, kp, n = shape
    q, k, v, e, f = _draw(b, z, seq, a, kp, seed=seq + n)
    cfg = _cfg(pkg, b, z, seq, a, kp, n)
    ch = lambda x: orc.chunks_of(x, n)  # noqa: E731
    fwd = spm.sparse_ring_attention_forward(ch(q), ch(k), ch(v), pkg.SparseWeights(e, f), cfg)
    want, ring = orc.sparse_ring_forward(ch(q), ch(k), ch(v), e, f, exact=False)
    # the low-rank K'/V' are rounded to bf16 before the attention GEMMs
    _gate(_np(pkg.gather_sequence(fwd.outputs)), np.concatenate(want, -2), rel_tol=1.5e-2)
    assert all(t.ring_p2p_elements == ring for t in fwd.ledger.devices)
    if n > 1 and kp < seq:
        assert spm.full_length_dims(fwd.shape_logs, cfg) == []


def test_identity_projection_matches_dense_ring(sp):
    pkg, spm = sp
    from paper_2105_13120_b200.ring_attention import ring_attention_forward

    b, z, seq, a, n = 1, 2, 256, 64, 2
    q, k, v, _, _ = _draw(b, z, seq, a, 8, seed=13)
    cfg = _cfg(pkg, b, z, seq, a, seq, n)
    ch = lambda x: orc.chunks_of(x, n)  # noqa: E731
    fwd = spm.sparse_ring_attention_forward(ch(q), ch(k), ch(v), pkg.SparseWeights(np.eye(seq), np.eye(seq)), cfg)
    dense = ring_attention_forward(ch(q), ch(k), ch(v), cfg.base)
    _gate(_np(pkg.gather_sequence(fwd.outputs)), _np(pkg.gather_sequence(dense.outputs)))


def test_errors_and_split(sp):
    pkg, spm = sp
    shards = spm.split_projection_columns(np.arange(36.0).reshape(3, 12), 4)
    assert all(s.shape == (3, 3) for s in shards)
    assert np.array_equal(np.concatenate(shards, 1), np.arange(36.0).reshape(3, 12))
    with pytest.raises(pkg.ShapeError, match="not divisible"):
        spm.split_projection_columns(np.zeros((2, 10)), 4)
    with pytest.raises(pkg.ShapeError, match="2-D"):
        spm.split_projection_columns(np.zeros((2, 3, 4)), 1)
    cfg = _cfg(pkg, 1, 1, 8, 2, 3, 2)
    chunks = orc.chunks_of(np.zeros((1, 1, 8, 2)), 2)
    with pytest.raises(pkg.ShapeError, match="projection"):
        spm.sparse_ring_attention_forward(chunks, chunks, chunks, pkg.SparseWeights(np.zeros((3, 6)), np.zeros((3, 8))), cfg)
    bad = [np.zeros((1, 1, 3, 2))] * 2
    with pytest.raises(pkg.ShapeError, match="expected"):
        spm.sparse_ring_attention_forward(chunks, bad, chunks, pkg.SparseWeights(np.zeros((3, 8)), np.zeros((3, 8))), cfg)
    logs = [[(1, 1, 10, 2), (1, 1, 40, 2)], [(4, 10)]]
    assert spm.full_length_dims(logs, _cfg(pkg, 1, 1, 40, 2, 4, 4)) == [(1, 1, 40, 2)]


@pytest.mark.parametrize("shape", [(1, 2, 256, 64, 64, 1), (2, 2, 256, 64, 64, 2), (1, 3, 512, 64, 128, 4),
                                   (2, 3, 40, 5, 7, 4)])
def test_backward_matches_oracle(sp, shape):
    """sparse_ring_attention_backward vs the oracle's chain rule (linformer_backward, pinned by
    finite differences in tests/test_oracle.py) on the same bf16 inputs; every input's gradient."""
    pkg, spm = sp
    b, z, seq, a, kp, n = shape
    q, k, v, e, f = _draw(b, z, seq, a, kp, seed=sum(shape))
    g = orc.bf16_round(orc.make_rng(7).standard_normal((b, z, seq, a)))
    cfg = _cfg(pkg, b, z, seq, a, kp, n)
    ch = lambda x: orc.chunks_of(x, n)  # noqa: E731
    res = spm.sparse_ring_attention_backward(ch(q), ch(k), ch(v), pkg.SparseWeights(e, f), cfg, ch(g))
    torch.cuda.synchronize()
    want = orc.linformer_backward(q, k, v, e, f, g, exact=False)
    cat = lambda xs: np.concatenate([_np(x) for x in xs], axis=-2)  # noqa: E731
    got = [cat(res.grad_q), cat(res.grad_k), cat(res.grad_v), _np(res.grad_key_proj), _np(res.grad_value_proj)]
    for name, val, ref in zip(("dq", "dk", "dv", "dE", "dF"), got, want):
        rel = np.linalg.norm(val - ref) / np.linalg.norm(ref)
        assert rel <= 2e-2, (name, rel)
    per_rank = 2 * (n - 1) * b * z * kp * a
    assert all(t.ring_p2p_elements == per_rank for t in res.ledger.devices)

"""Stream mode (``mode="stream"``): the RSA forward keeps O plus two fp32 numbers per row
(reference point m, row scale r) instead of the (c x L) probability panel, and the
backward recomputes each probability tile on chip (csrc/bwd_stream.cu).

Parity: the float64 oracle with the gates of test_gpu_rsa.py -- and, stronger, bitwise
equality with the panel mode.  Both modes run the same tensor-core products and the same
exp2 rounding (exp2_pack32), and accumulate every sum in the same order, so
``mode="stream"`` must return exactly the outputs, probabilities and gradients of
``mode="panel"`` (ringseq/ring_attention.py:124-217 either way).
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

from oracle import ringseq_np as orc

pytestmark = pytest.mark.gpu

REL_F = 1e-2
MAX_ABS = 2e-2
PROB_ABS = 4e-3


@pytest.fixture(scope="module")
def rsa():
    import paper_2105_13120_b200 as pkg
    from paper_2105_13120_b200 import ring_attention as ra

    return pkg, ra


def _gate(name, got, want):
    got, want = np.asarray(got, np.float64), np.asarray(want, np.float64)
    rel = np.linalg.norm(got - want) / max(np.linalg.norm(want), 1e-30)
    mx = np.max(np.abs(got - want))
    assert rel <= REL_F, f"{name}: relative Frobenius error {rel:.3e}"
    assert mx <= MAX_ABS * max(1.0, np.max(np.abs(want))), f"{name}: max |diff| {mx:.3e}"


def _np(t):
    return t.double().cpu().numpy()


def _inputs(b, z, seq, a, seed):
    rng = orc.make_rng(seed)
    return [orc.bf16_round(rng.standard_normal((b, z, seq, a))) for _ in range(4)]


STREAM_SHAPES = [  # (B, Z, L, N)
    (1, 2, 256, 2),
    (2, 3, 512, 1),
    (2, 3, 512, 4),     # c = 128
    (1, 2, 400, 2),     # c = 200: ragged key and query tiles
    (2, 1, 96, 4),      # c = 24: mostly padding
    (1, 2, 1280, 1),    # 10 key tiles per row
    (1, 2, 2048, 4),    # c = 512, four origins
]


@pytest.mark.parametrize("shape", STREAM_SHAPES)
def test_stream_mode_matches_oracle_and_panel_mode_bitwise(rsa, shape, monkeypatch):
    pkg, ra = rsa
    monkeypatch.setenv("RSA_B200_DETERMINISTIC", "1")  # the fixed-order two-kernel backward
    b, z, seq, n = shape
    a = 64
    q, k, v, g = _inputs(b, z, seq, a, seed=101 + seq + n)
    cfg = pkg.AttentionConfig(batch_size=b, seq_len=seq, hidden_size=z * a, num_heads=z, head_size=a, num_devices=n)
    ch = lambda x: orc.chunks_of(x, n)  # noqa: E731
    fs = ra.ring_attention_forward(ch(q), ch(k), ch(v), cfg, mode="stream")
    bs = ra.ring_attention_backward(ch(q), ch(k), ch(v), fs.probs, ch(g), cfg)
    assert isinstance(fs.probs, ra.StreamPanels)
    assert all(list.__getitem__(fs.probs, d) is None for d in range(n))  # nothing materialised by the backward
    fp = ra.ring_attention_forward(ch(q), ch(k), ch(v), cfg, mode="panel")
    bp = ra.ring_attention_backward(ch(q), ch(k), ch(v), fp.probs, ch(g), cfg)
    torch.cuda.synchronize()
    # bitwise equal to the panel mode
    for d in range(n):
        assert torch.equal(fs.outputs[d], fp.outputs[d])
        assert torch.equal(bs.grad_q[d], bp.grad_q[d])
        assert torch.equal(bs.grad_k[d], bp.grad_k[d])
        assert torch.equal(bs.grad_v[d], bp.grad_v[d])
        assert torch.equal(fs.probs[d], fp.probs[d])  # lazily recomputed panel == saved panel
    # and against the float64 oracle
    outs, probs, _ = orc.ring_forward(ch(q), ch(k), ch(v), exact=False)
    dq, dk, dv, _ = orc.ring_backward(ch(q), ch(k), ch(v), probs, ch(g), exact=False)
    cat = lambda xs: np.concatenate(xs, axis=-2)  # noqa: E731
    _gate("out", _np(pkg.gather_sequence(fs.outputs)), cat(outs))
    for d in range(n):
        assert np.max(np.abs(_np(fs.probs[d]) - probs[d])) <= PROB_ABS
    _gate("dq", _np(pkg.gather_sequence(bs.grad_q)), cat(dq))
    _gate("dk", _np(pkg.gather_sequence(bs.grad_k)), cat(dk))
    _gate("dv", _np(pkg.gather_sequence(bs.grad_v)), cat(dv))
    assert fs.ledger.devices[0].ring_p2p_elements == fp.ledger.devices[0].ring_p2p_elements
    # the default one-pass backward (rsa_bwd_stream_fused: dQ partials added in L2 in arrival
    # order, query tiles walked from a per-item offset): oracle gates, and within bf16
    # rounding of the fixed-order result
    monkeypatch.setenv("RSA_B200_DETERMINISTIC", "0")
    bf = ra.ring_attention_backward(ch(q), ch(k), ch(v), fs.probs, ch(g), cfg)
    torch.cuda.synchronize()
    for name, got, ref, want in (("dq", bf.grad_q, bs.grad_q, dq), ("dk", bf.grad_k, bs.grad_k, dk),
                                 ("dv", bf.grad_v, bs.grad_v, dv)):
        _gate(name, _np(pkg.gather_sequence(got)), cat(want))
        g_, r_ = _np(pkg.gather_sequence(got)), _np(pkg.gather_sequence(ref))
        assert np.linalg.norm(g_ - r_) <= 4e-3 * np.linalg.norm(r_), name


def test_stream_mode_multi_unit_grid_capped(rsa, monkeypatch):
    """Every persistent CTA of both stream kernels walks many items (grid capped at 3)."""
    from paper_2105_13120_b200 import engine
    from paper_2105_13120_b200._native import lib

    monkeypatch.setenv("RSA_B200_DETERMINISTIC", "1")  # the fixed-order panel backward as reference

    dev = torch.device("cuda", 0)
    gen = torch.Generator(device=dev).manual_seed(9)
    tq, tk, tv, tg = (torch.randn((2, 3, 2, 384, 64), generator=gen, device=dev).to(torch.bfloat16)
                      for _ in range(4))
    ref_f = engine.forward(tq, tk, tv, path="fused")
    ref_b = engine.backward(tq, tk, tv, ref_f.panel, tg, outputs=ref_f.out, rowscale=ref_f.rowscale, path="fused")
    lib().rsa_set_max_ctas(3)
    try:
        sf = engine.forward_stream(tq, tk, tv)
        sb = engine.backward_stream(tq, tk, tv, tg, sf.out, sf.rowscale, sf.rowmax, fused=False)
        sfu = engine.backward_stream(tq, tk, tv, tg, sf.out, sf.rowscale, sf.rowmax, fused=True)
        torch.cuda.synchronize()
    finally:
        lib().rsa_set_max_ctas(0)
    assert int(sf.flag.item()) == 0
    assert torch.equal(sf.out, ref_f.out) and torch.equal(sf.rowscale, ref_f.rowscale)
    for x, y in zip(sb, ref_b):
        assert torch.equal(x, y)
    for x, y in zip(sfu, ref_b):  # the one-pass form: same sums in another order
        x, y = x.double(), y.double()
        assert torch.linalg.norm(x - y) <= 4e-3 * torch.linalg.norm(y)


def test_stream_fallback_on_far_row_max(rsa):
    """A row whose max lies 2^369 above its first key tile's max: flag bit 1, the stream
    forward reruns on the true row maxima (rsa_fwd_stats + given reference points) and the
    whole fwd+bwd still matches the oracle."""
    from paper_2105_13120_b200 import engine

    pkg, ra = rsa
    b, z, seq, a, n = 1, 2, 256, 64, 1
    q, k, v, g = _inputs(b, z, seq, a, seed=77)
    q[..., 0, :] = 4.0
    k[..., 200, :] = 4.0
    dev = torch.device("cuda", 0)
    tq, tk, tv = (torch.from_numpy(x[None]).to(dev, torch.bfloat16) for x in (q, k, v))
    res = engine.forward_stream(tq, tk, tv)
    torch.cuda.synchronize()
    assert int(res.flag.item()) == 2
    cfg = pkg.AttentionConfig(batch_size=b, seq_len=seq, hidden_size=z * a, num_heads=z, head_size=a, num_devices=n)
    ch = lambda x: orc.chunks_of(x, n)  # noqa: E731
    fwd = ra.ring_attention_forward(ch(q), ch(k), ch(v), cfg, mode="stream")
    bwd = ra.ring_attention_backward(ch(q), ch(k), ch(v), fwd.probs, ch(g), cfg)
    outs, probs, _ = orc.ring_forward(ch(q), ch(k), ch(v), exact=False)
    dq, dk, dv, _ = orc.ring_backward(ch(q), ch(k), ch(v), probs, ch(g), exact=False)
    cat = lambda xs: np.concatenate(xs, axis=-2)  # noqa: E731
    _gate("out", _np(pkg.gather_sequence(fwd.outputs)), cat(outs))
    assert np.max(np.abs(_np(fwd.probs[0]) - probs[0])) <= PROB_ABS
    _gate("dq", _np(pkg.gather_sequence(bwd.grad_q)), cat(dq))
    _gate("dk", _np(pkg.gather_sequence(bwd.grad_k)), cat(dk))
    _gate("dv", _np(pkg.gather_sequence(bwd.grad_v)), cat(dv))


def test_stream_nonfinite_key_beyond_first_tile(rsa):
    """A -inf key entry outside the first key tile, against queries that are all positive in
    that dimension: every row scores -inf there, so P~ = 0 and the row sum stays finite.  The
    stream forward checks no score after the first tile (the row sum bounds the rest), and
    the key scan in rsa_fwd_factored_ex must still raise NumericError, as the reference's
    softmax_rows does on non-finite scores (ringseq/tensor_ops.py:80-81)."""
    pkg, ra = rsa
    b, z, seq, a, n = 1, 2, 512, 64, 2
    q, k, v, _ = _inputs(b, z, seq, a, seed=79)
    q[..., :, 5] = np.abs(q[..., :, 5]) + 0.5
    k[..., 300, 5] = -np.inf
    cfg = pkg.AttentionConfig(batch_size=b, seq_len=seq, hidden_size=z * a, num_heads=z, head_size=a, num_devices=n)
    ch = lambda x: orc.chunks_of(x, n)  # noqa: E731
    with pytest.raises(pkg.NumericError):
        ra.ring_attention_forward(ch(q), ch(k), ch(v), cfg, mode="stream")
    k[..., 300, 5] = 1.0  # finite again: no error
    ra.ring_attention_forward(ch(q), ch(k), ch(v), cfg, mode="stream")


def test_stream_mode_long_chunk_sampled(rsa):
    """c = 2048 per rank with 8 resident ranks (L = 16K, config 4's chunk): sampled rows and
    keys of two heads against the blockwise oracle; the saved state is O(L) per head."""
    from paper_2105_13120_b200 import engine

    n, b, z, c, a = 8, 1, 2, 2048, 64
    dev = torch.device("cuda", 0)
    gen = torch.Generator(device=dev).manual_seed(78)
    tq, tk, tv, tg = (torch.randn((n, b, z, c, a), generator=gen, device=dev).to(torch.bfloat16) for _ in range(4))
    sf = engine.forward_stream(tq, tk, tv)
    dq, dk, dv = engine.backward_stream(tq, tk, tv, tg, sf.out, sf.rowscale, sf.rowmax)
    torch.cuda.synchronize()
    assert int(sf.flag.item()) == 0
    seq = n * c
    rng = np.random.default_rng(4)
    rows = np.unique(np.concatenate([[0, c - 1, c, seq - 1], rng.integers(0, seq, 124)]))
    keys = np.unique(np.concatenate([[0, 127, 128, seq - 1], rng.integers(0, seq, 124)]))
    head = lambda t, zi: torch.cat([t[d, 0, zi] for d in range(n)], 0).double().cpu().numpy()  # noqa: E731
    for zi in range(z):
        want = orc.attention_head_sampled(head(tq, zi), head(tk, zi), head(tv, zi), head(tg, zi), rows, keys)
        _gate("out", head(sf.out, zi)[rows], want["out"])
        _gate("dq", head(dq, zi)[rows], want["dq"])
        _gate("dk", head(dk, zi)[keys], want["dk"])
        _gate("dv", head(dv, zi)[keys], want["dv"])

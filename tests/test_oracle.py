"""Pin the CPU oracle (oracle/ringseq_np.py) before trusting it.

Three kinds of evidence, all CPU-only:

* golden fixtures produced by the unmodified reference (tests/golden/):
  bitwise equality in exact mode, <= 1e-12 in BLAS mode;
* the reference's own known-answer tests for this path, restated
  (tests/test_tensor_ops.py:88-110, tests/test_reference_models.py:27-49,
  109-118, tests/test_ring_attention.py:78-84, tests/test_acceptance.py:183-204);
* the stdlib-loop cross-check the reference uses (tests/oracles.py:14-64).
"""

from __future__ import annotations

import math

import numpy as np
import pytest

from conftest import golden_cases
from oracle import ringseq_np as orc


def _inputs(b, z, seq, a, seed, n_tensors=4, rounded=False):
    rng = orc.make_rng(seed)
    xs = [rng.standard_normal((b, z, seq, a)) for _ in range(n_tensors)]
    if rounded:
        xs = [orc.bf16_round(x) for x in xs]
    return xs, rng


def _parse(case):
    return tuple(int(t) for t in case.split("_"))


@pytest.mark.parametrize("exact", [True, False])
def test_rsa_small_matches_reference_goldens(golden, exact):
    cases = golden_cases(golden, "rsa_small")
    assert len(cases) >= 7
    for case, want in cases.items():
        b, z, seq, a, n, seed = _parse(case)
        (q, k, v, g), _ = _inputs(b, z, seq, a, seed)
        ch = lambda x: orc.chunks_of(x, n)  # noqa: E731
        outs, probs, ring_f = orc.ring_forward(ch(q), ch(k), ch(v), exact=exact)
        dq, dk, dv, (ring_b, ar_b) = orc.ring_backward(ch(q), ch(k), ch(v), probs, ch(g), exact=exact)
        got = {
            "out": np.concatenate(outs, axis=-2),
            "probs": np.stack(probs),
            "dq": np.concatenate(dq, axis=-2),
            "dk": np.concatenate(dk, axis=-2),
            "dv": np.concatenate(dv, axis=-2),
        }
        for key, val in got.items():
            if exact:
                assert np.array_equal(val, want[key]), (case, key)
            else:
                assert np.max(np.abs(val - want[key])) <= 1e-12, (case, key)
        assert (want["ledger_fwd_ring"] == ring_f).all()
        assert (want["ledger_bwd_ring"] == ring_b).all()
        assert (want["ledger_bwd_ar"] == ar_b).all()


def test_rsa_mid_matches_reference_goldens(golden):
    cases = golden_cases(golden, "rsa_mid")
    assert len(cases) == 2
    for case, want in cases.items():
        b, z, seq, a, n, seed = _parse(case)
        (q, k, v, g), _ = _inputs(b, z, seq, a, seed, rounded=True)
        ch = lambda x: orc.chunks_of(x, n)  # noqa: E731
        outs, probs, _ = orc.ring_forward(ch(q), ch(k), ch(v), exact=False)
        dq, dk, dv, _ = orc.ring_backward(ch(q), ch(k), ch(v), probs, ch(g), exact=False)
        got = {"out": outs, "dq": dq, "dk": dk, "dv": dv}
        for key, parts in got.items():
            val = np.concatenate(parts, axis=-2)
            # fixtures are stored as float32
            assert np.max(np.abs(val - want[key])) <= 1e-5 * max(1.0, np.abs(val).max()), (case, key)
        if "probs" in want:
            assert np.max(np.abs(np.stack(probs) - want["probs"])) <= 1e-6


def test_sparse_matches_reference_goldens(golden):
    for fam, rounded in (("sparse_small", False), ("sparse_mid", True)):
        cases = golden_cases(golden, fam)
        assert cases
        for case, want in cases.items():
            b, z, seq, a, kp, n, seed = _parse(case)
            (q, k, v), rng = _inputs(b, z, seq, a, seed, n_tensors=3, rounded=rounded)
            s = 1.0 / math.sqrt(seq)
            e = rng.standard_normal((kp, seq)) * s
            f = rng.standard_normal((kp, seq)) * s
            if rounded:
                e, f = orc.bf16_round(e), orc.bf16_round(f)
            ch = lambda x: orc.chunks_of(x, n)  # noqa: E731
            outs, ring = orc.sparse_ring_forward(ch(q), ch(k), ch(v), e, f, exact=not rounded)
            got = np.concatenate(outs, axis=-2)
            if rounded:
                assert np.max(np.abs(got - want["out"])) <= 1e-5
            else:
                assert np.array_equal(got, want["out"]), case
            assert (want["ledger_ring"] == ring).all()


# --- the reference's known-answer tests, restated against the oracle -------

def test_softmax_known_answers():
    got = orc.softmax_rows(np.array([[0.0, math.log(3.0)]]))
    assert np.max(np.abs(got - [[0.25, 0.75]])) <= 1e-12
    assert np.max(np.abs(orc.softmax_rows(np.full((2, 4), 3.7)) - 0.25)) <= 1e-12
    assert np.array_equal(orc.softmax_rows(np.array([[1000.0, 1000.0]])), [[0.5, 0.5]])
    with pytest.raises(FloatingPointError):
        orc.softmax_rows(np.array([[0.0, np.inf]]))
    with pytest.raises(FloatingPointError):
        orc.softmax_rows(np.array([[np.nan, 1.0]]))


def test_attention_known_answers():
    got = orc.attention_forward([[0.0], [0.0]], [[1.0], [-1.0]], [[2.0], [4.0]])
    assert np.max(np.abs(got - [[3.0], [3.0]])) <= 1e-12
    eye = np.eye(3) * 50.0
    v = np.arange(9.0).reshape(3, 3)
    assert np.max(np.abs(orc.attention_forward(eye, eye, v) - v)) <= 1e-9
    # uniform probabilities: grad_v is the column mean of g for every row
    rng = orc.make_rng(8)
    g = rng.standard_normal((4, 2))
    _, _, dv = orc.attention_backward(np.zeros((4, 2)), rng.standard_normal((4, 2)),
                                      rng.standard_normal((4, 2)), g)
    assert np.max(np.abs(dv - g.mean(axis=0, keepdims=True))) <= 1e-12


def _loop_matmul(a, b):
    out = np.zeros((a.shape[0], b.shape[1]))
    for i in range(a.shape[0]):
        for j in range(b.shape[1]):
            acc = 0.0
            for k in range(a.shape[1]):
                acc += a[i, k] * b[k, j]
            out[i, j] = acc
    return out


def test_matmul_exact_equals_triple_loop():
    rng = orc.make_rng(13)
    a = rng.standard_normal((5, 7))
    b = rng.standard_normal((7, 3))
    assert np.array_equal(orc.matmul(a, b), _loop_matmul(a, b))


def test_single_device_ring_is_bitwise_attention():
    (q, k, v, g), _ = _inputs(1, 2, 8, 4, 7)
    outs, probs, ring = orc.ring_forward([q], [k], [v])
    assert np.array_equal(outs[0], orc.attention_forward(q, k, v))
    assert ring == 0
    dq, dk, dv, _ = orc.ring_backward([q], [k], [v], probs, [g])
    want = orc.attention_backward(q, k, v, g)
    for got, ref in zip((dq[0], dk[0], dv[0]), want):
        assert np.max(np.abs(got - ref)) <= 1e-12


def test_bert_base_ledger_point():
    # tests/test_acceptance.py:183-204: B2 Z12 L512 A64 N4
    chunk = 2 * 12 * 128 * 64
    assert orc.ledger_forward(4, chunk) == 1_179_648
    ring, ar = orc.ledger_backward(4, chunk)
    assert ring + ar == 3_538_944
    assert orc.ledger_forward(4, chunk) + ring + ar == 4_718_592


def test_bf16_round_is_idempotent_and_nearest():
    x = orc.make_rng(0).standard_normal(1000)
    r = orc.bf16_round(x)
    assert np.array_equal(orc.bf16_round(r), r)
    assert np.max(np.abs(r - x) / np.abs(x)) <= 2.0 ** -8


def layer_inputs(b, seq, z, a, seed, rounded=False):
    """x, grad_out and the weights exactly as tests/golden/make_golden.py:layer_case draws them
    (ringseq/reference.py:207-216: wq, wk, wv ~ N(0,1)/sqrt(H) of (H, Z*A), wo of (Z*A, H))."""
    h = z * a
    rng = orc.make_rng(seed)
    x = rng.standard_normal((b, seq, h))
    g = rng.standard_normal((b, seq, h))
    s = 1.0 / math.sqrt(h)
    ws = [rng.standard_normal(shape) * s for shape in ((h, h), (h, h), (h, h), (h, h))]
    if rounded:
        x, g = orc.bf16_round(x), orc.bf16_round(g)
        ws = [orc.bf16_round(w) for w in ws]
    return x, g, ws


@pytest.mark.parametrize("exact", [True, False])
def test_layer_forward_backward_match_reference_goldens(golden, exact):
    """multi_head_forward / multi_head_backward (ringseq/reference.py:122-174)."""
    cases = golden_cases(golden, "layer_small")
    assert cases
    for case, want in cases.items():
        b, seq, z, a, seed = _parse(case)
        x, g, ws = layer_inputs(b, seq, z, a, seed)
        y = orc.multi_head_forward(x, *ws, num_heads=z, exact=exact)
        gx, gwq, gwk, gwv, gwo = orc.multi_head_backward(x, *ws, g, num_heads=z, exact=exact)
        got = {"y": y, "grad_x": gx, "grad_wq": gwq, "grad_wk": gwk, "grad_wv": gwv, "grad_wo": gwo}
        for key, val in got.items():
            if exact:
                assert np.array_equal(val, want[key]), (case, key)
            else:
                assert np.max(np.abs(val - want[key])) <= 1e-12, (case, key)


def test_layer_backward_finite_differences():
    """grad_x and grad_wq of multi_head_backward against central differences of
    multi_head_forward (the reference's own gradient check style, tests/test_acceptance.py:99-147)."""
    b, seq, z, a = 1, 6, 2, 3
    x, g, ws = layer_inputs(b, seq, z, a, seed=8)
    gx, gwq, _, _, _ = orc.multi_head_backward(x, *ws, g, num_heads=z, exact=False)
    loss = lambda xx, wq: float(np.sum(orc.multi_head_forward(xx, wq, *ws[1:], num_heads=z, exact=False) * g))  # noqa: E731
    eps = 1e-6
    for idx in [(0, 0, 0), (0, 3, 5), (0, 5, 2)]:
        d = np.zeros_like(x)
        d[idx] = eps
        fd = (loss(x + d, ws[0]) - loss(x - d, ws[0])) / (2 * eps)
        assert abs(fd - gx[idx]) <= 1e-6 * max(1.0, abs(fd))
    for idx in [(0, 0), (4, 1), (5, 5)]:
        d = np.zeros_like(ws[0])
        d[idx] = eps
        fd = (loss(x, ws[0] + d) - loss(x, ws[0] - d)) / (2 * eps)
        assert abs(fd - gwq[idx]) <= 1e-6 * max(1.0, abs(fd))


def test_linformer_backward_finite_differences():
    """linformer_backward against central differences of linformer_forward (every input,
    including the shared projections)."""
    b, z, seq, a, kp = 2, 2, 12, 3, 5
    rng = orc.make_rng(71)
    q, k, v, g = (rng.standard_normal((b, z, seq, a)) for _ in range(4))
    e, f = (rng.standard_normal((kp, seq)) / math.sqrt(seq) for _ in range(2))
    grads = orc.linformer_backward(q, k, v, e, f, g, exact=False)
    args = [q, k, v, e, f]

    def loss(xs):
        return float(np.sum(orc.linformer_forward(*xs, exact=False) * g))

    eps = 1e-6
    for which, grad in enumerate(grads):
        x = args[which]
        for flat in (0, x.size // 2, x.size - 1):
            idx = np.unravel_index(flat, x.shape)
            d = np.zeros_like(x)
            d[idx] = eps
            plus = [y + d if i == which else y for i, y in enumerate(args)]
            minus = [y - d if i == which else y for i, y in enumerate(args)]
            fd = (loss(plus) - loss(minus)) / (2 * eps)
            assert abs(fd - grad[idx]) <= 1e-6 * max(1.0, abs(fd)), (which, idx, fd, grad[idx])


def mlp_inputs(b, seq, h, seed, rounded=False):
    """x and MlpWeights as tests/golden/make_golden.py:mlp_case draws them
    (ringseq/reference.py:219-224: up ~ N(0,1)/sqrt(H) of (H, 4H), down ~ N(0,1)/(2 sqrt(H)))."""
    rng = orc.make_rng(seed)
    x = rng.standard_normal((b, seq, h))
    s = 1.0 / math.sqrt(h)
    up = rng.standard_normal((h, 4 * h)) * s
    down = rng.standard_normal((4 * h, h)) * (s / 2.0)
    if rounded:
        x, up, down = orc.bf16_round(x), orc.bf16_round(up), orc.bf16_round(down)
    return x, up, down


@pytest.mark.parametrize("exact", [True, False])
def test_mlp_forward_matches_reference_goldens(golden, exact):
    cases = golden_cases(golden, "mlp_small")
    assert cases
    for case, want in cases.items():
        b, seq, h, seed = _parse(case)
        x, up, down = mlp_inputs(b, seq, h, seed)
        y = orc.mlp_forward(x, up, down, exact=exact)
        if exact:
            assert np.array_equal(y, want["y"]), case
        else:
            assert np.max(np.abs(y - want["y"])) <= 1e-12


def test_mlp_backward_finite_differences():
    b, seq, h = 1, 5, 3
    x, up, down = mlp_inputs(b, seq, h, seed=35)
    g = orc.make_rng(36).standard_normal((b, seq, h))
    grads = orc.mlp_backward(x, up, down, g, exact=False)
    args = [x, up, down]

    def loss(xs):
        return float(np.sum(orc.mlp_forward(*xs, exact=False) * g))

    eps = 1e-6
    for which, grad in enumerate(grads):
        arr = args[which]
        for flat in (0, arr.size // 2, arr.size - 1):
            idx = np.unravel_index(flat, arr.shape)
            d = np.zeros_like(arr)
            d[idx] = eps
            plus = [y + d if i == which else y for i, y in enumerate(args)]
            minus = [y - d if i == which else y for i, y in enumerate(args)]
            fd = (loss(plus) - loss(minus)) / (2 * eps)
            assert abs(fd - grad[idx]) <= 1e-6 * max(1.0, abs(fd)), (which, idx)


def test_attention_head_sampled_matches_dense_oracle():
    """The blockwise sampled-head oracle (used by the large-geometry GPU tests and by
    bench.py's parity field) against the dense attention oracle."""
    rng = orc.make_rng(5)
    seq, a = 300, 16
    q, k, v, g = (rng.standard_normal((seq, a)) for _ in range(4))
    rows, keys = [0, 7, 128, 299], [1, 64, 250]
    got = orc.attention_head_sampled(q, k, v, g, rows, keys, block=64)
    out = orc.attention_forward(q, k, v, exact=False)
    dq, dk, dv = orc.attention_backward(q, k, v, g, exact=False)
    probs = orc.softmax_rows(orc.matmul(q, k.T, exact=False) / np.sqrt(a))
    for name, want in (("out", out[rows]), ("probs", probs[rows]), ("dq", dq[rows]), ("dk", dk[keys]),
                       ("dv", dv[keys])):
        assert np.max(np.abs(got[name] - want)) <= 1e-12, name

"""GPU parity of the RSA path against the CPU oracle and the reference goldens.

Inputs are drawn exactly like the reference tests (make_rng(seed) normals,
q, k, v, grad in that order -- tests/test_acceptance.py:59-67), rounded to
bf16, and fed to both the device path and the float64 oracle, so the gates
measure kernel error only.

Tolerances (bf16 operands, fp32 accumulation, bf16 P and dS; derivation in
SURVEY.md section 8c and DESIGN.md "Numerics"):
  outputs / dq / dk / dv : relative Frobenius error <= 1e-2 and
                           max |diff| <= 2e-2 * max(1, max |ref|)
  probability panels     : max |diff| <= 4e-3 (one bf16 ulp at 1.0)
Ledgers are integers and must match exactly.
"""

from __future__ import annotations

import math

import numpy as np
import pytest
import torch

from conftest import golden_cases
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


def _cfg(pkg, b, z, seq, a, n):
    return pkg.AttentionConfig(batch_size=b, seq_len=seq, hidden_size=z * a, num_heads=z, head_size=a, num_devices=n)


def _inputs(b, z, seq, a, seed):
    rng = orc.make_rng(seed)
    return [orc.bf16_round(rng.standard_normal((b, z, seq, a))) for _ in range(4)]


def _np(t):
    return t.float().cpu().numpy().astype(np.float64)


def _gate(name, got, want):
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    assert got.shape == want.shape, (name, got.shape, want.shape)
    rel = np.linalg.norm(got - want) / max(np.linalg.norm(want), 1e-30)
    mx = np.max(np.abs(got - want))
    assert rel <= REL_F, f"{name}: relative Frobenius error {rel:.3e}"
    assert mx <= MAX_ABS * max(1.0, np.max(np.abs(want))), f"{name}: max |diff| {mx:.3e}"


def _run(pkg, ra, q, k, v, g, n, path):
    b, z, seq, a = q.shape
    cfg = _cfg(pkg, b, z, seq, a, n)
    ch = lambda x: orc.chunks_of(x, n)  # noqa: E731
    fwd = ra.ring_attention_forward(ch(q), ch(k), ch(v), cfg, path=path)
    bwd = ra.ring_attention_backward(ch(q), ch(k), ch(v), fwd.probs, ch(g), cfg, path=path)
    torch.cuda.synchronize()
    return cfg, fwd, bwd


def _oracle(q, k, v, g, n):
    ch = lambda x: orc.chunks_of(x, n)  # noqa: E731
    outs, probs, _ = orc.ring_forward(ch(q), ch(k), ch(v), exact=False)
    dq, dk, dv, _ = orc.ring_backward(ch(q), ch(k), ch(v), probs, ch(g), exact=False)
    cat = lambda xs: np.concatenate(xs, axis=-2)  # noqa: E731
    return cat(outs), probs, cat(dq), cat(dk), cat(dv)


def _check_all(pkg, fwd, bwd, want):
    out, probs, dq, dk, dv = want
    _gate("out", _np(pkg.gather_sequence(fwd.outputs)), out)
    for d, p in enumerate(fwd.probs):
        diff = np.max(np.abs(_np(p) - probs[d]))
        assert diff <= PROB_ABS, f"probs[{d}] max |diff| {diff:.3e}"
    _gate("dq", _np(pkg.gather_sequence(bwd.grad_q)), dq)
    _gate("dk", _np(pkg.gather_sequence(bwd.grad_k)), dk)
    _gate("dv", _np(pkg.gather_sequence(bwd.grad_v)), dv)


@pytest.mark.parametrize("path", ["fused", "staged"])
def test_matches_reference_goldens(rsa, golden, path):
    """Device results vs outputs of the unmodified reference on the same bf16 inputs."""
    pkg, ra = rsa
    for case, want in golden_cases(golden, "rsa_mid").items():
        b, z, seq, a, n, seed = (int(t) for t in case.split("_"))
        q, k, v, g = _inputs(b, z, seq, a, seed)
        _, fwd, bwd = _run(pkg, ra, q, k, v, g, n, path)
        _gate("out", _np(pkg.gather_sequence(fwd.outputs)), want["out"])
        _gate("dq", _np(pkg.gather_sequence(bwd.grad_q)), want["dq"])
        _gate("dk", _np(pkg.gather_sequence(bwd.grad_k)), want["dk"])
        _gate("dv", _np(pkg.gather_sequence(bwd.grad_v)), want["dv"])
        if "probs" in want:
            got = np.stack([_np(p) for p in fwd.probs])
            assert np.max(np.abs(got - want["probs"])) <= PROB_ABS


# (B, Z, L, A, N): BERT-base heads at config-1 length, ragged chunk tails
# (c = 200, 24), c = 64 (N = 8), and a single rank.
FUSED_SHAPES = [
    (2, 3, 512, 64, 4),
    (1, 2, 400, 64, 2),
    (1, 2, 512, 64, 8),
    (2, 1, 96, 64, 4),
    (1, 2, 384, 64, 1),
]


@pytest.mark.parametrize("shape", FUSED_SHAPES)
@pytest.mark.parametrize("path", ["fused", "staged"])
def test_matches_oracle(rsa, shape, path):
    pkg, ra = rsa
    b, z, seq, a, n = shape
    q, k, v, g = _inputs(b, z, seq, a, seed=sum(shape))
    _, fwd, bwd = _run(pkg, ra, q, k, v, g, n, path)
    _check_all(pkg, fwd, bwd, _oracle(q, k, v, g, n))


# The reference's own small grid (tests/test_acceptance.py:44-50 style shapes,
# head sizes 2..8) runs on the staged path (SIMT GEMM for unaligned heads).
SMALL_SHAPES = [(1, 2, 8, 4, 1), (1, 2, 12, 4, 3), (2, 2, 16, 4, 4), (1, 1, 8, 2, 2), (2, 3, 40, 5, 4),
                (2, 4, 32, 8, 8), (1, 2, 24, 3, 3)]


@pytest.mark.parametrize("shape", SMALL_SHAPES)
def test_small_reference_shapes(rsa, shape):
    pkg, ra = rsa
    b, z, seq, a, n = shape
    q, k, v, g = _inputs(b, z, seq, a, seed=7 + seq)
    _, fwd, bwd = _run(pkg, ra, q, k, v, g, n, "auto")
    _check_all(pkg, fwd, bwd, _oracle(q, k, v, g, n))


def test_fused_and_staged_agree(rsa):
    pkg, ra = rsa
    q, k, v, g = _inputs(2, 2, 256, 64, seed=5)
    _, f1, b1 = _run(pkg, ra, q, k, v, g, 2, "fused")
    _, f2, b2 = _run(pkg, ra, q, k, v, g, 2, "staged")
    for x, y in zip(f1.probs, f2.probs):
        assert np.max(np.abs(_np(x) - _np(y))) <= PROB_ABS
    for xs, ys in ((f1.outputs, f2.outputs), (b1.grad_q, b2.grad_q), (b1.grad_k, b2.grad_k), (b1.grad_v, b2.grad_v)):
        _gate("fused-vs-staged", _np(pkg.gather_sequence(xs)), _np(pkg.gather_sequence(ys)))


def test_probability_panels_are_rank_invariant(rsa):
    """ringseq tests/test_ring_attention.py:67-76: each rank's panel equals the
    matching rows of the single-device panel.  With c a multiple of the
    128-key tile the fused kernels reduce in the same order for every N, so the
    panels agree bitwise."""
    pkg, ra = rsa
    q, k, v, g = _inputs(1, 2, 512, 64, seed=3)
    _, f1, _ = _run(pkg, ra, q, k, v, g, 1, "fused")
    _, f4, _ = _run(pkg, ra, q, k, v, g, 4, "fused")
    full = f1.probs[0]
    for d in range(4):
        assert torch.equal(f4.probs[d], full[..., d * 128:(d + 1) * 128, :])


def test_single_rank_matches_attention_oracle(rsa):
    pkg, ra = rsa
    q, k, v, g = _inputs(1, 2, 256, 64, seed=11)
    _, fwd, bwd = _run(pkg, ra, q, k, v, g, 1, "auto")
    _gate("out", _np(fwd.outputs[0]), orc.attention_forward(q, k, v, exact=False))
    want = orc.attention_backward(q, k, v, g, exact=False)
    for got, ref, name in zip((bwd.grad_q[0], bwd.grad_k[0], bwd.grad_v[0]), want, "qkv"):
        _gate("d" + name, _np(got), ref)


def test_ledgers_are_exact(rsa):
    pkg, ra = rsa
    # tests/test_acceptance.py:183-204: B2 Z12 L512 A64 N4
    q, k, v, g = _inputs(2, 12, 512, 64, seed=0)
    _, fwd, bwd = _run(pkg, ra, q, k, v, g, 4, "auto")
    for t in fwd.ledger.devices:
        assert t.total_elements() == 1_179_648
    for t in bwd.ledger.devices:
        assert t.total_elements() == 3_538_944
        assert t.ring_p2p_elements == 2 * 3 * 2 * 12 * 128 * 64
    # tests/test_ring_attention.py:78-84
    q, k, v, g = _inputs(1, 2, 8, 4, seed=1)
    _, fwd, _ = _run(pkg, ra, q, k, v, g, 4, "auto")
    assert all(t.ring_p2p_elements == 96 for t in fwd.ledger.devices)
    _, fwd1, bwd1 = _run(pkg, ra, q, k, v, g, 1, "auto")
    assert fwd1.ledger.total_elements() == 0 and bwd1.ledger.total_elements() == 0


def test_errors_match_reference(rsa):
    pkg, ra = rsa
    cfg = _cfg(pkg, 1, 1, 8, 2, 4)
    x = orc.make_rng(0).standard_normal((1, 1, 8, 2))
    halves = orc.chunks_of(x, 2)
    with pytest.raises(pkg.ShapeError, match="chunks"):
        ra.ring_attention_forward(halves, halves, halves, cfg)
    cfg2 = _cfg(pkg, 1, 1, 8, 2, 2)
    good = orc.chunks_of(np.zeros((1, 1, 8, 2)), 2)
    bad = orc.chunks_of(np.zeros((1, 1, 8, 3)), 2)
    with pytest.raises(pkg.ShapeError, match="expected"):
        ra.ring_attention_forward(good, bad, good, cfg2)
    cfg3 = _cfg(pkg, 1, 1, 4, 2, 2)
    ch = orc.chunks_of(np.zeros((1, 1, 4, 2)), 2)
    with pytest.raises(pkg.StateError, match="saved"):
        ra.ring_attention_backward(ch, ch, ch, None, ch, cfg3)
    with pytest.raises(pkg.ShapeError, match="probs"):
        ra.ring_attention_backward(ch, ch, ch, [np.zeros((1, 1, 2, 2))] * 2, ch, cfg3)
    with pytest.raises(pkg.ConfigError):
        ra.ring_attention_forward(ch, ch, ch, cfg3, executor="bogus")


@pytest.mark.parametrize("path", ["fused", "staged"])
def test_nonfinite_input_raises_numeric_error(rsa, path):
    pkg, ra = rsa
    q, k, v, _ = _inputs(1, 1, 128, 64, seed=2)
    q[0, 0, 3, 5] = np.inf
    cfg = _cfg(pkg, 1, 1, 128, 64, 2)
    ch = lambda x: orc.chunks_of(x, 2)  # noqa: E731
    with pytest.raises(pkg.NumericError):
        ra.ring_attention_forward(ch(q), ch(k), ch(v), cfg, path=path)


def test_executor_choice_does_not_change_results(rsa):
    pkg, ra = rsa
    q, k, v, _ = _inputs(1, 2, 256, 64, seed=4)
    cfg = _cfg(pkg, 1, 2, 256, 64, 4)
    ch = lambda x: orc.chunks_of(x, 4)  # noqa: E731
    a = ra.ring_attention_forward(ch(q), ch(k), ch(v), cfg, executor="sequential")
    b = ra.ring_attention_forward(ch(q), ch(k), ch(v), cfg, executor="concurrent")
    for x, y in zip(a.outputs + list(a.probs), b.outputs + list(b.probs)):
        assert torch.equal(x, y)
    assert a.ledger == b.ledger


def test_layer_wrapper_matches_multi_head_oracle(rsa):
    pkg, ra = rsa
    b, seq, z, a, n = 2, 256, 2, 64, 4
    h = z * a
    rng = orc.make_rng(60)
    x = orc.bf16_round(rng.standard_normal((b, seq, h)))
    s = 1.0 / math.sqrt(h)
    ws = [orc.bf16_round(rng.standard_normal((h, h)) * s) for _ in range(4)]
    cfg = pkg.AttentionConfig(batch_size=b, seq_len=seq, hidden_size=h, num_heads=z, head_size=a, num_devices=n)
    w = pkg.AttentionWeights(*ws)
    results, ledger = ra.sequence_parallel_attention(orc.chunks_of(x, n), w, cfg)
    want = orc.multi_head_forward(x, *ws, num_heads=z, exact=False)
    # two extra bf16 roundings (projections, merged heads) before the output GEMM
    got = _np(pkg.gather_sequence(results))
    rel = np.linalg.norm(got - want) / np.linalg.norm(want)
    assert rel <= 2e-2, rel
    assert all(t.ring_p2p_elements == 2 * (n - 1) * b * z * (seq // n) * a for t in ledger.devices)


def _layer_inputs(b, seq, z, a, seed):
    """As tests/golden/make_golden.py:layer_case draws them, bf16-rounded."""
    h = z * a
    rng = orc.make_rng(seed)
    x, g = (orc.bf16_round(rng.standard_normal((b, seq, h))) for _ in range(2))
    s = 1.0 / math.sqrt(h)
    ws = [orc.bf16_round(rng.standard_normal((h, h)) * s) for _ in range(4)]
    return x, g, ws


# activations pass through extra bf16 roundings (projections, merged heads, dO*r) before
# the projection GEMMs, so the layer gates are looser than the attention-core gates
LAYER_REL = 2e-2


@pytest.mark.parametrize("n", [1, 2, 4])
def test_layer_backward_matches_reference_golden(rsa, golden, n):
    """sequence_parallel_attention_backward vs the unmodified reference's multi_head_backward
    (ringseq/reference.py:133-174) on the same bf16 inputs, for 1, 2 and 4 ring ranks."""
    pkg, ra = rsa
    cases = golden_cases(golden, "layer_mid")
    assert cases
    for case, want in cases.items():
        b, seq, z, a, seed = (int(t) for t in case.split("_"))
        x, g, ws = _layer_inputs(b, seq, z, a, seed)
        cfg = pkg.AttentionConfig(batch_size=b, seq_len=seq, hidden_size=z * a, num_heads=z, head_size=a,
                                  num_devices=n)
        w = pkg.AttentionWeights(*ws)
        y, _ = ra.sequence_parallel_attention(orc.chunks_of(x, n), w, cfg)
        gx, gw, ledger = ra.sequence_parallel_attention_backward(orc.chunks_of(x, n), w, cfg, orc.chunks_of(g, n))
        torch.cuda.synchronize()
        got = {"y": _np(pkg.gather_sequence(y)), "grad_x": _np(pkg.gather_sequence(gx)),
               "grad_wq": _np(gw.wq), "grad_wk": _np(gw.wk), "grad_wv": _np(gw.wv), "grad_wo": _np(gw.wo)}
        for key, val in got.items():
            ref = want[key].astype(np.float64)
            rel = np.linalg.norm(val - ref) / np.linalg.norm(ref)
            assert rel <= LAYER_REL, (key, rel)
        c = seq // n
        for t in ledger.devices:
            assert t.ring_p2p_elements == 2 * (n - 1) * b * z * c * a
        if n > 1:
            h = z * a
            want_ar = 2 * (n - 1) * b * z * seq * a * 2 / n + 2 * 4 * h * h * (n - 1) / n
            assert all(float(t.allreduce_elements) == want_ar for t in ledger.devices)


def test_layer_backward_matches_oracle_bench_like(rsa):
    """BERT-base-like heads (A = 64) at a ragged chunk length, against the float64 oracle."""
    pkg, ra = rsa
    b, seq, z, a, n = 1, 384, 3, 64, 2
    x, g, ws = _layer_inputs(b, seq, z, a, seed=90)
    cfg = pkg.AttentionConfig(batch_size=b, seq_len=seq, hidden_size=z * a, num_heads=z, head_size=a, num_devices=n)
    gx, gw, _ = ra.sequence_parallel_attention_backward(orc.chunks_of(x, n), pkg.AttentionWeights(*ws), cfg,
                                                        orc.chunks_of(g, n))
    want = orc.multi_head_backward(x, *ws, g, num_heads=z, exact=False)
    got = [_np(pkg.gather_sequence(gx)), _np(gw.wq), _np(gw.wk), _np(gw.wv), _np(gw.wo)]
    for name, val, ref in zip(("grad_x", "grad_wq", "grad_wk", "grad_wv", "grad_wo"), got, want):
        rel = np.linalg.norm(val - ref) / np.linalg.norm(ref)
        assert rel <= LAYER_REL, (name, rel)


# Single-pass backward (rsa_bwd_fused) vs the split rsa_bwd_dkdv + rsa_bwd_dq
# pair, both against the oracle: every geometry with <= 4 query tiles per head
# (resident N ranks x ceil(c/128)), including ragged tails and the bench shape.
SINGLE_PASS_SHAPES = [
    (2, 2, 512, 64, 1),   # bench geometry: 4 row tiles of one rank
    (2, 3, 512, 64, 4),   # c = 128: 4 ranks x 1 tile
    (1, 2, 400, 64, 2),   # c = 200: ragged second tile
    (2, 1, 96, 64, 4),    # c = 24: mostly padding
    (1, 3, 384, 64, 1),   # 3 tiles
    (3, 2, 128, 64, 1),   # one tile, several heads per CTA walk
]


@pytest.mark.parametrize("shape", SINGLE_PASS_SHAPES)
@pytest.mark.parametrize("single_pass", [True, False])
@pytest.mark.parametrize("factored", [True, False])
def test_backward_kernels_match_oracle(rsa, shape, single_pass, factored):
    from paper_2105_13120_b200 import engine

    b, z, seq, a, n = shape
    c = seq // n
    assert engine.single_pass_supported(n, b, z, c, a)
    q, k, v, g = _inputs(b, z, seq, a, seed=31 + sum(shape))
    dev = torch.device("cuda", 0)
    stack = lambda x: torch.from_numpy(np.stack(orc.chunks_of(x, n))).to(dev, torch.bfloat16)  # noqa: E731
    tq, tk, tv, tg = (stack(x) for x in (q, k, v, g))
    out, panel, rowscale, _ = engine.forward(tq, tk, tv, path="fused", factored=factored)
    assert (rowscale is not None) == factored
    dq, dk, dv = engine.backward(tq, tk, tv, panel, tg, outputs=out, rowscale=rowscale, path="fused",
                                 single_pass=single_pass)
    torch.cuda.synchronize()
    wout, wprobs, wdq, wdk, wdv = _oracle(q, k, v, g, n)
    _gate("out", np.concatenate([_np(out[d]) for d in range(n)], axis=-2), wout)
    for d in range(n):
        got = _np(engine.normalized_panel(panel[d], None if rowscale is None else rowscale[d]))
        assert np.max(np.abs(got - wprobs[d])) <= PROB_ABS
    cat = lambda t: np.concatenate([_np(t[d]) for d in range(n)], axis=-2)  # noqa: E731
    _gate("dq", cat(dq), wdq)
    _gate("dk", cat(dk), wdk)
    _gate("dv", cat(dv), wdv)


def test_single_pass_backward_is_deterministic(rsa):
    from paper_2105_13120_b200 import engine

    dev = torch.device("cuda", 0)
    gen = torch.Generator(device=dev).manual_seed(4)
    tq, tk, tv, tg = (torch.randn((1, 4, 3, 512, 64), generator=gen, device=dev).to(torch.bfloat16) for _ in range(4))
    out, panel, rowscale, _ = engine.forward(tq, tk, tv, path="fused")
    r1 = engine.backward(tq, tk, tv, panel, tg, outputs=out, rowscale=rowscale, path="fused", single_pass=True)
    r2 = engine.backward(tq, tk, tv, panel, tg, outputs=out, rowscale=rowscale, path="fused", single_pass=True)
    torch.cuda.synchronize()
    for x, y in zip(r1, r2):
        assert torch.equal(x, y)


def test_factored_panel_matches_normalised_kernel(rsa):
    """rsa_fwd_factored vs rsa_fwd_resident on the same inputs: r * P~ equals the
    normalised panel to bf16 rounding, outputs agree, and every factored row
    sums to one (the tensor-core row sum counts exactly the stored values)."""
    # (c = 256: each row's first key tile is keys 0..127 of origin 0)
    from paper_2105_13120_b200 import engine

    dev = torch.device("cuda", 0)
    gen = torch.Generator(device=dev).manual_seed(9)
    tq, tk, tv = (torch.randn((2, 2, 3, 256, 64), generator=gen, device=dev).to(torch.bfloat16) for _ in range(3))
    f = engine.forward(tq, tk, tv, path="fused", factored=True)
    n = engine.forward(tq, tk, tv, path="fused", factored=False)
    torch.cuda.synchronize()
    assert f.rowscale is not None and n.rowscale is None
    p_f = engine.normalized_panel(f.panel, f.rowscale)
    assert float((p_f - n.panel.float()).abs().max()) <= PROB_ABS
    assert float((f.out.float() - n.out.float()).abs().max()) <= 2e-2
    rows = (f.panel.float().sum(-1) * f.rowscale)
    assert float((rows - 1).abs().max()) <= 1e-4
    # the reference point is the row max over the first key tile, which maps to 2^0 exactly
    assert torch.all(f.panel[..., :128].float().amax(-1) == 1.0)


def test_rowdot_scale_and_panel_normalize(rsa):
    from paper_2105_13120_b200 import tensor_ops as ops

    dev = torch.device("cuda", 0)
    gen = torch.Generator(device=dev).manual_seed(5)
    for cols in (64, 40):
        a = torch.randn((3, 37, cols), generator=gen, device=dev).to(torch.bfloat16)
        b = torch.randn((3, 37, cols), generator=gen, device=dev).to(torch.bfloat16)
        s = torch.rand((3, 37), generator=gen, device=dev) + 0.5
        d, a_s = ops.rowdot_scale(a, b, s)
        want = (a.float() * b.float()).sum(-1) * s
        assert torch.allclose(d, want, rtol=1e-5, atol=1e-5)
        assert torch.equal(a_s, (a.float() * s[..., None]).to(torch.bfloat16))
    p = torch.rand((5, 64, 96), generator=gen, device=dev).to(torch.bfloat16)
    s = torch.rand((5, 64), generator=gen, device=dev)
    assert torch.equal(ops.panel_normalize(p, s), p.float() * s[..., None])
    assert torch.equal(ops.panel_normalize(p, s, torch.bfloat16), (p.float() * s[..., None]).to(torch.bfloat16))


def test_factored_fallback_when_row_max_is_far_beyond_first_tile(rsa):
    """A row whose best key lies 2^369 (in probability) above its first key
    tile's best key: the single-pass kernel flags it (bit 1) and the API
    recomputes with the two-pass kernel, matching the oracle."""
    from paper_2105_13120_b200 import engine

    pkg, ra = rsa
    b, z, seq, a, n = 1, 2, 256, 64, 1
    q, k, v, g = _inputs(b, z, seq, a, seed=77)
    q[..., 0, :] = 4.0       # query row 0 of each head ...
    k[..., 200, :] = 4.0     # ... scores 1024 against key 200 (second key tile), |score| < ~200 elsewhere
    dev = torch.device("cuda", 0)
    tq, tk, tv = (torch.from_numpy(x[None]).to(dev, torch.bfloat16) for x in (q, k, v))
    res = engine.forward(tq, tk, tv, path="fused")
    torch.cuda.synchronize()
    assert int(res.flag.item()) == 2
    _, fwd, bwd = _run(pkg, ra, q, k, v, g, n, "fused")
    _check_all(pkg, fwd, bwd, _oracle(q, k, v, g, n))
    assert fwd.probs.rowscale is None  # recomputed by the normalised two-pass kernel


def test_factored_flag_clear_on_ordinary_inputs(rsa):
    from paper_2105_13120_b200 import engine

    dev = torch.device("cuda", 0)
    gen = torch.Generator(device=dev).manual_seed(11)
    tq, tk, tv = (3 * torch.randn((1, 2, 4, 512, 64), generator=gen, device=dev).to(torch.bfloat16) for _ in range(3))
    res = engine.forward(tq, tk, tv, path="fused")
    torch.cuda.synchronize()
    assert int(res.flag.item()) == 0 and res.rowscale is not None


def test_backward_does_not_materialise_saved_panels(rsa):
    """Passing fwd.probs back hands the factored panel to the kernels; the
    per-rank probabilities are only built when the caller looks at them."""
    pkg, ra = rsa
    b, z, seq, a, n = 1, 2, 256, 64, 2
    q, k, v, g = _inputs(b, z, seq, a, seed=5)
    _, fwd, _ = _run(pkg, ra, q, k, v, g, n, "fused")
    assert all(list.__getitem__(fwd.probs, d) is None for d in range(n))
    assert fwd.probs[1].dtype == torch.float32 and list.__getitem__(fwd.probs, 1) is not None


@pytest.mark.parametrize("as_torch", [False, True])
def test_backward_follows_given_values_and_panels(rsa, as_torch):
    """The backward uses the values and panels it is GIVEN (ringseq/ring_attention.py:150-209):
    D = rowsum(dP * P) with dP = dO V_given^T.  The forward's saved O is reused only for
    the forward's own values and unmodified panels; a different V, or a replaced panel
    (probs[d] = X), must change the gradients exactly as the oracle's do."""
    pkg, ra = rsa
    b, z, seq, a, n = 1, 2, 256, 64, 2
    q, k, v, g = _inputs(b, z, seq, a, seed=41)
    v2 = orc.bf16_round(orc.make_rng(42).standard_normal(v.shape))
    q2 = orc.bf16_round(orc.make_rng(43).standard_normal(q.shape))
    cfg = _cfg(pkg, b, z, seq, a, n)
    dev = torch.device("cuda", 0)
    conv = (lambda x: torch.from_numpy(x).to(dev, torch.bfloat16)) if as_torch else (lambda x: x)  # noqa: E731
    ch = lambda x: [conv(c) for c in orc.chunks_of(x, n)]  # noqa: E731
    qc, kc, vc, gc = ch(q), ch(k), ch(v), ch(g)
    fwd = ra.ring_attention_forward(qc, kc, vc, cfg)
    # (1) other values than the forward's
    bwd = ra.ring_attention_backward(qc, kc, ch(v2), fwd.probs, gc, cfg)
    _, probs, _ = orc.ring_forward(orc.chunks_of(q, n), orc.chunks_of(k, n), orc.chunks_of(v, n), exact=False)
    want = orc.ring_backward(orc.chunks_of(q, n), orc.chunks_of(k, n), orc.chunks_of(v2, n), probs,
                             orc.chunks_of(g, n), exact=False)
    for name, got, ref in zip(("dq", "dk", "dv"), (bwd.grad_q, bwd.grad_k, bwd.grad_v), want[:3]):
        _gate(name, _np(pkg.gather_sequence(got)), np.concatenate(ref, -2))
    # (2) a replaced panel: rank 0's probabilities of other queries
    other = ra.ring_attention_forward(ch(q2), kc, vc, cfg)
    probs_mixed = fwd.probs
    probs_mixed[0] = other.probs[0]
    bwd = ra.ring_attention_backward(qc, kc, vc, probs_mixed, gc, cfg)
    given = [orc.bf16_round(_np(other.probs[0])), orc.bf16_round(_np(fwd.probs[1]))]
    want = orc.ring_backward(orc.chunks_of(q, n), orc.chunks_of(k, n), orc.chunks_of(v, n), given,
                             orc.chunks_of(g, n), exact=False)
    for name, got, ref in zip(("dq", "dk", "dv"), (bwd.grad_q, bwd.grad_k, bwd.grad_v), want[:3]):
        _gate(name, _np(pkg.gather_sequence(got)), np.concatenate(ref, -2))


def test_deferred_checks_raise_at_the_backward(rsa, monkeypatch):
    """RSA_B200_CHECK=deferred: the forward returns without a host sync; the NumericError
    for a non-finite score surfaces at check_forward and at the backward that consumes the
    panels; ordinary inputs pass through unchanged."""
    pkg, ra = rsa
    monkeypatch.setenv("RSA_B200_CHECK", "deferred")
    b, z, seq, a, n = 1, 2, 256, 64, 2
    q, k, v, g = _inputs(b, z, seq, a, seed=21)
    cfg = _cfg(pkg, b, z, seq, a, n)
    ch = lambda x: orc.chunks_of(x, n)  # noqa: E731
    fwd = ra.ring_attention_forward(ch(q), ch(k), ch(v), cfg)
    ra.check_forward(fwd)
    bwd = ra.ring_attention_backward(ch(q), ch(k), ch(v), fwd.probs, ch(g), cfg)
    _check_all(pkg, fwd, bwd, _oracle(q, k, v, g, n))
    bad = q.copy()
    bad[0, 0, 3, 0] = np.nan
    for mode in ("panel", "stream"):
        fwd = ra.ring_attention_forward(ch(bad), ch(k), ch(v), cfg, mode=mode)  # no raise here
        with pytest.raises(pkg.NumericError):
            ra.check_forward(fwd)
        with pytest.raises(pkg.NumericError):
            ra.ring_attention_backward(ch(bad), ch(k), ch(v), fwd.probs, ch(g), cfg)


@pytest.mark.parametrize("key", [50, 300])
def test_negative_overflow_score_raises_numeric_error(rsa, key):
    """A score that overflows the fp32 range to -inf while every other score of its row
    stays finite -- the case a max-only check misses -- raises NumericError
    (ringseq/tensor_ops.py:80-81), whether it sits in the first key tile (key 50) or a
    later one (key 300, where the factored kernel checks max |s|).  (The float64
    reference would not overflow here: scores beyond the fp32 range are the one
    documented behavioural difference.)"""
    pkg, ra = rsa
    q, k, v, _ = _inputs(1, 1, 512, 64, seed=12)
    q[0, 0, 7, 0] = -3.0e38
    k[0, 0, :, 0] = 0.0
    k[0, 0, key, 0] = 3.0e38
    cfg = _cfg(pkg, 1, 1, 512, 64, 1)
    with pytest.raises(pkg.NumericError):
        ra.ring_attention_forward([q], [k], [v], cfg, path="fused")


def test_gelu_kernels_match_torch_fp32(rsa):
    """rsa_gelu / rsa_gelu_bwd against a plain PyTorch fp32 reference of the same op."""
    from paper_2105_13120_b200 import tensor_ops as ops

    dev = torch.device("cuda", 0)
    gen = torch.Generator(device=dev).manual_seed(3)
    for n in (4096, 1001):
        x = 3 * torch.randn(n, generator=gen, device=dev)
        dy = torch.randn(n, generator=gen, device=dev)
        want = torch.nn.functional.gelu(x)  # exact (erf) form
        assert torch.allclose(ops.gelu(x, out_dtype=torch.float32), want, rtol=1e-5, atol=1e-6)
        xr = x.detach().requires_grad_(True)
        torch.nn.functional.gelu(xr).backward(dy)
        got = ops.gelu_backward(x, dy, out_dtype=torch.float32)
        assert torch.allclose(got, xr.grad, rtol=1e-4, atol=1e-5)
        xb = x.to(torch.bfloat16)
        assert torch.allclose(ops.gelu(xb).float(), torch.nn.functional.gelu(xb.float()), rtol=1e-2, atol=1e-2)


@pytest.mark.parametrize("n", [1, 2, 4])
def test_mlp_forward_backward(rsa, golden, n):
    """sequence_parallel_mlp vs the unmodified reference's mlp_forward (golden) and
    sequence_parallel_mlp_backward vs the oracle's chain rule, on the same bf16 inputs."""
    pkg, ra = rsa
    for case, want in golden_cases(golden, "mlp_mid").items():
        b, seq, h, seed = (int(t) for t in case.split("_"))
        rng = orc.make_rng(seed)
        x = orc.bf16_round(rng.standard_normal((b, seq, h)))
        s = 1.0 / math.sqrt(h)
        up = orc.bf16_round(rng.standard_normal((h, 4 * h)) * s)
        down = orc.bf16_round(rng.standard_normal((4 * h, h)) * (s / 2.0))
        w = pkg.MlpWeights(up, down)
        y, ledger = ra.sequence_parallel_mlp(orc.chunks_of(x, n), w)
        got = _np(pkg.gather_sequence(y))
        assert np.linalg.norm(got - want["y"]) / np.linalg.norm(want["y"]) <= 2e-2
        assert all(t.total_elements() == 0 for t in ledger.devices)
        g = orc.bf16_round(orc.make_rng(seed + 1).standard_normal((b, seq, h)))
        gx, gw, led = ra.sequence_parallel_mlp_backward(orc.chunks_of(x, n), w, orc.chunks_of(g, n))
        ref = orc.mlp_backward(x, up, down, g, exact=False)
        for name, val, r in zip(("grad_x", "grad_up", "grad_down"),
                                (_np(pkg.gather_sequence(gx)), _np(gw.up), _np(gw.down)), ref):
            rel = np.linalg.norm(val - r) / np.linalg.norm(r)
            assert rel <= 2e-2, (name, rel)
        if n > 1:
            assert all(float(t.allreduce_elements) == 2 * 2 * h * 4 * h * (n - 1) / n for t in led.devices)


@pytest.mark.parametrize("n", [1, 2])
def test_encoder_layer_matches_oracle(rsa, n):
    """EncoderLayer (x1 = x + MHA(x), y = x1 + MLP(x1)) forward and backward against the
    oracle composition of multi_head_forward/_backward and mlp_forward/_backward
    (ringseq/reference.py:122-185) on the same bf16 weights and inputs."""
    from paper_2105_13120_b200.encoder import EncoderLayer, EncoderWeights

    pkg, _ = rsa
    b, seq, z, a = 1, 256, 2, 64
    h = z * a
    cfg = pkg.AttentionConfig(batch_size=b, seq_len=seq, hidden_size=h, num_heads=z, head_size=a, num_devices=n)
    dev = torch.device("cuda", 0)
    gen = torch.Generator(device=dev).manual_seed(17)
    w = EncoderWeights.random(cfg, dev, gen)
    x = torch.randn((b, seq, h), generator=gen, device=dev).to(torch.bfloat16)
    gy = torch.randn((b, seq, h), generator=gen, device=dev).to(torch.bfloat16)
    stack = lambda t: torch.stack(torch.chunk(t, n, dim=-2))  # noqa: E731
    layer = EncoderLayer(cfg, w)
    y = layer.forward(stack(x))
    dx, gw = layer.backward(stack(gy))
    torch.cuda.synchronize()
    unstack = lambda t: _np(torch.cat(list(t), dim=-2))  # noqa: E731
    xn, gn = _np(x), _np(gy)
    wn = {k: _np(getattr(w, k)) for k in ("wq", "wk", "wv", "wo", "up", "down")}
    x1 = xn + orc.multi_head_forward(xn, wn["wq"], wn["wk"], wn["wv"], wn["wo"], num_heads=z, exact=False)
    want_y = x1 + orc.mlp_forward(x1, wn["up"], wn["down"], exact=False)
    gx1_m, g_up, g_down = orc.mlp_backward(x1, wn["up"], wn["down"], gn, exact=False)
    gx1 = gn + gx1_m
    gx_a, g_wq, g_wk, g_wv, g_wo = orc.multi_head_backward(xn, wn["wq"], wn["wk"], wn["wv"], wn["wo"], gx1,
                                                           num_heads=z, exact=False)
    want = {"y": want_y, "dx": gx1 + gx_a, "wq": g_wq, "wk": g_wk, "wv": g_wv, "wo": g_wo, "up": g_up,
            "down": g_down}
    got = {"y": unstack(y), "dx": unstack(dx), **{k: _np(getattr(gw, k)) for k in ("wq", "wk", "wv", "wo", "up",
                                                                                   "down")}}
    for key in want:
        rel = np.linalg.norm(got[key] - want[key]) / np.linalg.norm(want[key])
        assert rel <= 3e-2, (key, rel)


def test_tensor_parallel_comparator_matches_reference_goldens(rsa, golden):
    """tensor_parallel_attention / tensor_parallel_mlp (ringseq/tensor_parallel.py:79-122) against
    the unmodified reference on the same bf16 inputs, with the all-reduce ledger exact."""
    from paper_2105_13120_b200 import tensor_parallel as tp

    pkg, _ = rsa
    cases = golden_cases(golden, "tp_mid")
    assert len(cases) == 2
    for case, want in cases.items():
        b, seq, z, a, n, seed = (int(t) for t in case.split("_"))
        h = z * a
        cfg = pkg.AttentionConfig(batch_size=b, seq_len=seq, hidden_size=h, num_heads=z, head_size=a, num_devices=n)
        rng = orc.make_rng(seed)
        x = orc.bf16_round(rng.standard_normal((b, seq, h)))
        s = 1.0 / math.sqrt(h)
        ws = [orc.bf16_round(rng.standard_normal((h, h)) * s) for _ in range(4)]
        up = orc.bf16_round(rng.standard_normal((h, 4 * h)) * s)
        down = orc.bf16_round(rng.standard_normal((4 * h, h)) * (s / 2.0))
        y, led = tp.tensor_parallel_attention(x, pkg.AttentionWeights(*ws), cfg)
        rel = np.linalg.norm(_np(y) - want["y_attention"]) / np.linalg.norm(want["y_attention"])
        assert rel <= 2e-2, rel
        assert [float(t.allreduce_elements) for t in led.devices] == list(want["ledger_ar"])
        ym, _ = tp.tensor_parallel_mlp(x, pkg.MlpWeights(up, down), cfg)
        rel = np.linalg.norm(_np(ym) - want["y_mlp"]) / np.linalg.norm(want["y_mlp"])
        assert rel <= 2e-2, rel
    with pytest.raises(pkg.ConfigError):
        tp.tensor_parallel_attention(x, pkg.AttentionWeights(*ws),
                                     pkg.AttentionConfig(batch_size=b, seq_len=seq, hidden_size=h, num_heads=z,
                                                         head_size=a, num_devices=3))


def _random_geometries(count, seed):
    """Seeded (B, Z, L, A=64, N) draws: every chunk a multiple of 8 rows, some with more
    than 4 query tiles per head (the two-kernel backward), ragged last tiles included."""
    rng = np.random.default_rng(seed)
    shapes = []
    while len(shapes) < count:
        n = int(rng.integers(1, 5))
        c = 8 * int(rng.integers(1, 97))  # 8 .. 768 rows per rank
        b, z = int(rng.integers(1, 3)), int(rng.integers(1, 4))
        if b * z * (n * c) ** 2 > 3_000_000:  # keep the float64 oracle quick
            continue
        shapes.append((b, z, n * c, 64, n))
    return shapes


@pytest.mark.parametrize("shape", _random_geometries(10, seed=2105))
def test_fused_paths_match_oracle_random_geometry(rsa, shape):
    """Seeded geometry sweep of the fused forward (factored panel) and whichever backward
    the engine picks (single pass when <= 4 query tiles per head, else rsa_bwd_dkdv +
    rsa_bwd_dq), against the float64 oracle with the same gates as the fixed shapes."""
    from paper_2105_13120_b200 import engine

    b, z, seq, a, n = shape
    q, k, v, g = _inputs(b, z, seq, a, seed=7 + seq + 13 * n)
    dev = torch.device("cuda", 0)
    stack = lambda x: torch.from_numpy(np.stack(orc.chunks_of(x, n))).to(dev, torch.bfloat16)  # noqa: E731
    tq, tk, tv, tg = (stack(x) for x in (q, k, v, g))
    out, panel, rowscale, flag = engine.forward(tq, tk, tv, path="auto")
    assert int(flag.item()) == 0
    dq, dk, dv = engine.backward(tq, tk, tv, panel, tg, outputs=out, rowscale=rowscale, path="auto")
    torch.cuda.synchronize()
    wout, wprobs, wdq, wdk, wdv = _oracle(q, k, v, g, n)
    cat = lambda t: np.concatenate([_np(t[d]) for d in range(n)], axis=-2)  # noqa: E731
    _gate("out", cat(out), wout)
    for d in range(n):
        got = _np(engine.normalized_panel(panel[d], None if rowscale is None else rowscale[d]))
        assert np.max(np.abs(got - wprobs[d])) <= PROB_ABS
    _gate("dq", cat(dq), wdq)
    _gate("dk", cat(dk), wdk)
    _gate("dv", cat(dv), wdv)

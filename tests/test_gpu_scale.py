"""GPU parity at the geometries the benchmark and BASELINE.json's configs launch.

The fixed-shape tests in test_gpu_rsa.py launch fewer work units than the 148 SMs,
so each persistent CTA runs exactly one unit.  The benchmark does not: at
B64 Z12 L512 the forward walks 1536 units and the backward 768 heads on 148 CTAs,
which exercises K tiles kept resident across units, the next head's V / K / D
prefetch and the pipeline phase flips between heads.  These tests drive exactly
those launches and compare against the float64 oracle:

* the bench shape itself (B64 Z12 L512, one rank), sampled heads, through the
  same engine calls bench.py times and through the public API;
* config 1 exactly (B4 Z12 L512, N = 4 resident ranks), every head;
* small shapes with the grid capped at 1, 3 or 7 CTAs (rsa_set_max_ctas), so every
  CTA walks many units of several heads, for both backward forms;
* the config-4 chunk geometry (c = 2048, N = 8, the two-kernel backward), sampled
  query rows and keys of whole 16K-token heads.

Sampled heads use ``oracle.attention_head_sampled`` (ringseq/reference.py:66-103
restated blockwise): heads are independent and the ring returns exactly these sums.
Gates are those of test_gpu_rsa.py.
"""

from __future__ import annotations

import ctypes

import numpy as np
import pytest
import torch

from oracle import ringseq_np as orc

pytestmark = pytest.mark.gpu

REL_F = 1e-2
MAX_ABS = 2e-2
PROB_ABS = 4e-3


def _gate(name, got, want):
    got, want = np.asarray(got, np.float64), np.asarray(want, np.float64)
    assert got.shape == want.shape, (name, got.shape, want.shape)
    rel = np.linalg.norm(got - want) / max(np.linalg.norm(want), 1e-30)
    mx = np.max(np.abs(got - want))
    assert rel <= REL_F, f"{name}: relative Frobenius error {rel:.3e}"
    assert mx <= MAX_ABS * max(1.0, np.max(np.abs(want))), f"{name}: max |diff| {mx:.3e}"
    return rel


def _head(t, b, z):
    """Head (b, z) of a stacked [N][B][Z][c][...] tensor as one (N*c, ...) float64 array."""
    n = t.shape[0]
    return torch.cat([t[d, b, z] for d in range(n)], dim=0).double().cpu().numpy()


def _rand(shape, gen, dev):
    return torch.randn(shape, generator=gen, device=dev, dtype=torch.float32).to(torch.bfloat16)


def _check_heads(heads, tq, tk, tv, tg, out, probs, dq, dk, dv, rows=None, keys=None):
    """Gate sampled heads (b, z) of stacked device results against the oracle."""
    for b, z in heads:
        q, k, v, g = (_head(t, b, z) for t in (tq, tk, tv, tg))
        seq = q.shape[0]
        rr = np.arange(seq) if rows is None else rows
        kk = np.arange(seq) if keys is None else keys
        want = orc.attention_head_sampled(q, k, v, g, rr, kk)
        tag = f"head ({b},{z})"
        _gate(f"{tag} out", _head(out, b, z)[rr], want["out"])
        _gate(f"{tag} dq", _head(dq, b, z)[rr], want["dq"])
        _gate(f"{tag} dk", _head(dk, b, z)[kk], want["dk"])
        _gate(f"{tag} dv", _head(dv, b, z)[kk], want["dv"])
        if probs is not None:
            got = probs(b, z, rr)
            diff = np.max(np.abs(got - want["probs"]))
            assert diff <= PROB_ABS, f"{tag} probs max |diff| {diff:.3e}"


def _panel_rows(panel, rowscale):
    """probs(b, z, rows): the reference's probability rows (global row indices) of head
    (b, z), materialised from the (factored) stacked panel on the device."""
    from paper_2105_13120_b200 import engine

    c = panel.shape[3]

    def rows(b, z, rr):
        rr = np.asarray(rr)
        got = np.empty((len(rr), panel.shape[-1]))
        for d in np.unique(rr // c):
            sel = np.nonzero(rr // c == d)[0]
            idx = torch.as_tensor(rr[sel] % c, device=panel.device)
            p = panel[int(d), b, z].index_select(0, idx)
            s = None if rowscale is None else rowscale[int(d), b, z].index_select(0, idx)
            got[sel] = engine.normalized_panel(p, s).double().cpu().numpy()
        return got

    return rows


def _sample_heads(bsz, heads, count, seed, must=()):
    rng = np.random.default_rng(seed)
    items = set(must)
    while len(items) < count:
        items.add(int(rng.integers(0, bsz * heads)))
    return [(i // heads, i % heads) for i in sorted(items) if i < bsz * heads]


def test_bench_shape_sampled_heads():
    """B64 Z12 L512 on one rank -- bench.py's layer, its exact engine calls and buffers --
    with 20 sampled heads checked, including the first and last of the 768 backward
    items and heads of the final partial wave (items 740..767 run as the 6th head of
    their CTA)."""
    from paper_2105_13120_b200 import engine

    dev = torch.device("cuda", 0)
    gen = torch.Generator(device=dev).manual_seed(1234)
    B, Z, L, A = 64, 12, 512, 64
    tq, tk, tv, tg = (_rand((1, B, Z, L, A), gen, dev) for _ in range(4))
    out = torch.empty_like(tq)
    panel = torch.empty((1, B, Z, L, L), dtype=torch.bfloat16, device=dev)
    rowscale = torch.empty((1, B, Z, L), dtype=torch.float32, device=dev)
    flag = torch.zeros(1, dtype=torch.int32, device=dev)
    grads = tuple(torch.empty_like(tq) for _ in range(3))
    dvec = torch.empty((1, B, Z, L), dtype=torch.float32, device=dev)
    gsc = torch.empty_like(tq)
    engine.forward(tq, tk, tv, path="fused", flag=flag, out=out, panel=panel, rowscale=rowscale)
    dq, dk, dv = engine.backward(tq, tk, tv, panel, tg, outputs=out, path="fused", grads=grads, dvec=dvec,
                                 rowscale=rowscale, grad_scaled=gsc)
    torch.cuda.synchronize()
    assert int(flag.item()) == 0
    heads = _sample_heads(B, Z, 20, seed=5, must=(0, 147, 148, 295, 740, 755, 767))
    _check_heads(heads, tq, tk, tv, tg, out, _panel_rows(panel, rowscale), dq, dk, dv)

    # the public API on the same device chunks runs the same kernels: identical results
    from paper_2105_13120_b200 import AttentionConfig
    from paper_2105_13120_b200.ring_attention import ring_attention_backward, ring_attention_forward

    cfg = AttentionConfig(batch_size=B, seq_len=L, hidden_size=Z * A, num_heads=Z, head_size=A, num_devices=1)
    fwd = ring_attention_forward([tq[0]], [tk[0]], [tv[0]], cfg)
    bwd = ring_attention_backward([tq[0]], [tk[0]], [tv[0]], fwd.probs, [tg[0]], cfg)
    torch.cuda.synchronize()
    assert torch.equal(fwd.outputs[0], out[0])
    assert torch.equal(bwd.grad_q[0], dq[0]) and torch.equal(bwd.grad_k[0], dk[0]) and torch.equal(bwd.grad_v[0], dv[0])


def test_config1_every_head():
    """BASELINE.json configs[0] exactly: B4 Z12 L512 A64, 4 ring ranks resident on one GPU,
    through the public API, every head against the float64 ring oracle."""
    import paper_2105_13120_b200 as pkg
    from paper_2105_13120_b200.ring_attention import ring_attention_backward, ring_attention_forward

    b, z, seq, a, n = 4, 12, 512, 64, 4
    rng = orc.make_rng(0)
    q, k, v, g = (orc.bf16_round(rng.standard_normal((b, z, seq, a))) for _ in range(4))
    cfg = pkg.AttentionConfig(batch_size=b, seq_len=seq, hidden_size=z * a, num_heads=z, head_size=a, num_devices=n)
    ch = lambda x: orc.chunks_of(x, n)  # noqa: E731
    fwd = ring_attention_forward(ch(q), ch(k), ch(v), cfg)
    bwd = ring_attention_backward(ch(q), ch(k), ch(v), fwd.probs, ch(g), cfg)
    torch.cuda.synchronize()
    outs, probs, _ = orc.ring_forward(ch(q), ch(k), ch(v), exact=False)
    dq, dk, dv, _ = orc.ring_backward(ch(q), ch(k), ch(v), probs, ch(g), exact=False)
    npy = lambda t: t.double().cpu().numpy()  # noqa: E731
    cat = lambda xs: np.concatenate(xs, axis=-2)  # noqa: E731
    _gate("out", npy(pkg.gather_sequence(fwd.outputs)), cat(outs))
    for d in range(n):
        assert np.max(np.abs(npy(fwd.probs[d]) - probs[d])) <= PROB_ABS
    _gate("dq", npy(pkg.gather_sequence(bwd.grad_q)), cat(dq))
    _gate("dk", npy(pkg.gather_sequence(bwd.grad_k)), cat(dk))
    _gate("dv", npy(pkg.gather_sequence(bwd.grad_v)), cat(dv))
    assert all(t.ring_p2p_elements == 2 * (n - 1) * b * z * (seq // n) * a for t in fwd.ledger.devices)


@pytest.fixture
def grid_cap():
    from paper_2105_13120_b200._native import lib

    def set_cap(n):
        lib().rsa_set_max_ctas(n)

    yield set_cap
    lib().rsa_set_max_ctas(0)


CAPPED = [  # (B, Z, L, N, cap): every CTA walks several units of several heads
    (2, 3, 512, 1, 1),
    (2, 3, 512, 1, 4),
    (3, 2, 512, 4, 5),   # c = 128: 4 ranks x 1 tile per head
    (2, 3, 384, 2, 7),   # c = 192: ragged second tile
    (1, 5, 1280, 1, 3),  # 10 query tiles per head: two-kernel backward, K streamed (T > 4)
    (2, 2, 1024, 4, 3),  # c = 256: 8 query tiles per head, two-kernel backward
]


@pytest.mark.parametrize("shape", CAPPED)
def test_multi_unit_persistent_paths_match_oracle(grid_cap, shape):
    """Grid capped below the unit count: resident-K release and reload between heads,
    the next head's V / K / D prefetch, head_it / dq_empty phase flips and the
    two-kernel backward's item loop all run many times per CTA."""
    from paper_2105_13120_b200 import engine

    b, z, seq, n, cap = shape
    a, c = 64, seq // shape[3]
    grid_cap(cap)
    rng = orc.make_rng(17 + seq + n + cap)
    q, k, v, g = (orc.bf16_round(rng.standard_normal((b, z, seq, a))) for _ in range(4))
    dev = torch.device("cuda", 0)
    stack = lambda x: torch.from_numpy(np.stack(orc.chunks_of(x, n))).to(dev, torch.bfloat16)  # noqa: E731
    tq, tk, tv, tg = (stack(x) for x in (q, k, v, g))
    heads = [(bi, zi) for bi in range(b) for zi in range(z)]
    single = [True, False] if engine.single_pass_supported(n, b, z, c, a) else [False]
    for factored in (True, False):
        out, panel, rowscale, flag = engine.forward(tq, tk, tv, path="fused", factored=factored)
        for sp in single:
            dq, dk, dv = engine.backward(tq, tk, tv, panel, tg, outputs=out, rowscale=rowscale, path="fused",
                                         single_pass=sp)
            torch.cuda.synchronize()
            assert int(flag.item()) == 0
            _check_heads(heads, tq, tk, tv, tg, out, _panel_rows(panel, rowscale), dq, dk, dv)


def test_config4_chunk_geometry_sampled():
    """c = 2048 per rank, N = 8 resident ranks (BERT-large config 4's chunk, L = 16K):
    16 query tiles per head, so the two-kernel backward (rsa_bwd_dkdv + rsa_bwd_dq).
    Two heads, 192 sampled query rows and 192 sampled keys each, spread over every rank."""
    from paper_2105_13120_b200 import engine

    b, z, n, c, a = 1, 2, 8, 2048, 64
    dev = torch.device("cuda", 0)
    gen = torch.Generator(device=dev).manual_seed(77)
    tq, tk, tv, tg = (_rand((n, b, z, c, a), gen, dev) for _ in range(4))
    assert not engine.single_pass_supported(n, b, z, c, a)
    out, panel, rowscale, flag = engine.forward(tq, tk, tv, path="fused")
    dq, dk, dv = engine.backward(tq, tk, tv, panel, tg, outputs=out, rowscale=rowscale, path="fused")
    torch.cuda.synchronize()
    assert int(flag.item()) == 0
    rng = np.random.default_rng(3)
    seq = n * c
    rows = np.unique(np.concatenate([[0, c - 1, c, seq - 1], rng.integers(0, seq, 188)]))
    keys = np.unique(np.concatenate([[0, 127, 128, seq - 1], rng.integers(0, seq, 188)]))
    _check_heads([(0, 0), (0, 1)], tq, tk, tv, tg, out, _panel_rows(panel, rowscale), dq, dk, dv, rows, keys)


def test_grid_cap_hook_roundtrip():
    from paper_2105_13120_b200._native import lib

    assert lib().rsa_set_max_ctas(5) == 0
    assert lib().rsa_set_max_ctas(0) == 5
    assert isinstance(ctypes.c_int(lib().rsa_num_sms()).value, int)

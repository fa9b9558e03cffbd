"""The one-pass panel backward at any length (rsa_bwd_panel_fused).

rsa_bwd_fused needs a head's query rows in at most 4 tiles; beyond that (and for small
batches, where one CTA per head leaves SMs idle) the panel backward used to be
rsa_bwd_dkdv + rsa_bwd_dq, which read the panel twice.  rsa_bwd_panel_fused reads it once:
one CTA per key tile walks every query tile, keeps dK / dV in TMEM and adds dQ partials into
an fp32 accumulator in L2.  Parity (ringseq/ring_attention.py:150-217): the float64 oracle
with the gates of test_gpu_rsa.py, and agreement with the fixed-order pair
(RSA_B200_DETERMINISTIC=1) to bf16 rounding -- dQ's sum over key tiles is taken in arrival
order, and dK / dV sum the query tiles from a per-item starting tile.
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

from oracle import ringseq_np as orc

pytestmark = pytest.mark.gpu

REL_F = 1e-2
MAX_ABS = 2e-2


def _gate(name, got, want):
    got, want = np.asarray(got, np.float64), np.asarray(want, np.float64)
    rel = np.linalg.norm(got - want) / max(np.linalg.norm(want), 1e-30)
    mx = np.max(np.abs(got - want))
    assert rel <= REL_F, f"{name}: relative Frobenius error {rel:.3e}"
    assert mx <= MAX_ABS * max(1.0, np.max(np.abs(want))), f"{name}: max |diff| {mx:.3e}"


def _close(name, got, ref, tol=4e-3):
    got, ref = got.double(), ref.double()
    rel = float(torch.linalg.norm(got - ref) / torch.linalg.norm(ref))
    assert rel <= tol, f"{name}: one-pass vs fixed-order relative difference {rel:.3e}"


def _run(engine, monkeypatch, tq, tk, tv, tg):
    out, panel, rowscale, flag = engine.forward(tq, tk, tv, path="fused")
    monkeypatch.setenv("RSA_B200_DETERMINISTIC", "0")
    one = engine.backward(tq, tk, tv, panel, tg, outputs=out, rowscale=rowscale, path="fused", single_pass=False)
    monkeypatch.setenv("RSA_B200_DETERMINISTIC", "1")
    pair = engine.backward(tq, tk, tv, panel, tg, outputs=out, rowscale=rowscale, path="fused", single_pass=False)
    torch.cuda.synchronize()
    assert int(flag.item()) == 0
    return out, one, pair


SHAPES = [  # (B, Z, L, N)
    (1, 2, 256, 2),
    (2, 3, 512, 4),     # c = 128
    (1, 2, 400, 2),     # c = 200: ragged key and query tiles
    (2, 1, 96, 4),      # c = 24: mostly padding
    (1, 2, 1280, 1),    # 10 query tiles per head (beyond rsa_bwd_fused's 4)
    (1, 2, 2048, 4),    # c = 512, four origins, 16 query tiles per head
]


@pytest.mark.parametrize("shape", SHAPES)
def test_panel_onepass_matches_oracle_and_pair(shape, monkeypatch):
    from paper_2105_13120_b200 import engine

    b, z, seq, n = shape
    a = 64
    rng = orc.make_rng(500 + seq + n)
    q, k, v, g = (orc.bf16_round(rng.standard_normal((b, z, seq, a))) for _ in range(4))
    dev = torch.device("cuda", 0)
    stack = lambda x: torch.tensor(np.stack(orc.chunks_of(x, n)), dtype=torch.bfloat16, device=dev)  # noqa: E731
    tq, tk, tv, tg = (stack(x) for x in (q, k, v, g))
    _, (dq, dk, dv), pair = _run(engine, monkeypatch, tq, tk, tv, tg)
    ch = lambda x: orc.chunks_of(x, n)  # noqa: E731
    _, probs, _ = orc.ring_forward(ch(q), ch(k), ch(v), exact=False)
    wq, wk, wv, _ = orc.ring_backward(ch(q), ch(k), ch(v), probs, ch(g), exact=False)
    for name, got, want in (("dq", dq, wq), ("dk", dk, wk), ("dv", dv, wv)):
        _gate(name, got.double().cpu().numpy(), np.stack(want))
    for name, got, ref in zip(("dq", "dk", "dv"), (dq, dk, dv), pair):
        _close(name, got, ref)


def test_panel_onepass_config1_every_head(monkeypatch):
    """BASELINE config 1 exactly: B4 Z12 L512 over 4 resident ranks (192 key-tile items on
    148 CTAs, so some CTAs walk two items), every head against the oracle."""
    from paper_2105_13120_b200 import engine

    b, z, n, c, a = 4, 12, 4, 128, 64
    dev = torch.device("cuda", 0)
    gen = torch.Generator(device=dev).manual_seed(41)
    tq, tk, tv, tg = (torch.randn((n, b, z, c, a), generator=gen, device=dev).to(torch.bfloat16) for _ in range(4))
    _, (dq, dk, dv), pair = _run(engine, monkeypatch, tq, tk, tv, tg)
    for name, got, ref in zip(("dq", "dk", "dv"), (dq, dk, dv), pair):
        _close(name, got, ref)
    head = lambda t, bi, zi: torch.cat([t[d, bi, zi] for d in range(n)], 0).double().cpu().numpy()  # noqa: E731
    rows = np.arange(n * c)
    for bi in range(b):
        for zi in range(z):
            want = orc.attention_head_sampled(head(tq, bi, zi), head(tk, bi, zi), head(tv, bi, zi), head(tg, bi, zi),
                                              rows, rows)
            _gate(f"({bi},{zi}) dq", head(dq, bi, zi), want["dq"])
            _gate(f"({bi},{zi}) dk", head(dk, bi, zi), want["dk"])
            _gate(f"({bi},{zi}) dv", head(dv, bi, zi), want["dv"])


def test_panel_onepass_grid_capped(monkeypatch):
    """Every CTA walks many key-tile items of several heads (grid capped at 3)."""
    from paper_2105_13120_b200 import engine
    from paper_2105_13120_b200._native import lib

    dev = torch.device("cuda", 0)
    gen = torch.Generator(device=dev).manual_seed(12)
    tq, tk, tv, tg = (torch.randn((2, 3, 2, 384, 64), generator=gen, device=dev).to(torch.bfloat16) for _ in range(4))
    lib().rsa_set_max_ctas(3)
    try:
        _, one, pair = _run(engine, monkeypatch, tq, tk, tv, tg)
    finally:
        lib().rsa_set_max_ctas(0)
    for name, got, ref in zip(("dq", "dk", "dv"), one, pair):
        _close(name, got, ref)


def test_panel_onepass_long_chunk_sampled(monkeypatch):
    """c = 2048 per rank over 8 resident ranks (config 4's chunk, L = 16K): 128 query tiles
    walked per key tile; sampled rows and keys against the blockwise oracle."""
    from paper_2105_13120_b200 import engine

    n, b, z, c, a = 8, 1, 2, 2048, 64
    dev = torch.device("cuda", 0)
    gen = torch.Generator(device=dev).manual_seed(79)
    tq, tk, tv, tg = (torch.randn((n, b, z, c, a), generator=gen, device=dev).to(torch.bfloat16) for _ in range(4))
    _, (dq, dk, dv), pair = _run(engine, monkeypatch, tq, tk, tv, tg)
    for name, got, ref in zip(("dq", "dk", "dv"), (dq, dk, dv), pair):
        _close(name, got, ref)
    seq = n * c
    rng = np.random.default_rng(6)
    rows = np.unique(np.concatenate([[0, c - 1, c, seq - 1], rng.integers(0, seq, 124)]))
    keys = np.unique(np.concatenate([[0, 127, 128, seq - 1], rng.integers(0, seq, 124)]))
    head = lambda t, zi: torch.cat([t[d, 0, zi] for d in range(n)], 0).double().cpu().numpy()  # noqa: E731
    for zi in range(z):
        want = orc.attention_head_sampled(head(tq, zi), head(tk, zi), head(tv, zi), head(tg, zi), rows, keys)
        _gate("dq", head(dq, zi)[rows], want["dq"])
        _gate("dk", head(dk, zi)[keys], want["dk"])
        _gate("dv", head(dv, zi)[keys], want["dv"])

"""rsa_linformer_project (csrc/linformer.cu): the Linformer's sequence-sharded K/V projection
K' = sum_d E_d K_d, V' = sum_d F_d V_d (ringseq/sparse_attention.py:111-123) for every head
at once, against a float64 restatement of the same sums and against the generic path
(rsa_gemm per (rank, head) + rsa_sum_ranks) it replaces."""

from __future__ import annotations

import ctypes

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("shape", [(8, 1, 4, 128, 128), (8, 4, 12, 1024, 256), (3, 2, 2, 192, 384),
                                   (1, 2, 6, 512, 128)])
def test_linformer_projection_matches_float64(shape):
    from paper_2105_13120_b200 import engine
    from paper_2105_13120_b200._native import check, lib

    n, b, z, c, kdim = shape
    a, L = 64, shape[0] * shape[3]
    dev = torch.device("cuda", 0)
    gen = torch.Generator(device=dev).manual_seed(c + kdim)
    k, v = (torch.randn((n, b, z, c, a), generator=gen, device=dev).to(torch.bfloat16) for _ in range(2))
    e, f = ((torch.randn((kdim, L), generator=gen, device=dev) / L ** 0.5).to(torch.bfloat16) for _ in range(2))
    acc = torch.empty((2, b, z, kdim, a), dtype=torch.float32, device=dev)
    low = torch.empty((2, b, z, kdim, a), dtype=torch.bfloat16, device=dev)
    g = engine._geom(n, b, z, c, a, L, 0, n)
    check(lib().rsa_linformer_project(ctypes.byref(g), kdim, e.data_ptr(), f.data_ptr(), e.stride(0), engine._view(k),
                                      engine._view(v), acc[0].data_ptr(), acc[1].data_ptr(), low[0].data_ptr(),
                                      low[1].data_ptr(), torch.cuda.current_stream().cuda_stream),
          "rsa_linformer_project")
    torch.cuda.synchronize()
    for j, (p, x) in enumerate(((e, k), (f, v))):
        pd = p.double().cpu().numpy()
        xd = x.double().cpu().numpy()
        want = sum(np.einsum("kc,bzca->bzka", pd[:, d * c:(d + 1) * c], xd[d]) for d in range(n))
        got = acc[j].double().cpu().numpy()
        rel = np.linalg.norm(got - want) / np.linalg.norm(want)
        assert rel <= 1e-5, (j, rel)  # fp32 accumulation of exact bf16 products
        assert torch.equal(low[j], acc[j].to(torch.bfloat16))


def test_linformer_projection_rejects_untileable():
    from paper_2105_13120_b200 import engine
    from paper_2105_13120_b200._native import lib

    n, b, z, c, kdim, a = 2, 1, 3, 128, 128, 64  # B*Z = 3: not a multiple of four heads
    dev = torch.device("cuda", 0)
    k = torch.zeros((n, b, z, c, a), dtype=torch.bfloat16, device=dev)
    e = torch.zeros((kdim, n * c), dtype=torch.bfloat16, device=dev)
    acc = torch.empty((b, z, kdim, a), dtype=torch.float32, device=dev)
    g = engine._geom(n, b, z, c, a, n * c, 0, n)
    rc = lib().rsa_linformer_project(ctypes.byref(g), kdim, e.data_ptr(), e.data_ptr(), e.stride(0), engine._view(k),
                                     engine._view(k), acc.data_ptr(), acc.data_ptr(), None, None,
                                     torch.cuda.current_stream().cuda_stream)
    assert rc != 0


@pytest.mark.parametrize("shape", [(8, 1, 4, 256, 128), (2, 4, 12, 1024, 256), (3, 1, 3, 512, 384)])
def test_linformer_projection_gradients_match_float64(shape):
    """rsa_linformer_proj_grad: dE[:, d-block] = sum_h dK'_h K_{d,h}^T for every rank (and dF)."""
    from paper_2105_13120_b200 import engine
    from paper_2105_13120_b200._native import check, lib

    n, b, z, c, kdim = shape
    a, L = 64, shape[0] * shape[3]
    dev = torch.device("cuda", 0)
    gen = torch.Generator(device=dev).manual_seed(7 * c + kdim)
    k, v = (torch.randn((n, b, z, c, a), generator=gen, device=dev).to(torch.bfloat16) for _ in range(2))
    dkl, dvl = (torch.randn((b, z, kdim, a), generator=gen, device=dev).to(torch.bfloat16) for _ in range(2))
    ge, gf = (torch.full((kdim, L), float("nan"), dtype=torch.float32, device=dev) for _ in range(2))
    g = engine._geom(n, b, z, c, a, L, 0, n)
    check(lib().rsa_linformer_proj_grad(ctypes.byref(g), kdim, dkl.data_ptr(), dvl.data_ptr(), engine._view(k),
                                        engine._view(v), ge.data_ptr(), gf.data_ptr(), ge.stride(0),
                                        torch.cuda.current_stream().cuda_stream), "rsa_linformer_proj_grad")
    torch.cuda.synchronize()
    for got, low, x in ((ge, dkl, k), (gf, dvl, v)):
        ld, xd = low.double().cpu().numpy(), x.double().cpu().numpy()
        want = np.concatenate([np.einsum("bzka,bzca->kc", ld, xd[d]) for d in range(n)], axis=1)
        g64 = got.double().cpu().numpy()
        assert np.isfinite(g64).all()
        rel = np.linalg.norm(g64 - want) / np.linalg.norm(want)
        assert rel <= 1e-5, rel


def test_sparse_api_sequence_views_match_separate_chunks():
    """Chunks that are consecutive slices of one device tensor run zero-copy as one resident
    rank of L rows (sparse_attention._sequence_view); the results equal those of the same
    values passed as separate per-rank tensors (stacked first) to fp32 summation-order noise."""
    import math

    from paper_2105_13120_b200 import AttentionConfig, SparseAttentionConfig
    from paper_2105_13120_b200.sparse_attention import (_sequence_view, sparse_ring_attention_backward,
                                                        sparse_ring_attention_forward)
    from paper_2105_13120_b200.weights import SparseWeights

    n, b, z, L, a, kdim = 4, 1, 4, 2048, 64, 128
    c = L // n
    dev = torch.device("cuda", 0)
    gen = torch.Generator(device=dev).manual_seed(3)
    q, k, v, g = (torch.randn((b, z, L, a), generator=gen, device=dev).to(torch.bfloat16) for _ in range(4))
    w = SparseWeights(*((torch.randn((kdim, L), generator=gen, device=dev) / math.sqrt(L)).to(torch.bfloat16)
                        for _ in range(2)))
    cfg = SparseAttentionConfig(base=AttentionConfig(batch_size=b, seq_len=L, hidden_size=z * a, num_heads=z,
                                                     head_size=a, num_devices=n), proj_dim=kdim)
    views = [[t[:, :, d * c:(d + 1) * c] for d in range(n)] for t in (q, k, v, g)]
    seps = [[x.clone() for x in ch] for ch in views]
    assert _sequence_view(views[0]) is not None and _sequence_view(seps[0]) is None
    fv = sparse_ring_attention_forward(*views[:3], w, cfg)
    fs = sparse_ring_attention_forward(*seps[:3], w, cfg)
    bv = sparse_ring_attention_backward(*views[:3], w, cfg, views[3])
    bs = sparse_ring_attention_backward(*seps[:3], w, cfg, seps[3])
    torch.cuda.synchronize()

    def close(x, y, tol=2e-3):
        x, y = x.double(), y.double()
        assert float(torch.linalg.norm(x - y) / torch.linalg.norm(y)) <= tol

    for d in range(n):
        close(fv.outputs[d], fs.outputs[d])
        close(bv.grad_q[d], bs.grad_q[d])
        close(bv.grad_k[d], bs.grad_k[d])
        close(bv.grad_v[d], bs.grad_v[d])
    close(bv.grad_key_proj, bs.grad_key_proj)
    close(bv.grad_value_proj, bs.grad_value_proj)


@pytest.mark.parametrize("shape", [(8, 1, 4, 256, 128), (2, 4, 12, 1024, 256), (3, 1, 4, 384, 192)])
def test_linformer_projection_transposes_match_float64(shape):
    """rsa_linformer_proj_back: dK_d = E_d^T dK', dV_d = F_d^T dV' for every rank and head."""
    from paper_2105_13120_b200 import engine
    from paper_2105_13120_b200._native import check, lib

    n, b, z, c, kdim = shape
    a, L = 64, shape[0] * shape[3]
    dev = torch.device("cuda", 0)
    gen = torch.Generator(device=dev).manual_seed(5 * c + kdim)
    e, f = ((torch.randn((kdim, L), generator=gen, device=dev) / L ** 0.5).to(torch.bfloat16) for _ in range(2))
    dkl, dvl = (torch.randn((b, z, kdim, a), generator=gen, device=dev).to(torch.bfloat16) for _ in range(2))
    dk, dv = (torch.full((n, b, z, c, a), float("nan"), dtype=torch.bfloat16, device=dev) for _ in range(2))
    g = engine._geom(n, b, z, c, a, L, 0, n)
    check(lib().rsa_linformer_proj_back(ctypes.byref(g), kdim, e.data_ptr(), f.data_ptr(), e.stride(0),
                                        dkl.data_ptr(), dvl.data_ptr(), engine._view(dk), engine._view(dv),
                                        torch.cuda.current_stream().cuda_stream), "rsa_linformer_proj_back")
    torch.cuda.synchronize()
    for got, p, low in ((dk, e, dkl), (dv, f, dvl)):
        pd, ld = p.double().cpu().numpy(), low.double().cpu().numpy()
        want = np.stack([np.einsum("kc,bzka->bzca", pd[:, d * c:(d + 1) * c], ld) for d in range(n)])
        g64 = got.double().cpu().numpy()
        assert np.isfinite(g64).all()
        rel = np.linalg.norm(g64 - want) / np.linalg.norm(want)
        assert rel <= 5e-3, rel  # one bf16 rounding of an fp32 sum

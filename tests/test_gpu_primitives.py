"""GPU checks of the primitive kernels against a plain torch fp32 reference.

tcgen05 GEMM (every operand major, batching, broadcast, tails), the SIMT
GEMM, softmax_rows (values, NumericError) and the softmax Jacobian.  Inputs
are bf16; the references compute in fp32 on the same bf16 values, so the
only differences are accumulation order (tolerance 2e-5 relative).
"""

import itertools

import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ops():
    from paper_2105_13120_b200 import tensor_ops

    yield tensor_ops
    tensor_ops.set_gemm_backend("auto")


def _rand(*shape, seed=0):
    g = torch.Generator(device="cpu").manual_seed(seed)
    return torch.randn(*shape, generator=g).to("cuda", torch.bfloat16)


def _close(got, want, tol=2e-5):
    err = (got.float() - want.float()).abs().max().item()
    scale = max(want.float().abs().max().item(), 1.0)
    assert err <= tol * scale * max(1, want.shape[-1] ** 0.5), (err, scale)


@pytest.mark.parametrize("backend", ["tcgen05", "simt"])
@pytest.mark.parametrize("m,n,k", [(128, 128, 64), (200, 72, 40), (512, 512, 64), (256, 64, 512), (64, 256, 128), (1, 8, 64)])
def test_gemm_all_majors(ops, backend, m, n, k):
    ops.set_gemm_backend(backend)
    a = _rand(m, k, seed=1)
    b = _rand(k, n, seed=2)
    want = a.float() @ b.float()
    for ta, tb in itertools.product([False, True], repeat=2):
        aa = a.t().contiguous().t() if ta else a  # same values, M-contiguous storage
        bb = b.t().contiguous().t() if tb else b
        got = ops.matmul(aa, bb)
        _close(got, want)


@pytest.mark.parametrize("backend", ["tcgen05", "simt"])
def test_gemm_batched_broadcast_and_bf16_out(ops, backend):
    ops.set_gemm_backend(backend)
    a = _rand(3, 1, 130, 64, seed=3)
    b = _rand(1, 4, 64, 96, seed=4)
    want = a.float() @ b.float()
    _close(ops.matmul(a, b), want)
    got16 = ops.matmul(a, b, out_dtype=torch.bfloat16)
    assert got16.dtype == torch.bfloat16
    assert (got16.float() - want).abs().max().item() <= 2e-2 * want.abs().max().item()
    # shared LHS (stride-0 batch): the Linformer projection shape
    e = _rand(64, 256, seed=5)
    kk = _rand(2, 3, 256, 64, seed=6)
    _close(ops.matmul(e, kk), e.float() @ kk.float())


def test_gemm_accumulate_and_alpha(ops):
    ops.set_gemm_backend("auto")
    a = _rand(2, 128, 64, seed=7)
    b = _rand(2, 64, 128, seed=8)
    out = torch.ones(2, 128, 128, device="cuda")
    ops.matmul(a, b, alpha=0.5, out=out, accumulate=True)
    _close(out, 0.5 * (a.float() @ b.float()) + 1.0)


def test_gemm_strided_panel_block(ops):
    # write a 128x128 score block into column block 1 of a (128 x 512) panel
    ops.set_gemm_backend("tcgen05")
    q = _rand(2, 128, 64, seed=9)
    k = _rand(2, 128, 64, seed=10)
    panel = torch.zeros(2, 128, 512, device="cuda")
    ops.matmul(q, k.transpose(-1, -2), out=panel[..., 128:256])
    _close(panel[..., 128:256], q.float() @ k.float().transpose(-1, -2))
    assert panel[..., :128].abs().max().item() == 0 and panel[..., 256:].abs().max().item() == 0


@pytest.mark.parametrize("cols", [512, 100, 4096, 3])
def test_softmax_rows(ops, cols):
    x = torch.randn(37, cols, device="cuda") * 4
    got = ops.softmax_rows(x, scale=0.125)
    want = torch.softmax(x * 0.125, dim=-1)
    assert (got - want).abs().max().item() <= 1e-6
    got16 = ops.softmax_rows(x, scale=0.125, out_dtype=torch.bfloat16)
    assert (got16.float() - want).abs().max().item() <= 4e-3


def test_softmax_known_answers_and_nonfinite(ops):
    import math

    from paper_2105_13120_b200.errors import NumericError

    got = ops.softmax_rows(torch.tensor([[0.0, math.log(3.0)]], device="cuda"))
    assert (got.cpu() - torch.tensor([[0.25, 0.75]])).abs().max().item() <= 1e-6
    got = ops.softmax_rows(torch.tensor([[1000.0, 1000.0]], device="cuda"))
    assert got.cpu().tolist() == [[0.5, 0.5]]
    with pytest.raises(NumericError):
        ops.softmax_rows(torch.tensor([[0.0, float("inf")]], device="cuda"))
    with pytest.raises(NumericError):
        ops.softmax_rows(torch.tensor([[float("nan"), 1.0]], device="cuda"))


def test_softmax_backward(ops):
    p = torch.softmax(torch.randn(64, 512, device="cuda"), -1)
    dp = torch.randn(64, 512, device="cuda")
    got = ops.softmax_backward(p, dp, 0.125, out_dtype=torch.float32)
    want = p * (dp - (dp * p).sum(-1, keepdim=True)) * 0.125
    assert (got - want).abs().max().item() <= 1e-6

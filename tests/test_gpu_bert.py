"""The BERT harness kernels around the encoder (bert.py) against plain PyTorch fp32
references of the same ops, and one masked-LM step end to end."""

from __future__ import annotations

import pytest
import torch

pytestmark = pytest.mark.gpu


def test_embed_and_backward_match_torch():
    from paper_2105_13120_b200 import bert

    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev).manual_seed(3)
    n, b, c, h, vocab = 2, 3, 40, 64, 500
    tok = torch.randn((vocab, h), generator=g, device=dev).to(torch.bfloat16)
    pos = torch.randn((n * c, h), generator=g, device=dev).to(torch.bfloat16)
    ids = torch.randint(0, vocab, (n, b, c), generator=g, device=dev, dtype=torch.int32)
    x = bert.embed(ids, tok, pos)
    positions = (torch.arange(n, device=dev)[:, None, None] * c + torch.arange(c, device=dev)[None, None, :]).expand(n, b, c)
    want = tok.float()[ids.long()] + pos.float()[positions]
    assert torch.allclose(x.float(), want, atol=2e-2, rtol=1e-2)
    dx = torch.randn((n, b, c, h), generator=g, device=dev).to(torch.bfloat16)
    dtok = torch.zeros((vocab, h), device=dev)
    dpos = torch.empty((n * c, h), device=dev)
    bert.embed_backward(ids, dx, dtok, dpos)
    wt = torch.zeros_like(dtok).index_add_(0, ids.reshape(-1).long(), dx.reshape(-1, h).float())
    wp = torch.zeros_like(dpos).index_add_(0, positions.reshape(-1), dx.reshape(-1, h).float())
    assert torch.allclose(dtok, wt, atol=1e-4) and torch.allclose(dpos, wp, atol=1e-4)


def test_softmax_xent_matches_torch():
    from paper_2105_13120_b200 import bert

    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev).manual_seed(4)
    m, v = 37, 30522
    logits = torch.randn((m, v), generator=g, device=dev) * 4
    targets = torch.randint(0, v, (m,), generator=g, device=dev, dtype=torch.int32)
    loss, dl = bert.softmax_xent(logits, targets, 1.0 / m)
    want = torch.nn.functional.cross_entropy(logits, targets.long(), reduction="none")
    assert torch.allclose(loss, want, atol=1e-4, rtol=1e-5)
    wd = (torch.softmax(logits, -1) - torch.nn.functional.one_hot(targets.long(), v).float()) / m
    assert torch.allclose(dl.float(), wd, atol=1e-5, rtol=1e-2)


def test_mlm_step_runs_and_head_matches_torch():
    """A small BERT MLM step (2 layers, 2 ring ranks): finite loss equal to torch's
    cross-entropy of the same final hidden states, and gradients for every parameter."""
    from paper_2105_13120_b200 import AttentionConfig
    from paper_2105_13120_b200.bert import BertMLM

    dev = torch.device("cuda", 0)
    g = torch.Generator(device=dev).manual_seed(5)
    cfg = AttentionConfig(batch_size=2, seq_len=256, hidden_size=128, num_heads=2, head_size=64, num_devices=2)
    model = BertMLM(cfg, 2, vocab=1000, device=dev, generator=g)
    ids = torch.randint(0, 1000, (2, 2, 128), generator=g, device=dev, dtype=torch.int32)
    mask_rows = torch.randperm(ids.numel(), generator=g, device=dev)[:77].sort().values
    targets = torch.randint(0, 1000, (77,), generator=g, device=dev, dtype=torch.int32)
    loss, grads = model.step(ids, mask_rows, targets)
    torch.cuda.synchronize()
    # the head on the model's own final hidden states, in torch fp32
    from paper_2105_13120_b200.bert import embed

    x = embed(ids, model.tok, model.pos)
    for ly in model.layers:
        x = ly.forward(x)
    xm = x.view(-1, 128).index_select(0, mask_rows).float()
    want = torch.nn.functional.cross_entropy(xm @ model.tok[:1000].float().t(), targets.long())
    assert torch.isfinite(loss) and abs(float(loss) - float(want)) <= 2e-3 * max(1.0, float(want))
    assert grads["tok"].shape == (1000, 128) and torch.isfinite(grads["tok"]).all()
    assert torch.isfinite(grads["pos"]).all() and len(grads["layers"]) == 2

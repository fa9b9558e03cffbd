"""BERT masked-LM training step over the RSA encoder.

The paper's throughput figures are whole-model BERT training steps (PAPER.md:308, 353:
tokens/s over the last 100 of 150 iterations); the reference itself simulates attention
only.  ``BertMLM`` puts the pieces around the sequence-parallel encoder stack
(``encoder.EncoderLayer``: ring self-attention + GELU MLP with residuals):

* token + position embeddings (``rsa_embed``), positions following the contiguous chunk
  layout of ringseq/cluster.py:73-88 (rank d holds tokens d*c .. d*c + c - 1);
* the masked-LM head on the masked positions only: logits = x_m @ tok^T (tied weights,
  ``rsa_gemm``), loss = mean cross-entropy and its gradient in one pass
  (``rsa_softmax_xent``);
* the backward of all of it: head GEMMs, the encoder layers in reverse, the embedding
  gradient (``rsa_embed_bwd``).

Layer norm and dropout are not in the reference and are left out; the
residual-branch projections are scaled by 1/sqrt(2 * layers) instead
(``EncoderWeights.random``).  Gathering the masked rows and scattering their gradient
back are index_select / index_copy on the device (harness plumbing, not the RSA path).
"""

from __future__ import annotations

import torch

from . import tensor_ops as ops
from ._native import BF16, F32, check, lib
from .config import AttentionConfig
from .encoder import EncoderLayer, EncoderWeights

__all__ = ["BertMLM"]


def _stream(t: torch.Tensor) -> int:
    return torch.cuda.current_stream(t.device).cuda_stream


def embed(ids: torch.Tensor, tok: torch.Tensor, pos: torch.Tensor) -> torch.Tensor:
    """[N][B][c] int32 token ids -> [N][B][c][H] bf16 token + position embeddings."""
    n, b, c = ids.shape
    h = tok.shape[1]
    x = torch.empty((n, b, c, h), dtype=torch.bfloat16, device=ids.device)
    check(lib().rsa_embed(ids.data_ptr(), n, b, c, tok.data_ptr(), pos.data_ptr(), h, x.data_ptr(), _stream(ids)),
          "rsa_embed")
    return x


def embed_backward(ids: torch.Tensor, dx: torch.Tensor, dtok: torch.Tensor, dpos: torch.Tensor) -> None:
    """dtok[ids] += dx (fp32 atomics); dpos[positions] = sum over the batch of dx (fp32,
    written; a deterministic rsa_sum_ranks per rank -- atomics would contend B-way)."""
    n, b, c = ids.shape
    h = dx.shape[-1]
    dx = dx.contiguous()
    st = _stream(ids)
    check(lib().rsa_embed_bwd(ids.data_ptr(), n, b, c, dx.data_ptr(), h, dtok.data_ptr(), None, st), "rsa_embed_bwd")
    for d in range(n):  # rank d holds positions d*c .. d*c + c - 1 of every sequence
        check(lib().rsa_sum_ranks(dx[d].data_ptr(), BF16, b, c * h, c * h, dpos[d * c:(d + 1) * c].data_ptr(), F32,
                                  st), "rsa_sum_ranks")


def softmax_xent(logits: torch.Tensor, targets: torch.Tensor, grad_scale: float, vocab: int | None = None):
    """Per-row cross-entropy of fp32 logits [M][V] against int32 targets, and
    dlogits = (softmax - onehot) * grad_scale as bf16.  ``vocab`` < V: only the first
    ``vocab`` columns take part (padded columns get a zero gradient)."""
    m, width = logits.shape
    v = width if vocab is None else vocab
    loss = torch.empty(m, dtype=torch.float32, device=logits.device)
    dl = (torch.empty if v == width else torch.zeros)((m, width), dtype=torch.bfloat16, device=logits.device)
    check(lib().rsa_softmax_xent(logits.data_ptr(), logits.stride(0), targets.data_ptr(), m, v, loss.data_ptr(),
                                 dl.data_ptr(), width, float(grad_scale), _stream(logits)), "rsa_softmax_xent")
    return loss, dl


class BertMLM:
    """BERT-base / -large masked-LM model over N ring ranks resident on one GPU."""

    def __init__(self, cfg: AttentionConfig, n_layers: int, vocab: int = 30522, device=None, generator=None):
        self.cfg, self.vocab = cfg, vocab
        h = cfg.hidden_size
        s = h ** -0.5
        # the table is padded to a multiple of 64 rows so every head GEMM operand row is
        # 16-byte aligned (the tcgen05 / TMA path); padded rows are zero, and the softmax
        # runs over the real vocabulary only
        self.vocab_padded = (vocab + 63) // 64 * 64
        self.tok = torch.zeros((self.vocab_padded, h), dtype=torch.bfloat16, device=device)
        self.tok[:vocab] = (torch.randn((vocab, h), generator=generator, device=device) * s).to(torch.bfloat16)
        self.pos = (torch.randn((cfg.seq_len, h), generator=generator, device=device) * s).to(torch.bfloat16)
        rs = (2 * n_layers) ** -0.5
        self.layers = [EncoderLayer(cfg, EncoderWeights.random(cfg, device, generator, residual_scale=rs))
                       for _ in range(n_layers)]

    def step(self, ids: torch.Tensor, mask_rows: torch.Tensor, targets: torch.Tensor):
        """One training step's forward and backward.

        ids: [N][B][c] int32; mask_rows: int64 indices of the masked tokens into the
        flattened [N*B*c] rows; targets: int32 [M] original tokens there.  Returns the mean
        masked-LM loss (fp32 scalar tensor on the device) and the gradients
        (dict: tok, pos fp32; layers: list of EncoderWeights)."""
        cfg = self.cfg
        h = cfg.hidden_size
        x = embed(ids, self.tok, self.pos)
        for ly in self.layers:
            x = ly.forward(x, check=False)
        # every layer's status flag in ONE host read (the layers' own backward would sync each)
        status = torch.cat([ly.flag for ly in self.layers]).cpu()
        if int(status.max()):
            from .errors import NumericError

            raise NumericError(f"encoder layer status flags {status.tolist()} (1: non-finite score, 2: a row beyond "
                               "the single-pass headroom; rerun with check=True)")
        for ly in self.layers:
            ly.unchecked = False
        flat = x.view(-1, h)
        xm = flat.index_select(0, mask_rows)                         # [M][H] bf16
        logits = ops.matmul(xm, self.tok.transpose(0, 1))             # [M][V_pad] fp32
        m = mask_rows.numel()
        rows_loss, dlogits = softmax_xent(logits, targets, 1.0 / m, vocab=self.vocab)
        loss = rows_loss.mean()
        # head backward (tied weights): dx_m = dlogits tok, dtok = dlogits^T x_m
        dxm = ops.matmul(dlogits, self.tok, out_dtype=torch.bfloat16)
        dtok = ops.matmul(dlogits.transpose(0, 1), xm)               # [V][H] fp32
        dx = torch.zeros_like(flat)
        dx.index_copy_(0, mask_rows, dxm)
        g = dx.view_as(x)
        grads = []
        for ly in reversed(self.layers):
            g, gw = ly.backward(g)
            grads.append(gw)
        dpos = torch.empty((cfg.seq_len, h), dtype=torch.float32, device=x.device)
        embed_backward(ids, g, dtok, dpos)
        return loss, {"tok": dtok[:self.vocab], "pos": dpos, "layers": grads[::-1]}

    def flags(self) -> list:
        return [int(ly.flag.item()) for ly in self.layers]

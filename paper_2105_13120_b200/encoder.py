"""Sequence-parallel transformer encoder layer.

The reference composes its sequence-parallel attention layer and its local MLP
(ringseq/ring_attention.py:220-256, ringseq/reference.py:122-185) but ships no
training step; the paper's BERT experiments run whole encoder
layers.  ``EncoderLayer`` is that layer on the B200 path:

    x1 = x + MHA(x)            MHA = sequence_parallel_attention (ring self-attention)
    y  = x1 + MLP(x1)          MLP = gelu(x1 @ up) @ down

with a forward that saves what the backward needs (q/k/v, the factored probability
panel and its row scale, the attention output, x1 and the MLP pre-activation) and a
backward that consumes it -- unlike the reference-shaped ``*_backward`` functions,
which recompute the forward.  Layer norm and dropout are not part of the reference
 and are left out.  Every rank's chunk is resident on this GPU
([N][B][c][H] stacks); the attention stages run the fused RSA kernels, the
projections rsa_gemm, the activation rsa_gelu.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

from . import engine
from . import tensor_ops as ops
from .config import AttentionConfig
from .errors import NumericError, ShapeError

__all__ = ["EncoderWeights", "EncoderLayer"]


@dataclass
class EncoderWeights:
    """wq/wk/wv (H, Z*A), wo (Z*A, H), up (H, 4H), down (4H, H); bf16 on the device."""

    wq: torch.Tensor
    wk: torch.Tensor
    wv: torch.Tensor
    wo: torch.Tensor
    up: torch.Tensor
    down: torch.Tensor

    @staticmethod
    def random(cfg: AttentionConfig, device, generator=None, residual_scale: float = 1.0) -> "EncoderWeights":
        """Gaussian weights at the reference's scales (ringseq/reference.py:207-224).
        ``residual_scale`` multiplies the two projections that feed the residual stream
        (wo, down) -- e.g. 1/sqrt(2 * layers) keeps a deep stack without layer norm bounded."""
        h, za = cfg.hidden_size, cfg.num_heads * cfg.head_size
        s = h ** -0.5

        def w(shape, scale):
            return (torch.randn(shape, generator=generator, device=device) * scale).to(torch.bfloat16)

        r = residual_scale
        return EncoderWeights(w((h, za), s), w((h, za), s), w((h, za), s), w((za, h), s * r), w((h, 4 * h), s),
                              w((4 * h, h), s / 2 * r))


class EncoderLayer:
    """One encoder layer over N resident ring ranks; ``forward`` then ``backward``."""

    def __init__(self, cfg: AttentionConfig, weights: EncoderWeights):
        self.cfg, self.w = cfg, weights
        self.saved = None

    def _split(self, y):
        c = self.cfg
        return y.view(c.num_devices, c.batch_size, c.chunk_len, c.num_heads, c.head_size).permute(
            0, 1, 3, 2, 4).contiguous()

    @staticmethod
    def _merge(t):
        n, b, z, c, a = t.shape
        return t.permute(0, 1, 3, 2, 4).reshape(n, b, c, z * a)

    def forward(self, x: torch.Tensor, check: bool = True) -> torch.Tensor:
        """x: [N][B][c][H] bf16 -> y: [N][B][c][H] bf16.  ``check=False`` skips the
        host read of the non-finite flag (the caller reads ``self.flag`` later)."""
        c, w = self.cfg, self.w
        if x.shape != (c.num_devices, c.batch_size, c.chunk_len, c.hidden_size):
            raise ShapeError(f"x has shape {tuple(x.shape)}")
        q, k, v = (self._split(ops.matmul(x, m, out_dtype=torch.bfloat16)) for m in (w.wq, w.wk, w.wv))
        res = engine.forward(q, k, v, path="auto")
        if check:
            status = int(res.flag.item())
            if status == 2:  # factored kernel's headroom fallback (ring_attention._forward_checked)
                res.flag.zero_()
                res = engine.forward(q, k, v, path="auto", factored=False, flag=res.flag, out=res.out,
                                     panel=res.panel)
                status = int(res.flag.item())
            if status:
                raise NumericError("softmax_rows requires finite inputs")
        merged = self._merge(res.out)
        x1 = ops.matmul(merged, w.wo)  # fp32
        x1 += x
        x1b = x1.to(torch.bfloat16)
        hpre = ops.matmul(x1b, w.up, out_dtype=torch.bfloat16)
        act = ops.gelu(hpre)
        y = ops.matmul(act, w.down)
        y += x1
        self.flag = res.flag
        self.unchecked = not check
        self.saved = (x, q, k, v, res, merged, x1b, hpre, act)
        return y.to(torch.bfloat16)

    def backward(self, gy: torch.Tensor):
        """gy: dL/dy [N][B][c][H] -> (dL/dx bf16, EncoderWeights of fp32 gradients)."""
        c, w = self.cfg, self.w
        x, q, k, v, res, merged, x1b, hpre, act = self.saved
        if getattr(self, "unchecked", False):
            # an unchecked forward is checked here, at its first synchronising use: its
            # outputs already flowed on, so a flagged layer cannot be recomputed silently
            status = int(res.flag.item())
            if status & 1:
                raise NumericError("softmax_rows requires finite inputs")
            if status & 2:
                raise NumericError("a row exceeded the single-pass panel's headroom in an unchecked forward; "
                                   "rerun the layer with forward(check=True)")
        h, inner, za = c.hidden_size, w.up.shape[1], c.num_heads * c.head_size
        gy = gy.to(torch.bfloat16)
        # MLP
        g_down = ops.matmul(act.reshape(-1, inner).transpose(0, 1), gy.reshape(-1, h))
        dact = ops.matmul(gy, w.down.transpose(0, 1))
        dh = ops.gelu_backward(hpre, dact)
        g_up = ops.matmul(x1b.reshape(-1, h).transpose(0, 1), dh.reshape(-1, inner))
        dx1 = ops.matmul(dh, w.up.transpose(0, 1))
        dx1 += gy
        dx1b = dx1.to(torch.bfloat16)
        # attention output projection and the ring backward
        g_wo = ops.matmul(merged.reshape(-1, za).transpose(0, 1), dx1b.reshape(-1, h))
        d_out = self._split(ops.matmul(dx1b, w.wo.transpose(0, 1), out_dtype=torch.bfloat16))
        dq, dk, dv = engine.backward(q, k, v, res.panel, d_out, outputs=res.out, rowscale=res.rowscale, path="auto")
        x2 = x.reshape(-1, h)
        grads = []
        dx = dx1
        for t, m in ((dq, w.wq), (dk, w.wk), (dv, w.wv)):
            t2 = self._merge(t)
            grads.append(ops.matmul(x2.transpose(0, 1), t2.reshape(-1, za)))
            ops.matmul(t2, m.transpose(0, 1), out=dx, accumulate=True)
        self.saved = None
        return dx.to(torch.bfloat16), EncoderWeights(grads[0], grads[1], grads[2], g_wo, g_up, g_down)

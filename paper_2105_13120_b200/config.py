"""Layer geometry and partitioning, mirrored from ``ringseq/config.py:10-56``.

The two frozen dataclasses keep the reference's field names, order,
defaults and validation messages' meaning so callers construct them the
same way:

* ``AttentionConfig(batch_size, seq_len, hidden_size, num_heads, head_size,
  num_devices=1)`` -- B, L, H, Z, A, N with H == Z*A and L % N == 0
  (``ringseq/config.py:26-39``); ``chunk_len`` is c = L/N
  (``ringseq/config.py:41-44``).
* ``SparseAttentionConfig(base, proj_dim)`` -- adds the Linformer projected
  length K (``ringseq/config.py:47-56``).

Device-side constraints (tile alignment, head size limits) are *not*
checked here: the reference accepts any positive integers, and so does this
boundary.  Shapes the tensor-core path cannot tile are routed to the
generic CUDA path by the dispatcher, never rejected.
"""

from __future__ import annotations

from dataclasses import dataclass

from .errors import ConfigError

__all__ = ["AttentionConfig", "SparseAttentionConfig"]

_POSITIVE_FIELDS = ("batch_size", "seq_len", "hidden_size", "num_heads", "head_size", "num_devices")


def _require_positive_int(name: str, value) -> None:
    # bool is an int subclass; the reference's isinstance check lets it
    # through, and so do we, to stay behaviour-identical.
    if not isinstance(value, int) or value < 1:
        raise ConfigError(f"{name} must be a positive integer, got {value!r}")


@dataclass(frozen=True)
class AttentionConfig:
    """Shapes of one attention layer and its sequence partitioning."""

    batch_size: int
    seq_len: int
    hidden_size: int
    num_heads: int
    head_size: int
    num_devices: int = 1

    def __post_init__(self) -> None:
        for name in _POSITIVE_FIELDS:
            _require_positive_int(name, getattr(self, name))
        if self.num_heads * self.head_size != self.hidden_size:
            raise ConfigError(
                f"hidden_size={self.hidden_size} must equal "
                f"num_heads*head_size={self.num_heads * self.head_size}"
            )
        if self.seq_len % self.num_devices:
            raise ConfigError(
                f"seq_len={self.seq_len} not divisible by num_devices={self.num_devices}"
            )

    @property
    def chunk_len(self) -> int:
        """c = L/N: contiguous tokens owned by each ring rank."""
        return self.seq_len // self.num_devices

    # Convenience views used by the device path (not in the reference).
    @property
    def heads_total(self) -> int:
        """B*Z, the number of independent (batch, head) attention problems."""
        return self.batch_size * self.num_heads

    def chunk_shape(self) -> tuple:
        """(B, Z, c, A): one rank's per-head chunk (ringseq/ring_attention.py:120-121)."""
        return (self.batch_size, self.num_heads, self.chunk_len, self.head_size)

    def panel_shape(self) -> tuple:
        """(B, Z, c, L): one rank's probability panel (ringseq/ring_attention.py:166)."""
        return (self.batch_size, self.num_heads, self.chunk_len, self.seq_len)


@dataclass(frozen=True)
class SparseAttentionConfig:
    """AttentionConfig plus the Linformer projected sequence length K."""

    base: AttentionConfig
    proj_dim: int

    def __post_init__(self) -> None:
        if not isinstance(self.proj_dim, int) or self.proj_dim < 1:
            raise ConfigError(f"proj_dim must be a positive integer, got {self.proj_dim!r}")

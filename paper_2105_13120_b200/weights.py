"""Weight containers of the attention layers, mirrored from ringseq/reference.py:36-59.

The API accepts these or the reference's own dataclasses interchangeably
(anything with the same attribute names), so weights drawn with
``ringseq.random_attention_weights`` can be passed straight through.
"""

from __future__ import annotations

from dataclasses import dataclass

__all__ = ["AttentionWeights", "SparseWeights", "MlpWeights"]


@dataclass(frozen=True)
class AttentionWeights:
    """wq/wk/wv are (H, Z*A), wo is (Z*A, H) (ringseq/reference.py:36-43)."""

    wq: object
    wk: object
    wv: object
    wo: object


@dataclass(frozen=True)
class SparseWeights:
    """Linformer sequence projections E (key_proj) and F (value_proj), each (K, L)
    (ringseq/reference.py:54-59)."""

    key_proj: object
    value_proj: object


@dataclass(frozen=True)
class MlpWeights:
    """Feed-forward weights: up is (H, 4H), down is (4H, H) (ringseq/reference.py:46-51)."""

    up: object
    down: object

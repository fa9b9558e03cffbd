"""B200-native Ring Self-Attention (arXiv 2105.13120) behind the ``ringseq`` API.

Drop-in for the reference package's sequence-parallel attention path
(ringseq.ring_attention / ringseq.sparse_attention / ringseq.tensor_ops):
same function names, signatures, result types, errors and contiguous L/N
chunk layout.  Arithmetic runs in hand-written sm_100a kernels
(librsa_b200.so, see include/rsa_b200.h); there is no CPU fallback.
"""

from .config import AttentionConfig, SparseAttentionConfig
from .errors import (
    ConfigError,
    DeadlockError,
    NativeError,
    NativeUnavailable,
    NumericError,
    ProtocolError,
    ShapeError,
    StateError,
)
from .cluster import (
    EXECUTOR_ENV_VAR,
    EXECUTORS,
    CommLedger,
    DeviceTraffic,
    RingTopology,
    ShardedSequence,
    gather_sequence,
    resolve_executor,
    scatter_sequence,
)

__version__ = "0.1.0"


_LAZY = {
    # device-facing names -> defining module (imported on first use so the
    # config/ledger layer stays importable without touching CUDA)
    "matmul": "tensor_ops",
    "softmax_rows": "tensor_ops",
    "split_heads": "tensor_ops",
    "merge_heads": "tensor_ops",
    "RingAttentionForward": "ring_attention",
    "RingAttentionBackward": "ring_attention",
    "ring_attention_forward": "ring_attention",
    "ring_attention_backward": "ring_attention",
    "sequence_parallel_attention": "ring_attention",
    "sequence_parallel_attention_backward": "ring_attention",
    "sequence_parallel_mlp": "ring_attention",
    "sequence_parallel_mlp_backward": "ring_attention",
    "MlpWeights": "weights",
    "tensor_parallel_attention": "tensor_parallel",
    "tensor_parallel_mlp": "tensor_parallel",
    "split_attention_heads": "tensor_parallel",
    "split_mlp_weights": "tensor_parallel",
    "ColumnRowSplitWeights": "tensor_parallel",
    "SparseRingForward": "sparse_attention",
    "sparse_ring_attention_forward": "sparse_attention",
    "sparse_ring_attention_backward": "sparse_attention",
    "SparseRingBackward": "sparse_attention",
    "split_projection_columns": "sparse_attention",
    "full_length_dims": "sparse_attention",
    "AttentionWeights": "weights",
    "SparseWeights": "weights",
}


def __getattr__(name):
    mod = _LAZY.get(name)
    if mod is None:
        raise AttributeError(f"module {__name__!r} has no attribute {name!r}")
    import importlib

    return getattr(importlib.import_module(f".{mod}", __name__), name)

"""Ring topology, sequence sharding and the communication ledger.

This is the *contract* half of ``ringseq/cluster.py``: the ring direction
(data moves rank d -> d+1, ``ringseq/cluster.py:52-62``), the contiguous
chunk layout (``ringseq/cluster.py:73-101``), and the per-device element
ledger with its charging convention (``ringseq/cluster.py:104-155``): a ring
hop charges the full buffer to the sender, an all-reduce of E elements
charges 2E(N-1)/N to every participant, kept as an exact Fraction.

The reference's thread executor (``ringseq/cluster.py:162-411``) has no
counterpart here: on a B200 the ranks are either (a) logical ranks whose
chunks all live in one GPU's HBM, where a ring hop is a pointer rotation
that the fused kernels perform implicitly, or (b) real ranks under
``torch.distributed`` where hops are NCCL send/recv (see ``distributed.py``).
Both charge the ledger exactly as the reference does, so the ledger gates
of the reference's tests carry over unchanged.

``DeviceTraffic.wire_bytes`` is an addition: the bytes this implementation
actually put on the wire (bf16 ring chunks, fp32 reduce-scatter), which is
what the roofline's link term uses.  It is excluded from equality so two
ledgers compare exactly as in the reference.
"""

from __future__ import annotations

import json
import os
from dataclasses import dataclass, field
from fractions import Fraction

from .errors import ConfigError, ShapeError

__all__ = [
    "EXECUTOR_ENV_VAR",
    "EXECUTORS",
    "RingTopology",
    "ShardedSequence",
    "scatter_sequence",
    "gather_sequence",
    "DeviceTraffic",
    "CommLedger",
    "resolve_executor",
]

EXECUTOR_ENV_VAR = "RINGSEQ_EXECUTOR"
EXECUTORS = ("sequential", "concurrent")


@dataclass(frozen=True)
class RingTopology:
    """Ranks 0..n-1 on a ring; buffers travel from rank i to rank i+1."""

    n_devices: int

    def next_device(self, i: int) -> int:
        return (i + 1) % self.n_devices

    def prev_device(self, i: int) -> int:
        return (i - 1) % self.n_devices

    def origin_at_hop(self, device: int, hop: int) -> int:
        """Rank whose chunk sits on ``device`` after ``hop`` passes.

        Hop 0 is the device's own chunk; every pass moves chunks one rank
        forward, so hop h delivers origin (device - h) mod N
        (ringseq/ring_attention.py:67-79).
        """
        return (device - hop) % self.n_devices


@dataclass(frozen=True)
class ShardedSequence:
    """One rank's contiguous slice of a sequence-partitioned tensor."""

    device_index: int
    chunk: object


def _is_torch(x) -> bool:
    mod = type(x).__module__
    return mod.startswith("torch")


def scatter_sequence(x, n_devices: int, axis: int = -2) -> list:
    """Split ``x`` into ``n_devices`` equal contiguous chunks along ``axis``.

    Accepts numpy arrays (returned as float64, like the reference) or torch
    tensors (dtype and device preserved).  Mirrors
    ringseq/cluster.py:73-88.
    """
    if n_devices < 1:
        raise ConfigError(f"device count must be positive, got {n_devices}")
    if _is_torch(x):
        length = x.shape[axis]
        if length % n_devices:
            raise ConfigError(f"sequence length {length} not divisible by device count {n_devices}")
        pieces = x.chunk(n_devices, dim=axis)
        return [ShardedSequence(i, p.contiguous()) for i, p in enumerate(pieces)]
    import numpy as np

    arr = np.asarray(x, dtype=np.float64)
    length = arr.shape[axis]
    if length % n_devices:
        raise ConfigError(f"sequence length {length} not divisible by device count {n_devices}")
    return [ShardedSequence(i, np.ascontiguousarray(p)) for i, p in enumerate(np.split(arr, n_devices, axis=axis))]


def gather_sequence(shards, axis: int = -2):
    """Concatenate shards in rank order (inverse of ``scatter_sequence``).

    ringseq/cluster.py:91-101: ShardedSequence items are sorted by rank and
    must form a complete range; plain arrays/tensors are taken as given.
    """
    items = list(shards)
    if not items:
        raise ShapeError("gather_sequence needs at least one shard")
    if isinstance(items[0], ShardedSequence):
        ranks = sorted(s.device_index for s in items)
        if ranks != list(range(len(items))):
            raise ShapeError(f"shard indices {ranks} do not form a complete range")
        items = [s.chunk for s in sorted(items, key=lambda s: s.device_index)]
    if _is_torch(items[0]):
        import torch

        return torch.cat(items, dim=axis)
    import numpy as np

    return np.concatenate(items, axis=axis)


def _fraction_json(value: Fraction):
    return int(value) if value.denominator == 1 else f"{value.numerator}/{value.denominator}"


@dataclass
class DeviceTraffic:
    """Elements one rank sent, split by mechanism (ringseq/cluster.py:110-121)."""

    ring_p2p_elements: int = 0
    allreduce_elements: Fraction = field(default_factory=Fraction)
    # Bytes this implementation really moved for this rank (not compared).
    wire_bytes: int = field(default=0, compare=False)

    def total_elements(self) -> Fraction:
        return self.ring_p2p_elements + self.allreduce_elements

    def total_bytes(self) -> Fraction:
        """Reference convention: 8 bytes (fp64) per element."""
        return 8 * self.total_elements()


class CommLedger:
    """Per-rank transfer accounting for one protocol run (ringseq/cluster.py:124-155)."""

    def __init__(self, n_devices: int):
        self.devices = [DeviceTraffic() for _ in range(n_devices)]

    @property
    def n_devices(self) -> int:
        return len(self.devices)

    def record_ring_send(self, device: int, elements: int, wire_bytes: int = 0) -> None:
        self.devices[device].ring_p2p_elements += int(elements)
        self.devices[device].wire_bytes += int(wire_bytes)

    def record_allreduce(self, device: int, elements: int, wire_bytes: int = 0) -> None:
        n = len(self.devices)
        self.devices[device].allreduce_elements += Fraction(2 * int(elements) * (n - 1), n)
        self.devices[device].wire_bytes += int(wire_bytes)

    def total_elements(self) -> Fraction:
        return sum((d.total_elements() for d in self.devices), Fraction(0))

    def total_wire_bytes(self) -> int:
        return sum(d.wire_bytes for d in self.devices)

    def as_json_obj(self) -> list:
        return [
            {
                "device_id": i,
                "ring_p2p_elements": d.ring_p2p_elements,
                "allreduce_elements": _fraction_json(d.allreduce_elements),
                "total_bytes": _fraction_json(d.total_bytes()),
            }
            for i, d in enumerate(self.devices)
        ]

    def dumps(self) -> str:
        return json.dumps(self.as_json_obj(), indent=2, sort_keys=True)

    def merge(self, other: "CommLedger") -> "CommLedger":
        """Elementwise sum of two ledgers over the same ring (fwd + bwd totals)."""
        if other.n_devices != self.n_devices:
            raise ShapeError("cannot merge ledgers of different ring sizes")
        out = CommLedger(self.n_devices)
        for o, a, b in zip(out.devices, self.devices, other.devices):
            o.ring_p2p_elements = a.ring_p2p_elements + b.ring_p2p_elements
            o.allreduce_elements = a.allreduce_elements + b.allreduce_elements
            o.wire_bytes = a.wire_bytes + b.wire_bytes
        return out

    def __eq__(self, other) -> bool:
        return isinstance(other, CommLedger) and self.devices == other.devices

    def __repr__(self) -> str:
        return f"CommLedger({self.as_json_obj()!r})"


def resolve_executor(executor: str | None = None) -> str:
    """Argument, then $RINGSEQ_EXECUTOR, then "sequential" (ringseq/cluster.py:370-375).

    Both executors run the identical device schedule here -- the interleaving
    freedom the reference simulates does not exist on a GPU stream -- so the
    choice is validated and otherwise has no effect on results.
    """
    mode = executor or os.environ.get(EXECUTOR_ENV_VAR) or "sequential"
    if mode not in EXECUTORS:
        raise ConfigError(f"unknown executor {mode!r}, expected one of {EXECUTORS}")
    return mode

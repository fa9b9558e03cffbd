"""Exception taxonomy of the drop-in boundary.

Mirrors ``ringseq/errors.py:4-25`` name for name and base class for base
class, so ``except ringseq.ShapeError`` style handlers written against the
reference keep working when this package is swapped in.  Two extra types
cover failures that only exist on a real device: ``NativeError`` (the CUDA
extension reported a launch/runtime failure) and ``NativeUnavailable`` (the
extension could not be loaded, which is always fatal -- there is no CPU
fallback on the product path).
"""

from __future__ import annotations

__all__ = [
    "ShapeError",
    "ConfigError",
    "NumericError",
    "ProtocolError",
    "DeadlockError",
    "StateError",
    "NativeError",
    "NativeUnavailable",
]


# --- value-type errors (ringseq/errors.py:4-13) ---------------------------

class ShapeError(ValueError):
    """Operand shapes are inconsistent with the configuration."""


class ConfigError(ValueError):
    """A configuration field is out of range or breaks a divisibility rule."""


class NumericError(ValueError):
    """Non-finite values reached an operation that rejects them (softmax)."""


# --- runtime-type errors (ringseq/errors.py:16-25) -------------------------

class ProtocolError(RuntimeError):
    """Ranks disagreed about a collective (shape mismatch, bad participation)."""


class DeadlockError(ProtocolError):
    """The ring could not make progress (a peer never posted its half)."""


class StateError(RuntimeError):
    """Saved state a call depends on (e.g. the probability panels) is missing."""


# --- device-only errors (no reference counterpart) ------------------------

class NativeError(RuntimeError):
    """The sm_100a extension returned a non-zero status code."""


class NativeUnavailable(ImportError):
    """librsa_b200.so is missing or could not be loaded on this host."""

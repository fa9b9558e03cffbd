"""ctypes binding of librsa_b200.so (declared in include/rsa_b200.h).

The product path has exactly one implementation: the sm_100a kernels in this
library.  If the library is missing or fails to load, every call raises
``NativeUnavailable`` -- there is deliberately no NumPy/PyTorch fallback.

Status codes map onto the reference's exception taxonomy
(ringseq/errors.py:4-25): RSA_ERR_INVALID -> ShapeError, RSA_ERR_NUMERIC ->
NumericError, anything else -> NativeError.
"""

from __future__ import annotations

import ctypes
import os
from ctypes import c_float, c_int, c_int32, c_int64, c_void_p
from pathlib import Path

from .errors import NativeError, NativeUnavailable, NumericError, ShapeError

__all__ = ["lib", "check", "RsaView", "RsaGeom", "RsaFwdExt", "LIB_PATH", "ABI_VERSION", "F32", "BF16", "EXPORTS"]

LIB_PATH = Path(os.environ.get("RSA_B200_LIB", Path(__file__).resolve().parent / "librsa_b200.so"))
ABI_VERSION = 4
F32, BF16 = 0, 1

RSA_OK, RSA_ERR_INVALID, RSA_ERR_UNSUPPORTED, RSA_ERR_CUDA, RSA_ERR_NUMERIC = 0, 1, 2, 3, 4


class RsaView(ctypes.Structure):
    """struct rsa_view: [rank][b][z][row][col] strides in elements."""

    _fields_ = [
        ("ptr", c_void_p),
        ("s_rank", c_int64),
        ("s_b", c_int64),
        ("s_z", c_int64),
        ("s_row", c_int64),
    ]


class RsaGeom(ctypes.Structure):
    """struct rsa_geom."""

    _fields_ = [
        ("n_rank", c_int32),
        ("batch", c_int32),
        ("heads", c_int32),
        ("chunk", c_int32),
        ("head_dim", c_int32),
        ("seq_len", c_int32),
        ("org_lo", c_int32),
        ("n_org", c_int32),
        ("scale", c_float),
        ("key_chunk", c_int32),
    ]


class RsaFwdExt(ctypes.Structure):
    """struct rsa_fwd_ext (options of rsa_fwd_factored_ex)."""

    _fields_ = [
        ("panel", RsaView),
        ("rowmax", c_void_p),
        ("rowmax_in", c_void_p),
        ("rowmax_in_stride", c_int32),
        ("rowmax_exact", c_int32),
        ("o_acc", RsaView),
        ("l_acc", c_void_p),
        ("acc_in", c_int32),
        ("final_hop", c_int32),
    ]


_P = ctypes.POINTER
_GEOM = _P(RsaGeom)
_V = RsaView

# name -> (restype, argtypes); every symbol include/rsa_b200.h declares.
EXPORTS = {
    "rsa_abi_version": (c_int, []),
    "rsa_last_error": (ctypes.c_char_p, []),
    "rsa_num_sms": (c_int, []),
    "rsa_set_max_ctas": (c_int, [c_int]),
    "rsa_gemm": (
        c_int,
        [c_int, c_int, c_int,
         c_void_p, c_int, c_int64, c_int, c_int64, c_int64,
         c_void_p, c_int, c_int64, c_int, c_int64, c_int64,
         c_void_p, c_int, c_int64, c_int64, c_int64,
         c_int, c_int, c_float, c_int, c_void_p],
    ),
    "rsa_gemm_set_backend": (c_int, [c_int]),
    "rsa_softmax_rows": (
        c_int,
        [c_void_p, c_int, c_int64, c_int64, c_int64, c_float, c_void_p, c_int, c_int64, c_void_p, c_void_p],
    ),
    "rsa_softmax_bwd": (
        c_int,
        [c_void_p, c_int, c_int64, c_void_p, c_int64, c_int64, c_int64, c_float, c_void_p, c_int, c_int64, c_void_p],
    ),
    "rsa_rowdot": (c_int, [c_void_p, c_int64, c_void_p, c_int64, c_int64, c_int64, c_void_p, c_void_p]),
    "rsa_rowdot_scale": (
        c_int,
        [c_void_p, c_int64, c_void_p, c_int64, c_void_p, c_int64, c_int64, c_void_p, c_void_p, c_int64, c_void_p],
    ),
    "rsa_gelu": (c_int, [c_void_p, c_int, c_int64, c_void_p, c_int, c_void_p]),
    "rsa_sum_ranks": (c_int, [c_void_p, c_int, c_int64, c_int64, c_int64, c_void_p, c_int, c_void_p]),
    "rsa_gelu_bwd": (c_int, [c_void_p, c_int, c_void_p, c_int, c_int64, c_void_p, c_int, c_void_p]),
    "rsa_panel_normalize": (c_int, [c_void_p, c_int64, c_void_p, c_int64, c_int64, c_void_p, c_int, c_int64, c_void_p]),
    "rsa_fwd_stats": (c_int, [_GEOM, _V, _V, c_void_p, c_int, c_void_p, c_void_p]),
    "rsa_fwd_probs_pv": (c_int, [_GEOM, _V, _V, _V, c_void_p, c_int, _V, _V, c_int, _V, c_void_p]),
    "rsa_fwd_resident": (c_int, [_GEOM, _V, _V, _V, _V, _V, c_void_p, c_void_p]),
    "rsa_fwd_factored": (c_int, [_GEOM, _V, _V, _V, _V, _V, c_void_p, c_void_p, c_void_p]),
    "rsa_fwd_factored_peer": (c_int, [_GEOM, _V, _P(RsaView), _P(RsaView), _V, _V, c_void_p, c_void_p, c_void_p]),
    "rsa_bwd_fused_peer": (c_int, [_GEOM, _V, _P(RsaView), _P(RsaView), _V, _V, c_void_p, _V, _V, _V, c_void_p]),
    "rsa_ipc_alloc": (c_int, [ctypes.c_size_t, _P(c_void_p), c_void_p]),
    "rsa_ipc_open": (c_int, [c_void_p, _P(c_void_p)]),
    "rsa_ipc_close": (c_int, [c_void_p]),
    "rsa_ipc_free": (c_int, [c_void_p]),
    "rsa_bwd_dkdv": (c_int, [_GEOM, _V, _V, _V, _V, c_void_p, _V, _V, c_int, c_int, c_void_p]),
    "rsa_bwd_dq": (c_int, [_GEOM, _V, _V, _V, _V, c_void_p, _V, c_int, _V, c_void_p]),
    "rsa_fused_supported": (c_int, [_GEOM]),
    "rsa_bwd_fused": (c_int, [_GEOM, _V, _V, _V, _V, _V, c_void_p, _V, c_int, _V, _V, _V, c_int, c_int, c_void_p]),
    "rsa_bwd_fused_supported": (c_int, [_GEOM]),
    "rsa_embed": (c_int, [c_void_p, c_int64, c_int64, c_int64, c_void_p, c_void_p, c_int64, c_void_p, c_void_p]),
    "rsa_embed_bwd": (c_int, [c_void_p, c_int64, c_int64, c_int64, c_void_p, c_int64, c_void_p, c_void_p, c_void_p]),
    "rsa_softmax_xent": (c_int, [c_void_p, c_int64, c_void_p, c_int64, c_int64, c_void_p, c_void_p, c_int64, c_float,
                                 c_void_p]),
    "rsa_fwd_factored_ex": (c_int, [_GEOM, _V, _V, _V, _P(RsaFwdExt), _V, c_void_p, c_void_p, c_void_p]),
    "rsa_bwd_kv_stream": (c_int, [_GEOM, _V, _V, _V, _V, c_void_p, c_void_p, _V, _V, c_int, c_int, c_void_p]),
    "rsa_bwd_q_stream": (c_int, [_GEOM, _V, _V, _V, _V, c_void_p, c_void_p, _V, c_int, _V, c_void_p]),
    "rsa_bwd_stream_fused": (c_int, [_GEOM, _V, _V, _V, _V, c_void_p, c_void_p, _V, _V, c_int, c_int, c_void_p, c_int,
                                     _V, c_void_p]),
    "rsa_linformer_project": (c_int, [_GEOM, c_int, c_void_p, c_void_p, c_int64, _V, _V, c_void_p, c_void_p, c_void_p,
                                      c_void_p, c_void_p]),
    "rsa_linformer_proj_grad": (c_int, [_GEOM, c_int, c_void_p, c_void_p, _V, _V, c_void_p, c_void_p, c_int64,
                                        c_void_p]),
    "rsa_linformer_proj_back": (c_int, [_GEOM, c_int, c_void_p, c_void_p, c_int64, c_void_p, c_void_p, _V, _V,
                                        c_void_p]),
    "rsa_bwd_panel_fused": (c_int, [_GEOM, _V, _V, _V, _V, _V, c_void_p, _V, _V, c_int, c_int, c_void_p, c_int, _V,
                                    c_void_p]),
}

_lib = None
_load_error: str | None = None


def lib():
    """Load (once) and return the CDLL; raise NativeUnavailable on failure."""
    global _lib, _load_error
    if _lib is not None:
        return _lib
    if _load_error is not None:
        raise NativeUnavailable(_load_error)
    try:
        handle = ctypes.CDLL(str(LIB_PATH))
    except OSError as exc:
        _load_error = (
            f"cannot load {LIB_PATH}: {exc}. Build it with "
            "`python -c 'import __graft_entry__ as g; g.build()'` (make -C paper_2105_13120_b200/csrc)."
        )
        raise NativeUnavailable(_load_error) from exc
    for name, (restype, argtypes) in EXPORTS.items():
        fn = getattr(handle, name)
        fn.restype = restype
        fn.argtypes = argtypes
    ver = handle.rsa_abi_version()
    if ver != ABI_VERSION:
        _load_error = f"{LIB_PATH} has ABI version {ver}, expected {ABI_VERSION}; rebuild it"
        raise NativeUnavailable(_load_error)
    _lib = handle
    return _lib


def last_error() -> str:
    msg = lib().rsa_last_error()
    return msg.decode() if msg else ""


def check(code: int, what: str) -> None:
    """Raise the boundary exception matching a non-zero status code."""
    if code == RSA_OK:
        return
    msg = f"{what}: {last_error()}"
    if code == RSA_ERR_INVALID:
        raise ShapeError(msg)
    if code == RSA_ERR_NUMERIC:
        raise NumericError(msg)
    raise NativeError(f"[status {code}] {msg}")

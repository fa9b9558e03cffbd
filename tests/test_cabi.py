"""The C ABI library loads and exports exactly what include/rsa_b200.h declares.

CPU-only: nothing here launches a kernel.  Also checks that the ctypes
binding in paper_2105_13120_b200/_native.py covers every declared entry
point, that the library was built for sm_100a, and that the product path
refuses to run without it (no CPU fallback).
"""

from __future__ import annotations

import ctypes
import re
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "rsa_b200.h"
LIB = ROOT / "paper_2105_13120_b200" / "librsa_b200.so"


def declared_functions():
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(rsa_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_boundary():
    names = declared_functions()
    for required in ("rsa_gemm", "rsa_softmax_rows", "rsa_softmax_bwd", "rsa_fwd_stats", "rsa_fwd_probs_pv",
                     "rsa_bwd_dkdv", "rsa_bwd_dq", "rsa_last_error", "rsa_abi_version"):
        assert required in names


@pytest.mark.skipif(not LIB.exists(), reason="librsa_b200.so not built")
def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(str(LIB))
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing
    lib.rsa_abi_version.restype = ctypes.c_int
    from paper_2105_13120_b200 import _native

    assert lib.rsa_abi_version() == _native.ABI_VERSION
    assert set(declared_functions()) == set(_native.EXPORTS), "ctypes binding out of sync with the header"


@pytest.mark.skipif(not LIB.exists(), reason="librsa_b200.so not built")
def test_library_is_sm100a_with_tcgen05_and_tma():
    sass = subprocess.run(["cuobjdump", "-sass", str(LIB)], capture_output=True, text=True).stdout
    assert "sm_100a" in subprocess.run(["cuobjdump", "-lelf", str(LIB)], capture_output=True, text=True).stdout
    assert "UTCHMMA" in sass, "no tcgen05.mma in the library"
    assert "UTMALDG" in sass, "no TMA loads in the library"
    assert "UTMASTG" in sass, "no TMA stores in the library"
    assert "LDTM" in sass, "no tcgen05.ld in the library"


def test_product_path_fails_loudly_without_cuda(monkeypatch):
    import torch

    if torch.cuda.is_available():
        pytest.skip("CUDA present")
    from paper_2105_13120_b200 import AttentionConfig, NativeUnavailable
    from paper_2105_13120_b200.ring_attention import ring_attention_forward

    import numpy as np

    cfg = AttentionConfig(batch_size=1, seq_len=8, hidden_size=4, num_heads=1, head_size=4, num_devices=2)
    chunks = [np.zeros((1, 1, 4, 4))] * 2
    with pytest.raises(NativeUnavailable):
        ring_attention_forward(chunks, chunks, chunks, cfg)

"""Shared pytest configuration.

``-m gpu`` selects the parity tests that need a B200 and the built
librsa_b200.so; ``-m "not gpu"`` runs everything that works on a CPU-only
host (oracle pins, host logic, ledger, C-ABI symbol checks, gloo rings).
"""

from __future__ import annotations

import os
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))

GOLDEN = ROOT / "tests" / "golden" / "ringseq_golden.npz"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA (sm_100a) device and the built extension")


def pytest_collection_modifyitems(config, items):
    # A gpu test collected on a host without CUDA is a configuration error
    # when explicitly requested, and silently deselected otherwise.
    try:
        import torch

        has_cuda = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        has_cuda = False
    if has_cuda:
        return
    markexpr = config.getoption("-m") or ""
    if "gpu" in markexpr and "not gpu" not in markexpr:
        return  # let them run and fail loudly
    skip = pytest.mark.skip(reason="no CUDA device on this host")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@pytest.fixture(scope="session")
def golden():
    data = np.load(GOLDEN)
    return {k: data[k] for k in data.files}


def golden_cases(golden, prefix):
    """{case_key: {field: array}} for one fixture family."""
    out = {}
    for key, val in golden.items():
        fam, case, field = key.split("/")
        if fam == prefix:
            out.setdefault(case, {})[field] = val
    return out

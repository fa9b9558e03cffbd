"""TMA streaming read GB/s: panel-style 64x128 boxes at row stride 2L vs contiguous 32 KB boxes."""
import ctypes
import subprocess
import sys
from pathlib import Path

import torch

here = Path(__file__).resolve().parent
so = here / "tma_stream.so"
if not so.exists():
    subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-shared", "-Xcompiler", "-fPIC",
                    "-o", str(so), str(here / "tma_stream.cu"), "-lcuda"], check=True)
lib = ctypes.CDLL(str(so))
lib.tma_stream.restype = ctypes.c_float
lib.tma_stream.argtypes = [ctypes.c_int, ctypes.c_void_p, ctypes.c_longlong, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int]
buf = torch.empty(4 << 30, dtype=torch.uint8, device="cuda")
for L in [512, 8192]:
    rows = (4 << 30) // (2 * L)
    for mode in (0, 1):
        ms = lib.tma_stream(mode, buf.data_ptr(), rows, L, 5, 6, 0)
        print(f"L={L} {'panel boxes' if mode == 0 else 'contiguous '}: {ms:.3f} ms, {(4 << 30) / ms / 1e6:.0f} GB/s",
              flush=True)
L = 512
rows = (4 << 30) // (2 * L)
for hold in (0, 1000, 2000):
    print(f"hold {hold} clk per tile:", " ".join(
        f"st{st}={(4 << 30) / lib.tma_stream(0, buf.data_ptr(), rows, L, 3, st, hold) / 1e6:.0f}" for st in (1, 2, 3, 4, 6)),
        "GB/s", flush=True)
lib.tma_store_stream.restype = ctypes.c_float
lib.tma_store_stream.argtypes = [ctypes.c_void_p, ctypes.c_longlong, ctypes.c_int, ctypes.c_int, ctypes.c_int]
for L in (512, 8192):
    rows = (4 << 30) // (2 * L)
    print(f"TMA stores, 4 KB per-warp boxes, L={L}:", " ".join(
        f"depth{d}={(4 << 30) / lib.tma_store_stream(buf.data_ptr(), rows, L, 3, d) / 1e6:.0f}" for d in (1, 2)),
        "GB/s", flush=True)
us = here / "umma_rate.so"
if not us.exists():
    subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-shared", "-Xcompiler", "-fPIC",
                    "-o", str(us), str(here / "umma_rate.cu")], check=True)
ul = ctypes.CDLL(str(us))
ul.umma_rate.restype = ctypes.c_double
ul.umma_rate.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int]
for mn in (0, 1):
    print(f"tcgen05.mma SS M=128 K=16 ({'MN' if mn else 'K'}-major operands), clk per instruction, all 148 SMs:",
          " ".join(f"N={n}: {ul.umma_rate(4096, n, mn):.1f}" for n in (64, 128, 256)), flush=True)

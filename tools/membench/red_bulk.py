"""L2 reduction throughput for dQ partials (red_bulk.cu): bulk reduce-add vs bulk store vs red.v4."""
import ctypes
import subprocess
from pathlib import Path

import torch

here = Path(__file__).resolve().parent
so = here / "red_bulk.so"
if not so.exists():
    subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-shared", "-Xcompiler", "-fPIC",
                    "-o", str(so), str(here / "red_bulk.cu")], check=True)
lib = ctypes.CDLL(str(so))
lib.red_bulk.restype = ctypes.c_float
lib.red_bulk.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int, ctypes.c_int]
T, steps = 64, 512
for kpc in (64, 16, 148):  # CTAs per head: 64 (L=8K, one head's key tiles), 16 (L=2K), all on one head
    heads = (148 + kpc - 1) // kpc
    acc = torch.zeros(heads * T * 128 * 64, dtype=torch.float32, device="cuda")
    for mode, name in ((0, "bulk reduce-add"), (1, "bulk store     "), (2, "red.v4 (regs)  ")):
        for depth in ((1, 2, 4) if mode < 2 else (1,)):
            ms = lib.red_bulk(acc.data_ptr(), steps, T, kpc, mode, depth)
            b = 148 * steps * 128 * 64 * 4
            print(f"kpc={kpc:3d} {name} depth {depth}: {ms:.3f} ms, {b / ms / 1e6:.0f} GB/s,"
                  f" {b / 148 / (ms * 1e-3 * 1.965e9):.1f} B/clk/SM", flush=True)

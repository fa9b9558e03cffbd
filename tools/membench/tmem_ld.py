"""TMEM read bytes/clk per SM for 4..16 warps issuing tcgen05.ld 32x32b.x32 (tools/membench/tmem_ld.cu)."""
import ctypes
import subprocess
from pathlib import Path

here = Path(__file__).resolve().parent
so = here / "tmem_ld.so"
if not so.exists():
    subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-shared", "-Xcompiler", "-fPIC",
                    "-o", str(so), str(here / "tmem_ld.cu")], check=True)
lib = ctypes.CDLL(str(so))
lib.tmem_ld_rate.restype = ctypes.c_double
lib.tmem_ld_rate.argtypes = [ctypes.c_int, ctypes.c_int, ctypes.c_int]
for warps in (4, 8, 16):
    print(f"{warps} warps:", " ".join(f"batch{b}={lib.tmem_ld_rate(warps, 4096, b):.0f}" for b in (1, 2, 4)),
          "B/clk/SM", flush=True)

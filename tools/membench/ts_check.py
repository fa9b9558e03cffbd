"""Check the tcgen05 TS-form layout (tools/membench/ts_check.cu) against torch, and time it."""
import ctypes
import subprocess
from pathlib import Path

import torch

here = Path(__file__).resolve().parent
so = here / "ts_check.so"
if not so.exists():
    subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-shared", "-Xcompiler", "-fPIC",
                    "-o", str(so), str(here / "ts_check.cu")], check=True)
lib = ctypes.CDLL(str(so))
g = torch.Generator(device="cuda").manual_seed(0)
for n in (64, 128):
    for b_mn in (0, 1):
        a = torch.randn((128, 64), generator=g, device="cuda").to(torch.bfloat16)
        bm = torch.randn((64, n), generator=g, device="cuda").to(torch.bfloat16)  # K x N
        b_store = bm.contiguous() if b_mn else bm.t().contiguous()  # MN-major: [k][n]; K-major: [n][k]
        d = torch.zeros((128, n), device="cuda")
        clk = torch.zeros(148, dtype=torch.int64, device="cuda")
        rc = lib.ts_check(ctypes.c_void_p(a.data_ptr()), ctypes.c_void_p(b_store.data_ptr()), n, b_mn,
                          ctypes.c_void_p(d.data_ptr()), 1, 1, ctypes.c_void_p(0))
        want = a.float() @ bm.float()
        err = (d - want).abs().max().item()
        lib.ts_check(ctypes.c_void_p(a.data_ptr()), ctypes.c_void_p(b_store.data_ptr()), n, b_mn,
                     ctypes.c_void_p(d.data_ptr()), 1024, 148, ctypes.c_void_p(clk.data_ptr()))
        print(f"N={n} B {'MN' if b_mn else 'K'}-major: rc {rc} max|diff| {err:.3e}; "
              f"{clk.float().mean().item() / 4096:.1f} clk per M128 K16 TS product", flush=True)

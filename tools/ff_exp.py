"""Time one kernel variant per RSA_FF_DBG setting (experiment driver, not a test)."""
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2105_13120_b200 import engine  # noqa: E402

B, Z, L, A = 64, 12, 512, 64
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(0)
q, k, v, dO = (torch.randn((1, B, Z, L, A), generator=g, device=dev).to(torch.bfloat16) for _ in range(4))
out = torch.empty_like(q)
panel = torch.empty((1, B, Z, L, L), dtype=torch.bfloat16, device=dev)
rs = torch.empty((1, B, Z, L), dtype=torch.float32, device=dev)
for dbg in sys.argv[1:]:
    os.environ["RSA_FF_DBG"] = dbg
    for _ in range(3):
        engine.forward(q, k, v, path="fused", out=out, panel=panel, rowscale=rs)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        engine.forward(q, k, v, path="fused", out=out, panel=panel, rowscale=rs)
    e1.record()
    torch.cuda.synchronize()
    print(f"dbg={dbg}: {e0.elapsed_time(e1) / 20 * 1e3:.1f} us", flush=True)

if os.environ.get("TRACE_OUT"):
    os.environ["RSA_FF_DBG"] = "0"
    os.environ["RSA_FF_TRACE"] = os.environ["TRACE_OUT"]
    engine.forward(q, k, v, path="fused", out=out, panel=panel, rowscale=rs)
    torch.cuda.synchronize()
    del os.environ["RSA_FF_TRACE"]

if os.environ.get("BF_TRACE_OUT"):
    out2, panel2, rs2, _ = engine.forward(q, k, v, path="fused")
    for _ in range(2):
        engine.backward(q, k, v, panel2, dO, outputs=out2, rowscale=rs2, path="fused")
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        engine.backward(q, k, v, panel2, dO, outputs=out2, rowscale=rs2, path="fused")
    e1.record()
    torch.cuda.synchronize()
    print(f"bwd (rowdot + bwd_fused): {e0.elapsed_time(e1) / 10 * 1e3:.1f} us", flush=True)
    os.environ["RSA_BF_TRACE"] = os.environ["BF_TRACE_OUT"]
    engine.backward(q, k, v, panel2, dO, outputs=out2, rowscale=rs2, path="fused")
    torch.cuda.synchronize()
    del os.environ["RSA_BF_TRACE"]

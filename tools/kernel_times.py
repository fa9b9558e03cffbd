import sys, torch
sys.path.insert(0, '/root/repo')
from paper_2105_13120_b200 import engine
dev = torch.device('cuda', 0)
for (n, b, z, L) in [(8, 4, 16, 16384), (1, 4, 12, 8192), (1, 64, 12, 512)]:
    c = L // n
    g = torch.Generator(device=dev).manual_seed(0)
    q, k, v, d = (torch.randn((n, b, z, c, 64), generator=g, device=dev).to(torch.bfloat16) for _ in range(4))
    tm = engine.KernelTimer()
    for it in range(3):
        if it == 2: tm.reset()
        f = engine.forward(q, k, v, path='fused', timer=tm)
        engine.backward(q, k, v, f.panel, d, outputs=f.out, rowscale=f.rowscale, path='fused', timer=tm)
    tot = tm.totals()
    pe = n * b * z * c * L
    print((n, b, z, L), {k: round(v[1] * 1e3 / v[0], 1) for k, v in tot.items()}, 'P_e GB bf16', pe * 2 / 1e9)

import sys, time, torch
sys.path.insert(0, '/root/repo')
from paper_2105_13120_b200 import engine
dev = torch.device('cuda', 0)
B, Z, L, A = 64, 12, 512, 64
g = torch.Generator(device=dev).manual_seed(0)
layers = []
for _ in range(12):
    ly = {k: torch.randn((1, B, Z, L, A), generator=g, device=dev).to(torch.bfloat16) for k in 'qkvg'}
    ly['o'] = torch.empty_like(ly['q']); ly['p'] = torch.empty((1, B, Z, L, L), dtype=torch.bfloat16, device=dev)
    ly['r'] = torch.empty((1, B, Z, L), dtype=torch.float32, device=dev)
    ly['grads'] = tuple(torch.empty_like(ly['q']) for _ in range(3))
    layers.append(ly)
flag = torch.zeros(1, dtype=torch.int32, device=dev)
dvec = torch.empty((1, B, Z, L), dtype=torch.float32, device=dev); gs = torch.empty_like(layers[0]['q'])
def step():
    for ly in layers:
        engine.forward(ly['q'], ly['k'], ly['v'], path='fused', flag=flag, out=ly['o'], panel=ly['p'], rowscale=ly['r'])
    for ly in reversed(layers):
        engine.backward(ly['q'], ly['k'], ly['v'], ly['p'], ly['g'], outputs=ly['o'], path='fused', grads=ly['grads'], dvec=dvec, rowscale=ly['r'], grad_scaled=gs)
for _ in range(3): step()
torch.cuda.synchronize()
t0 = time.perf_counter()
for _ in range(20): step()
t1 = time.perf_counter()
torch.cuda.synchronize()
t2 = time.perf_counter()
print(f"cpu enqueue per step {(t1-t0)/20*1e3:.2f} ms, wall per step {(t2-t0)/20*1e3:.2f} ms")

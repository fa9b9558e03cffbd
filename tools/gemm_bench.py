"""Our rsa_gemm (tcgen05) against cuBLAS (torch.matmul) on BERT-base projection / weight-gradient shapes."""
import sys, torch
sys.path.insert(0, '/root/repo')
from paper_2105_13120_b200 import tensor_ops as ops
dev = torch.device('cuda', 0)
def t(fn, it=10):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(it): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / it
for (M, N, K) in [(32768, 768, 768), (32768, 3072, 768), (32768, 768, 3072), (768, 768, 32768), (768, 3072, 32768)]:
    od = torch.float32 if K > M else torch.bfloat16  # weight gradients accumulate in fp32
    a = torch.randn((M, K), device=dev).to(torch.bfloat16)
    b = torch.randn((K, N), device=dev).to(torch.bfloat16)
    ms_r = t(lambda: ops.matmul(a, b, out_dtype=od))
    ms_c = t(lambda: torch.matmul(a, b))
    f = 2 * M * N * K
    print(M, N, K, str(od), f"rsa {f / ms_r / 1e9:.0f} TF/s  cublas {f / ms_c / 1e9:.0f} TF/s")

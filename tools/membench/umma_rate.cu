// Experiment (not product code): cycles per tcgen05.mma (cta_group::1, kind::f16, bf16 in,
// fp32 accumulate, K = 16) issued back to back, with both operands in shared memory (SS),
// for M = 128 and N = 64 / 128 / 256, K-major or MN-major operands.  One CTA per SM.
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

#include "../../paper_2105_13120_b200/csrc/ptx.cuh"

using namespace rsa;

__global__ void __launch_bounds__(128, 1) umma_kernel(int n_mma, int N, int mn, long long* out) {
  extern __shared__ uint8_t raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 96 * 1024);
  uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 1);
  const int warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < 96 * 1024 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0x3f803f80u;
  if (warp == 0) tmem_alloc(slot, 256);
  if (threadIdx.x == 0) mbar_init(bar, 1), fence_barrier_init();
  fence_proxy_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *slot;
  if (warp == 0) {
    const uint32_t idesc = idesc_bf16_f32(128, N, mn, mn);
    const uint32_t a = smem_u32(smem), b = smem_u32(smem + 32 * 1024);
    const uint64_t da = mn ? smem_desc_sw128(a, 16384, 1024) : smem_desc_sw128(a, 0, 1024);
    const uint64_t db = mn ? smem_desc_sw128(b, 16384, 1024) : smem_desc_sw128(b, 0, 1024);
    const long long t0 = clock64();
    for (int i = 0; i < n_mma; ++i) {
      const int k = i & 3;  // walk the 4 K-steps of a 64-wide K-major atom (or 4 MN-major 16-row groups)
      const uint64_t off = mn ? uint64_t(128 * k) : uint64_t(2 * k);
      umma_bf16_ws(tmem, da + off, db + off, idesc, i > 0);
    }
    umma_commit_ws(bar);
    mbar_wait(bar, 0);
    const long long t1 = clock64();
    if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 256);
}

extern "C" double umma_rate(int n_mma, int N, int mn) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  long long* d;
  cudaMalloc(&d, sms * sizeof(long long));
  const int smem = 96 * 1024 + 2048;
  cudaFuncSetAttribute(umma_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  umma_kernel<<<sms, 128, smem>>>(n_mma, N, mn, d);
  umma_kernel<<<sms, 128, smem>>>(n_mma, N, mn, d);
  long long h[256];
  cudaMemcpy(h, d, sms * sizeof(long long), cudaMemcpyDeviceToHost);
  cudaFree(d);
  if (cudaGetLastError() != cudaSuccess) return -1;
  double s = 0;
  for (int i = 0; i < sms; ++i) s += double(h[i]);
  return s / sms / n_mma;
}

// Experiment (not product code): TMEM read throughput.  `warps` warps of one CTA per SM each
// issue tcgen05.ld.32x32b.x32 (32 lanes x 32 columns x 4 B = 4 KB) back to back over
// their lane quarter (warp w -> lanes 32*(w%4)), waiting after every `batch` loads, and
// report clk per 4 KB load per warp -> bytes/clk per SM.
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

#include "../../paper_2105_13120_b200/csrc/ptx.cuh"

using namespace rsa;

__global__ void __launch_bounds__(512, 1) tmem_ld_kernel(int iters, int batch, long long* out, float* sink) {
  __shared__ uint32_t slot;
  const int warp = threadIdx.x >> 5;
  if (warp == 0) tmem_alloc(&slot, 512);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  const uint32_t base = tmem + ((uint32_t(warp & 3) * 32u) << 16) + uint32_t((warp >> 2) * 64) % 512u;
  float acc = 0.f;
  __syncthreads();
  const long long t0 = clock64();
  for (int i = 0; i < iters; i += batch) {
    for (int j = 0; j < batch; ++j) {
      float v[32];
      tmem_ld32(base + uint32_t(((i + j) * 32) % 256), v);
      if (j == batch - 1) {
        tmem_ld_wait();
#pragma unroll
        for (int e = 0; e < 32; ++e) acc += v[e];
      }
    }
  }
  tmem_ld_wait();
  const long long t1 = clock64();
  __syncthreads();
  if ((threadIdx.x & 31) == 0) out[blockIdx.x * 16 + warp] = t1 - t0;
  if (acc == 12345.f) sink[threadIdx.x] = acc;
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 512);
}

extern "C" double tmem_ld_rate(int warps, int iters, int batch) {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  long long* d;
  float* sink;
  cudaMalloc(&d, sms * 16 * sizeof(long long));
  cudaMalloc(&sink, 4096);
  tmem_ld_kernel<<<sms, 32 * warps>>>(iters, batch, d, sink);
  tmem_ld_kernel<<<sms, 32 * warps>>>(iters, batch, d, sink);
  static long long h[256 * 16];
  cudaMemcpy(h, d, sms * 16 * sizeof(long long), cudaMemcpyDeviceToHost);
  cudaFree(d);
  cudaFree(sink);
  if (cudaGetLastError() != cudaSuccess) return -1;
  double mx = 0;  // slowest warp of each SM, averaged
  for (int s = 0; s < sms; ++s) {
    long long m = 0;
    for (int w = 0; w < warps; ++w) m = h[s * 16 + w] > m ? h[s * 16 + w] : m;
    mx += double(m);
  }
  mx /= sms;
  return double(warps) * iters * 4096.0 / mx;  // bytes per clk per SM
}

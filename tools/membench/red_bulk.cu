// Experiment (not product code): L2 reduction throughput for a dQ-partial accumulate.
// 148 CTAs (one per SM); CTA c belongs to "head" c / kpc and, at step s, adds a 32 KB fp32
// tile (128 query rows x 64) into tile (c + s) % T of its head's dQ accumulator -- the
// pattern of a stream backward whose CTAs own key tiles and walk every query tile.
//   mode 0: cp.reduce.async.bulk .add.f32 from shared memory (TMA unit), `depth` in flight
//   mode 1: cp.async.bulk plain store from shared memory (reference write rate)
//   mode 2: red.global.add.v4.f32 from registers, 128 threads (one 64-float row each)
// Returns ms for `steps` steps per CTA.
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

#include "../../paper_2105_13120_b200/csrc/ptx.cuh"

using namespace rsa;

constexpr int TILE_B = 128 * 64 * 4;

__global__ void __launch_bounds__(128, 1) red_kernel(float* acc, int steps, int T, int kpc, int mode, int depth) {
  extern __shared__ __align__(1024) uint8_t sm[];
  float* buf = reinterpret_cast<float*>(sm);
  for (int i = threadIdx.x; i < TILE_B / 4; i += blockDim.x) buf[i] = 1.0f / 1024;
  __syncthreads();
  fence_proxy_async_smem();
  const int head = blockIdx.x / kpc;
  float* base = acc + size_t(head) * T * (TILE_B / 4);
  if (mode < 2) {
    if (threadIdx.x == 0) {
      for (int s = 0; s < steps; ++s) {
        float* dst = base + size_t((blockIdx.x + s) % T) * (TILE_B / 4);
        if (mode == 0)
          asm volatile("cp.reduce.async.bulk.global.shared::cta.bulk_group.add.f32 [%0], [%1], %2;" ::"l"(dst),
                       "r"(smem_u32(buf)), "r"(TILE_B)
                       : "memory");
        else
          asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(smem_u32(buf)),
                       "r"(TILE_B)
                       : "memory");
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        if (depth <= 1) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        else if (depth == 2) asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
        else asm volatile("cp.async.bulk.wait_group.read 3;" ::: "memory");
      }
      asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
    }
  } else {
    const int r = threadIdx.x;
    for (int s = 0; s < steps; ++s) {
      float* dst = base + size_t((blockIdx.x + s) % T) * (TILE_B / 4) + r * 64;
#pragma unroll
      for (int j = 0; j < 64; j += 4) {
        const float v = 1.0f / 1024;
        asm volatile("red.relaxed.gpu.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(dst + j), "f"(v), "f"(v),
                     "f"(v), "f"(v)
                     : "memory");
      }
    }
  }
}

extern "C" float red_bulk(float* acc, int steps, int T, int kpc, int mode, int depth) {
  cudaFuncSetAttribute(red_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, TILE_B + 1024);
  red_kernel<<<148, 128, TILE_B + 1024>>>(acc, 4, T, kpc, mode, depth);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0), cudaEventCreate(&e1);
  cudaEventRecord(e0);
  red_kernel<<<148, 128, TILE_B + 1024>>>(acc, steps, T, kpc, mode, depth);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  cudaError_t err = cudaGetLastError();
  if (err != cudaSuccess) printf("error %s\n", cudaGetErrorString(err));
  return ms;
}

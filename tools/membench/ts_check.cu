// Experiment (not product code): the tcgen05.mma "TS" form (A from TMEM) -- layout check and
// rate.  A (128 x 64 bf16) is written to TMEM with tcgen05.st (lane m = row m, column j =
// the pair (2j, 2j+1) of K), B (64 x N bf16, K x N) sits in shared memory in the SW128 layout
// either K-major (rows = n) or MN-major (rows = k); D = A B (fp32, 128 x N) is read back.
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

#include "../../paper_2105_13120_b200/csrc/ptx.cuh"

using namespace rsa;

__global__ void __launch_bounds__(128, 1) ts_kernel(const __nv_bfloat16* a, const __nv_bfloat16* b, int n, int b_mn,
                                                    float* d, int reps, long long* clk) {
  extern __shared__ uint8_t raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 64 * 1024);
  uint32_t* slot = reinterpret_cast<uint32_t*>(bar + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // B into smem, SW128 atoms of 128 rows x 128 B
  if (!b_mn) {  // K-major: row = n (N rows), 64 k per row
    for (int idx = threadIdx.x; idx < n * 8; idx += blockDim.x) {
      const int row = idx / 8, ch = idx % 8;
      const uint4 v = *reinterpret_cast<const uint4*>(b + row * 64 + ch * 8);  // b stored [n][k]
      *reinterpret_cast<uint4*>(smem + sw128_offset(row, ch)) = v;
    }
  } else {  // MN-major: row = k (64 rows), 64 n per atom, atoms of 64 n at +16 KB
    for (int idx = threadIdx.x; idx < 64 * (n / 8); idx += blockDim.x) {
      const int k = idx / (n / 8), c8 = idx % (n / 8), atom = c8 / 8, ch = c8 % 8;
      const uint4 v = *reinterpret_cast<const uint4*>(b + k * n + c8 * 8);  // b stored [k][n]
      *reinterpret_cast<uint4*>(smem + atom * 16384 + sw128_offset(k, ch)) = v;
    }
  }
  fence_proxy_async_smem();
  if (warp == 0) tmem_alloc(slot, 256);
  if (threadIdx.x == 0) mbar_init(bar, 1), fence_barrier_init();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *slot;
  const int row = warp * 32 + lane;
  {  // A row `row` -> TMEM lane row, columns 128..159 (bf16 pairs)
    uint32_t w[32];
    for (int j = 0; j < 32; ++j) {
      const __nv_bfloat162 p = *reinterpret_cast<const __nv_bfloat162*>(a + row * 64 + 2 * j);
      w[j] = *reinterpret_cast<const uint32_t*>(&p);
    }
    tmem_st32(tmem + ((uint32_t(warp) * 32u) << 16) + 128, w);
    tmem_st_wait();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  long long t0 = 0, t1 = 0;
  if (warp == 0) {
    const uint32_t idesc = idesc_bf16_f32(128, n, 0, b_mn);
    const uint32_t bb = smem_u32(smem);
    t0 = clock64();
    for (int r = 0; r < reps; ++r)
      for (int k = 0; k < 4; ++k) {
        const uint64_t db = b_mn ? smem_desc_sw128(bb + k * 2048, 16384, 1024) : smem_desc_sw128(bb + k * 32, 0, 1024);
        umma_bf16_ts_ws(tmem, tmem + 128 + 8 * k, db, idesc, k > 0);
      }
    umma_commit_ws(bar);
    mbar_wait(bar, 0);
    t1 = clock64();
    if (lane == 0 && clk) clk[blockIdx.x] = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  for (int c0 = 0; c0 < n; c0 += 32) {
    float v[32];
    tmem_ld32(tmem + ((uint32_t(warp) * 32u) << 16) + c0, v);
    tmem_ld_wait();
    if (blockIdx.x == 0)
      for (int j = 0; j < 32; ++j) d[row * n + c0 + j] = v[j];
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) tmem_dealloc(tmem, 256);
}

extern "C" int ts_check(const void* a, const void* b, int n, int b_mn, float* d, int reps, int grid, long long* clk) {
  const int smem = 64 * 1024 + 2048;
  cudaFuncSetAttribute(ts_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  ts_kernel<<<grid, 128, smem>>>(static_cast<const __nv_bfloat16*>(a), static_cast<const __nv_bfloat16*>(b), n, b_mn,
                                 d, reps, clk);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) printf("cuda error %s\n", cudaGetErrorString(e));
  return int(e);
}

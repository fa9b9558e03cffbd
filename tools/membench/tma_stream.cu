// Experiment (not product code): TMA streaming read bandwidth of a bf16 [rows][L] array,
// panel-style boxes (64 cols x 128 rows at a row stride of 2L bytes) versus the same
// bytes as contiguous 32 KB boxes.  Each CTA keeps STAGES tiles in flight.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

#include "../../paper_2105_13120_b200/csrc/ptx.cuh"

using namespace rsa;
constexpr int MAXST = 6;
constexpr uint32_t TILE_B = 32768;

struct Args {
  CUtensorMap m;
  int mode;  // 0: panel boxes, 1: contiguous
  int L, tiles_per_row_block, n_tiles, stages, hold;
};

__global__ void __launch_bounds__(64, 1) stream_kernel(const __grid_constant__ Args a) {
  extern __shared__ uint8_t raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + MAXST * TILE_B);
  const int STAGES = a.stages;
  uint64_t* empty = full + MAXST;
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) mbar_init(&full[s], 1), mbar_init(&empty[s], 1);
    fence_barrier_init();
  }
  __syncthreads();
  const int per = (a.n_tiles + gridDim.x - 1) / gridDim.x;
  const int t0 = blockIdx.x * per, t1 = min(a.n_tiles, t0 + per);
  if (threadIdx.x == 0) {
    for (int t = t0, i = 0; t < t1; ++t, ++i) {
      const int s = i % STAGES;
      mbar_wait(&empty[s], ((i / STAGES) & 1) ^ 1);
      mbar_arrive_expect_tx(&full[s], TILE_B);
      if (a.mode == 0) {  // tile t: row block t / tpr, key tile t % tpr
        const int rb = t / a.tiles_per_row_block, kt = t % a.tiles_per_row_block;
        tma_load_2d(smem + s * TILE_B, &a.m, &full[s], kt * 128, rb * 128);
        tma_load_2d(smem + s * TILE_B + 16384, &a.m, &full[s], kt * 128 + 64, rb * 128);
      } else {
        tma_load_2d(smem + s * TILE_B, &a.m, &full[s], 0, t * 256);
      }
    }
  } else if (threadIdx.x == 32) {
    for (int t = t0, i = 0; t < t1; ++t, ++i) {
      const int s = i % STAGES;
      mbar_wait(&full[s], (i / STAGES) & 1);
      if (a.hold) {  // hold the slot a while, as a consumer that processes the tile would
        const long long t_0 = clock64();
        while (clock64() - t_0 < a.hold) {
        }
      }
      mbar_arrive(&empty[s]);
    }
  }
}

static PFN_cuTensorMapEncodeTiled_v12000 enc() {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
}

extern "C" float tma_stream(int mode, void* ptr, long long rows, int L, int iters, int stages, int hold) {
  Args a{};
  a.mode = mode, a.L = L, a.stages = stages, a.hold = hold;
  const long long bytes = rows * L * 2;
  a.n_tiles = int(bytes / TILE_B);
  a.tiles_per_row_block = L / 128;
  cuuint64_t dims[2], str[1];
  cuuint32_t box[2], es[2] = {1, 1};
  if (mode == 0) dims[0] = L, dims[1] = rows, str[0] = uint64_t(L) * 2, box[0] = 64, box[1] = 128;
  else dims[0] = 64, dims[1] = bytes / 128, str[0] = 128, box[0] = 64, box[1] = 256;
  if (enc()(&a.m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, ptr, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
      CUDA_SUCCESS)
    return -1.f;
  const int smem = MAXST * TILE_B + 2048;
  cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  stream_kernel<<<sms, 64, smem>>>(a);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0), cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int i = 0; i < iters; ++i) stream_kernel<<<sms, 64, smem>>>(a);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  return cudaGetLastError() == cudaSuccess ? ms / iters : -2.f;
}

__device__ __forceinline__ void tma_store_2d_(const CUtensorMap* map, const void* src, int c0, int c1) {
  asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                   reinterpret_cast<uint64_t>(map)),
               "r"(smem_u32(src)), "r"(c0), "r"(c1)
               : "memory");
}

// TMA store streaming: 8 warps, each storing 4 KB boxes (64 cols x 32 rows) of a bf16
// [rows][L] array like fwd_factored's per-warp P~ stores, keeping `depth` stores in flight.
struct StArgs {
  CUtensorMap m;
  int L, n_tiles, depth;  // tiles of 128 rows x 128 cols (8 boxes each)
};

__global__ void __launch_bounds__(256, 1) store_kernel(const __grid_constant__ StArgs a) {
  extern __shared__ uint8_t raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int per = (a.n_tiles + gridDim.x - 1) / gridDim.x;
  const int t0 = blockIdx.x * per, t1 = min(a.n_tiles, t0 + per);
  const int tpr = a.L / 128;
  if (lane == 0) {
    for (int t = t0; t < t1; ++t) {
      const int rb = t / tpr, kt = t % tpr;
      // warp w: rows 32 * (w & 3).., columns 64 * (w >> 2)..
      if (a.depth == 1) tma_store_wait_read<0>();
      else tma_store_wait_read<1>();
      tma_store_2d_(&a.m, smem + warp * 4096, kt * 128 + (warp >> 2) * 64, rb * 128 + (warp & 3) * 32);
      tma_store_commit();
    }
    tma_store_wait_all<0>();
  }
}

extern "C" float tma_store_stream(void* ptr, long long rows, int L, int iters, int depth) {
  StArgs a{};
  a.L = L, a.depth = depth;
  const long long bytes = rows * L * 2;
  a.n_tiles = int(bytes / TILE_B);
  cuuint64_t dims[2] = {cuuint64_t(L), cuuint64_t(rows)}, str[1] = {cuuint64_t(L) * 2};
  cuuint32_t box[2] = {64, 32}, es[2] = {1, 1};
  if (enc()(&a.m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, ptr, dims, str, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) !=
      CUDA_SUCCESS)
    return -1.f;
  const int smem = 8 * 4096 + 2048;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  store_kernel<<<sms, 256, smem>>>(a);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0), cudaEventCreate(&e1);
  cudaEventRecord(e0);
  for (int i = 0; i < iters; ++i) store_kernel<<<sms, 256, smem>>>(a);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  return cudaGetLastError() == cudaSuccess ? ms / iters : -2.f;
}

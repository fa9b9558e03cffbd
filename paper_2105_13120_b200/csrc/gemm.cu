// Batched GEMM for `matmul` (ringseq/tensor_ops.py:44-72) and the staged
// RSA path.
//
// tcgen05 path: a persistent, warp-specialised kernel (one CTA per SM, 6 warps)
// walking (split, batch, 128 x BN tile) work items.  Warp 0 lane 0 streams A/B
// k-blocks (64 bf16 = one 128-byte swizzle row) through a 4-stage TMA ring;
// warp 1 issues tcgen05.mma (M=128, N=BN, K=16) into one of two TMEM
// accumulators while warps 2..5 drain the other (warp w owns TMEM lanes
// 32*(w%4).. = tile rows) and store fp32/bf16 rows with 256-bit accesses.
// fp32 outputs may split K: the slices of a tile add into C in slice order,
// gated by per-tile counters (deterministic, no atomics on the data).
// Operand majors are runtime: K-major tiles are single TMA boxes of
// 64 x rows; MN-major tiles are 64-wide boxes stacked 8 KB apart, which the
// UMMA MN-major descriptor walks with LBO = 8 KB, SBO = 1 KB.
//
// SIMT path: a plain fp32-accumulating kernel for layouts TMA cannot
// describe (odd strides, fp32 operands, head sizes like 2 or 5 from the
// reference's tests).  Both are CUDA; there is no host fallback.
#include <algorithm>

#include "common.h"
#include "ptx.cuh"

namespace rsa {
namespace {

constexpr int BM = 128;
constexpr int BK = 64;
constexpr int STAGES = 4;

struct GemmArgs {
  CUtensorMap ta;
  CUtensorMap tb;
  int M, N, K;
  int a_mn, b_mn;
  int nb2;
  int a_bc1, a_bc2, b_bc1, b_bc2;
  int n_tiles;   // N tiles
  int mn_tiles;  // M tiles * N tiles
  int batches;
  int splits;    // split-K slices (1: none); slices of a tile add into C in slice order
  int* flags;    // per (batch, tile) count of finished slices (split-K only)
  void* C;
  int c_bf16;
  int vec_ok;
  int64_t ldc, c_s1, c_s2;
  float alpha;
  int accumulate;
};

template <int BN>
struct GemmSmem {
  static constexpr uint32_t A_BYTES = BM * BK * 2;
  static constexpr uint32_t B_BYTES = BN * BK * 2;
  static constexpr uint32_t STAGE_BYTES = A_BYTES + B_BYTES;
  static constexpr uint32_t BAR_OFF = STAGES * STAGE_BYTES;
  static constexpr uint32_t TOTAL = BAR_OFF + 256 + 1024;  // barriers + alignment slack
  static constexpr uint32_t TMEM_COLS = 2 * BN < 32 ? 32 : 2 * BN;
};

struct Work {  // item -> (slice, batch, tile); slice-major, so every slice waits only on earlier items
  int ks, b1, b2, m0, n0, kb0, kb1, flag;
};

__device__ __forceinline__ Work work_of(const GemmArgs& p, int item, int kblocks, int bn) {
  Work w;
  const int per_split = p.batches * p.mn_tiles;
  w.ks = item / per_split;
  const int rem = item % per_split;
  const int bidx = rem / p.mn_tiles, tile = rem % p.mn_tiles;
  w.b1 = bidx / p.nb2, w.b2 = bidx % p.nb2;
  w.m0 = (tile / p.n_tiles) * BM;
  w.n0 = (tile % p.n_tiles) * bn;
  const int ksz = (kblocks + p.splits - 1) / p.splits;
  w.kb0 = w.ks * ksz;
  w.kb1 = min(kblocks, w.kb0 + ksz);
  w.flag = rem;
  return w;
}

// Persistent, warp-specialised tcgen05 GEMM: warp 0 streams A/B k-blocks through a
// 4-stage TMA ring, warp 1 issues tcgen05.mma into one of two TMEM accumulators, warps
// 2..5 drain the other accumulator (warp w owns TMEM lanes 32 * (w % 4) = tile rows),
// so a tile's epilogue overlaps the next tile's MMAs.
template <int BN>
__global__ void __launch_bounds__(192, 1) gemm_tc_kernel(const __grid_constant__ GemmArgs p) {
  using S = GemmSmem<BN>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S::BAR_OFF);
  uint64_t* empty = full + STAGES;
  uint64_t* acc_full = empty + STAGES;
  uint64_t* acc_empty = acc_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

  const uint32_t warp = warp_id(), lane = lane_id();
  const int kblocks = (p.K + BK - 1) / BK;
  const int items = p.splits * p.batches * p.mn_tiles;

  if (warp == 1) tmem_alloc(tmem_slot, S::TMEM_COLS);
  if (threadIdx.x == 0) {
    for (int s = 0; s < STAGES; ++s) mbar_init(&full[s], 1), mbar_init(&empty[s], 1);
    for (int s = 0; s < 2; ++s) mbar_init(&acc_full[s], 1), mbar_init(&acc_empty[s], 4);
    fence_barrier_init();
    tma_prefetch(&p.ta);
    tma_prefetch(&p.tb);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base(tmem_slot);

  if (warp == 0) {
    if (lane == 0) {
      uint32_t it = 0;
      for (int item = blockIdx.x; item < items; item += gridDim.x) {
        const Work w = work_of(p, item, kblocks, BN);
        const int ab1 = p.a_bc1 ? 0 : w.b1, ab2 = p.a_bc2 ? 0 : w.b2;
        const int bb1 = p.b_bc1 ? 0 : w.b1, bb2 = p.b_bc2 ? 0 : w.b2;
        for (int kb = w.kb0; kb < w.kb1; ++kb, ++it) {
          const uint32_t s = it % STAGES;
          mbar_wait(&empty[s], ((it / STAGES) & 1) ^ 1);
          mbar_arrive_expect_tx(&full[s], S::STAGE_BYTES);
          uint8_t* sa = smem + s * S::STAGE_BYTES;
          uint8_t* sb = sa + S::A_BYTES;
          const int k0 = kb * BK;
          if (!p.a_mn) {
            tma_load_4d(sa, &p.ta, &full[s], k0, w.m0, ab2, ab1);
          } else {
            tma_load_4d(sa, &p.ta, &full[s], w.m0, k0, ab2, ab1);
            tma_load_4d(sa + 8192, &p.ta, &full[s], w.m0 + 64, k0, ab2, ab1);
          }
          if (!p.b_mn) {
            tma_load_4d(sb, &p.tb, &full[s], k0, w.n0, bb2, bb1);
          } else {
#pragma unroll
            for (int i = 0; i < BN / 64; ++i) tma_load_4d(sb + i * 8192, &p.tb, &full[s], w.n0 + 64 * i, k0, bb2, bb1);
          }
        }
      }
    }
  } else if (warp == 1) {
    const uint32_t idesc = idesc_bf16_f32(BM, BN, p.a_mn, p.b_mn);
    uint32_t it = 0, tn = 0;
    for (int item = blockIdx.x; item < items; item += gridDim.x, ++tn) {
      const Work w = work_of(p, item, kblocks, BN);
      const uint32_t ab = tn & 1;
      mbar_wait(&acc_empty[ab], ((tn >> 1) & 1) ^ 1);
      tc_fence_after();
      for (int kb = w.kb0; kb < w.kb1; ++kb, ++it) {
        const uint32_t s = it % STAGES;
        mbar_wait(&full[s], (it / STAGES) & 1);
        tc_fence_after();
        const uint32_t sa = smem_u32(smem + s * S::STAGE_BYTES);
        const uint32_t sb = sa + S::A_BYTES;
#pragma unroll
        for (int k = 0; k < BK / 16; ++k) {
          const uint64_t ad = p.a_mn ? smem_desc_sw128(sa + k * 2048, 8192, 1024) : smem_desc_sw128(sa + k * 32, 0, 1024);
          const uint64_t bd = p.b_mn ? smem_desc_sw128(sb + k * 2048, 8192, 1024) : smem_desc_sw128(sb + k * 32, 0, 1024);
          umma_bf16_ws(tmem + ab * BN, ad, bd, idesc, (kb > w.kb0 || k > 0) ? 1u : 0u);
        }
        umma_commit_ws(&empty[s]);
      }
      umma_commit_ws(&acc_full[ab]);
    }
  } else {
    const uint32_t quad = warp & 3;
    uint32_t tn = 0;
    for (int item = blockIdx.x; item < items; item += gridDim.x, ++tn) {
      const Work w = work_of(p, item, kblocks, BN);
      const uint32_t ab = tn & 1;
      if (p.splits > 1 && w.ks > 0) {  // add into C only after the previous slice has
        if (threadIdx.x == 64) {
          volatile int* f = p.flags + w.flag;
          while (*f < w.ks) __nanosleep(64);
          __threadfence();
        }
        asm volatile("bar.sync 1, 128;" ::: "memory");
      }
      mbar_wait(&acc_full[ab], (tn >> 1) & 1);
      tc_fence_after();
      const int row = w.m0 + quad * 32 + lane;
      const int64_t cbase = int64_t(w.b1) * p.c_s1 + int64_t(w.b2) * p.c_s2 + int64_t(row) * p.ldc;
      const bool acc = p.accumulate || w.ks > 0;
#pragma unroll 1
      for (int cc = 0; cc < BN / 32; ++cc) {
        float v[32];
        __syncwarp();
        tmem_ld32(tmem + ((quad * 32u) << 16) + ab * BN + cc * 32, v);
        tmem_ld_wait();
        const int col0 = w.n0 + cc * 32;
        if (row >= p.M || col0 >= p.N) continue;
        const bool full_chunk = p.vec_ok && (col0 + 32 <= p.N);
        if (!p.c_bf16) {
          float* c = reinterpret_cast<float*>(p.C) + cbase + col0;
          if (full_chunk && (reinterpret_cast<uintptr_t>(c) & 31) == 0) {
            // 256-bit loads / stores: whole 32-byte sectors (each warp instruction touches 32 rows)
#pragma unroll
            for (int i = 0; i < 32; i += 8) {
              float o[8];
#pragma unroll
              for (int e = 0; e < 8; ++e) o[e] = p.alpha * v[i + e];
              if (acc) {
                float q[8];
                asm volatile("ld.global.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
                             : "=f"(q[0]), "=f"(q[1]), "=f"(q[2]), "=f"(q[3]), "=f"(q[4]), "=f"(q[5]), "=f"(q[6]),
                               "=f"(q[7])
                             : "l"(c + i));
#pragma unroll
                for (int e = 0; e < 8; ++e) o[e] += q[e];
              }
              asm volatile("st.global.v8.f32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(c + i), "f"(o[0]),
                           "f"(o[1]), "f"(o[2]), "f"(o[3]), "f"(o[4]), "f"(o[5]), "f"(o[6]), "f"(o[7])
                           : "memory");
            }
          } else if (full_chunk) {
#pragma unroll
            for (int i = 0; i < 32; i += 4) {
              float4 o = make_float4(p.alpha * v[i], p.alpha * v[i + 1], p.alpha * v[i + 2], p.alpha * v[i + 3]);
              if (acc) {
                const float4 old = *reinterpret_cast<const float4*>(c + i);
                o.x += old.x, o.y += old.y, o.z += old.z, o.w += old.w;
              }
              *reinterpret_cast<float4*>(c + i) = o;
            }
          } else {
#pragma unroll
            for (int i = 0; i < 32; ++i)
              if (col0 + i < p.N) c[i] = p.alpha * v[i] + (acc ? c[i] : 0.f);
          }
        } else {
          __nv_bfloat16* c = reinterpret_cast<__nv_bfloat16*>(p.C) + cbase + col0;
          if (acc) {
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] = p.alpha * v[i] + ((col0 + i < p.N) ? __bfloat162float(c[i]) : 0.f);
          } else {
#pragma unroll
            for (int i = 0; i < 32; ++i) v[i] *= p.alpha;
          }
          if (full_chunk && (reinterpret_cast<uintptr_t>(c) & 31) == 0) {
#pragma unroll
            for (int i = 0; i < 32; i += 16)
              asm volatile("st.global.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(c + i),
                           "r"(pack_bf16(v[i], v[i + 1])), "r"(pack_bf16(v[i + 2], v[i + 3])),
                           "r"(pack_bf16(v[i + 4], v[i + 5])), "r"(pack_bf16(v[i + 6], v[i + 7])),
                           "r"(pack_bf16(v[i + 8], v[i + 9])), "r"(pack_bf16(v[i + 10], v[i + 11])),
                           "r"(pack_bf16(v[i + 12], v[i + 13])), "r"(pack_bf16(v[i + 14], v[i + 15]))
                           : "memory");
          } else if (full_chunk) {
#pragma unroll
            for (int i = 0; i < 32; i += 8) {
              uint4 o = make_uint4(pack_bf16(v[i], v[i + 1]), pack_bf16(v[i + 2], v[i + 3]),
                                   pack_bf16(v[i + 4], v[i + 5]), pack_bf16(v[i + 6], v[i + 7]));
              *reinterpret_cast<uint4*>(c + i) = o;
            }
          } else {
#pragma unroll
            for (int i = 0; i < 32; ++i)
              if (col0 + i < p.N) c[i] = __float2bfloat16_rn(v[i]);
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[ab]);
      if (p.splits > 1 && w.ks + 1 < p.splits) {  // publish this slice to the next one
        __threadfence();
        asm volatile("bar.sync 1, 128;" ::: "memory");
        if (threadIdx.x == 64) atomicAdd(p.flags + w.flag, 1);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, S::TMEM_COLS);
}

// ----------------------------------------------------------- SIMT path

template <typename T>
__device__ __forceinline__ float ldf(const void* p, int64_t i) {
  if constexpr (sizeof(T) == 2)
    return __bfloat162float(reinterpret_cast<const __nv_bfloat16*>(p)[i]);
  else
    return reinterpret_cast<const float*>(p)[i];
}

struct SimtArgs {
  int M, N, K;
  const void* A;
  int64_t lda, a_s1, a_s2;
  int ta;
  const void* B;
  int64_t ldb, b_s1, b_s2;
  int tb;
  void* C;
  int c_bf16;
  int64_t ldc, c_s1, c_s2;
  int nb2;
  float alpha;
  int accumulate;
};

template <typename TA, typename TB>
__global__ void __launch_bounds__(256) gemm_simt_kernel(const SimtArgs p) {
  __shared__ float sa[16][17];
  __shared__ float sb[16][17];
  const int b1 = blockIdx.z / p.nb2, b2 = blockIdx.z % p.nb2;
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int m = blockIdx.y * 16 + ty, n = blockIdx.x * 16 + tx;
  const int64_t aoff = int64_t(b1) * p.a_s1 + int64_t(b2) * p.a_s2;
  const int64_t boff = int64_t(b1) * p.b_s1 + int64_t(b2) * p.b_s2;
  float acc = 0.f;
  for (int k0 = 0; k0 < p.K; k0 += 16) {
    {  // A tile: rows m (ty), cols k0+tx
      const int mm = blockIdx.y * 16 + ty, kk = k0 + tx;
      float x = 0.f;
      if (mm < p.M && kk < p.K) x = ldf<TA>(p.A, aoff + (p.ta ? int64_t(kk) * p.lda + mm : int64_t(mm) * p.lda + kk));
      sa[ty][tx] = x;
    }
    {  // B tile: rows k0+ty, cols n (tx)
      const int kk = k0 + ty, nn = blockIdx.x * 16 + tx;
      float x = 0.f;
      if (kk < p.K && nn < p.N) x = ldf<TB>(p.B, boff + (p.tb ? int64_t(nn) * p.ldb + kk : int64_t(kk) * p.ldb + nn));
      sb[ty][tx] = x;
    }
    __syncthreads();
#pragma unroll
    for (int k = 0; k < 16; ++k) acc += sa[ty][k] * sb[k][tx];
    __syncthreads();
  }
  if (m < p.M && n < p.N) {
    const int64_t ci = int64_t(b1) * p.c_s1 + int64_t(b2) * p.c_s2 + int64_t(m) * p.ldc + n;
    if (p.c_bf16) {
      __nv_bfloat16* c = reinterpret_cast<__nv_bfloat16*>(p.C);
      float old = p.accumulate ? __bfloat162float(c[ci]) : 0.f;
      c[ci] = __float2bfloat16_rn(p.alpha * acc + old);
    } else {
      float* c = reinterpret_cast<float*>(p.C);
      c[ci] = p.alpha * acc + (p.accumulate ? c[ci] : 0.f);
    }
  }
}

int g_backend = 0;  // 0 auto, 1 tcgen05 only, 2 simt only

// Describe one bf16 operand as a 4-D TMA map (inner, outer, nb2, nb1).
bool operand_map(CUtensorMap* map, const void* ptr, uint64_t inner, uint64_t outer, int64_t ld, int64_t s1, int64_t s2,
                 int nb1, int nb2, uint32_t box_inner, uint32_t box_outer, int* bc1, int* bc2) {
  *bc1 = (s1 == 0 || nb1 == 1);
  *bc2 = (s2 == 0 || nb2 == 1);
  const uint64_t plane = uint64_t(ld) * 2 * outer;
  uint64_t dims[4] = {inner, outer, *bc2 ? 1u : uint64_t(nb2), *bc1 ? 1u : uint64_t(nb1)};
  uint64_t str[3] = {uint64_t(ld) * 2, *bc2 ? plane : uint64_t(s2) * 2, *bc1 ? plane : uint64_t(s1) * 2};
  uint32_t box[4] = {box_inner, box_outer, 1, 1};
  return encode_tmap(map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, ptr, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B);
}

int* split_flags(int n, cudaStream_t st) {  // library scratch: per-tile slice counters
  static int* buf = nullptr;
  static int cap = 0;
  if (n > cap) {
    if (buf) cudaFree(buf);
    cap = n < 4096 ? 4096 : n;
    if (cudaMalloc(&buf, sizeof(int) * cap) != cudaSuccess) return buf = nullptr, cap = 0, nullptr;
  }
  cudaMemsetAsync(buf, 0, sizeof(int) * n, st);
  return buf;
}

template <int BN>
int launch_tc(GemmArgs& a, int batches, cudaStream_t st) {
  using S = GemmSmem<BN>;
  static bool attr_set = false;
  if (!attr_set) {
    cudaFuncSetAttribute(gemm_tc_kernel<BN>, cudaFuncAttributeMaxDynamicSharedMemorySize, S::TOTAL);
    attr_set = true;
  }
  const int mt = (a.M + BM - 1) / BM;
  a.n_tiles = (a.N + BN - 1) / BN;
  a.mn_tiles = mt * a.n_tiles;
  a.batches = batches;
  const int tiles = a.mn_tiles * batches, sms = num_sms();
  const int kblocks = (a.K + BK - 1) / BK;
  a.splits = 1;
  // split K when the tiles leave most SMs idle and each slice keeps >= 8 k-blocks;
  // only for fp32 C, where the slices add into C in a fixed order (deterministic)
  if (!a.c_bf16 && tiles * 2 <= sms && kblocks >= 16) {
    a.splits = std::min({(sms + tiles - 1) / tiles, kblocks / 8, 8});
    if (a.splits > 1 && !(a.flags = split_flags(tiles, st))) a.splits = 1;
  }
  const int items = tiles * a.splits;
  gemm_tc_kernel<BN><<<std::min(items, sms), 192, S::TOTAL, st>>>(a);
  return check_launch("gemm_tc_kernel");
}

int gemm_tc(int M, int N, int K, const void* A, int64_t lda, int ta, int64_t a_s1, int64_t a_s2, const void* B,
            int64_t ldb, int tb, int64_t b_s1, int64_t b_s2, void* C, int c_dtype, int64_t ldc, int64_t c_s1,
            int64_t c_s2, int nb1, int nb2, float alpha, int accumulate, cudaStream_t st) {
  if (!aligned16(A) || !aligned16(B) || !stride_ok(lda * 2) || !stride_ok(ldb * 2) || !stride_ok(a_s1 * 2) ||
      !stride_ok(a_s2 * 2) || !stride_ok(b_s1 * 2) || !stride_ok(b_s2 * 2))
    return fail(RSA_ERR_UNSUPPORTED, "gemm: operands not 16-byte aligned for TMA");
  if (int64_t(nb1) * nb2 * ((int64_t(M) + 127) / 128) * ((int64_t(N) + 63) / 64) > (int64_t(1) << 30))
    return fail(RSA_ERR_UNSUPPORTED, "gemm: too many tiles");
  GemmArgs a{};
  const int BN = N <= 64 ? 64 : (N <= 128 ? 128 : 256);
  a.M = M, a.N = N, a.K = K;
  a.a_mn = ta ? 1 : 0;  // A stored K x M  => M contiguous
  a.b_mn = tb ? 0 : 1;  // B stored K x N  => N contiguous
  a.nb2 = nb2;
  bool ok;
  if (!a.a_mn)
    ok = operand_map(&a.ta, A, K, M, lda, a_s1, a_s2, nb1, nb2, 64, BM, &a.a_bc1, &a.a_bc2);
  else
    ok = operand_map(&a.ta, A, M, K, lda, a_s1, a_s2, nb1, nb2, 64, 64, &a.a_bc1, &a.a_bc2);
  if (!ok) return RSA_ERR_UNSUPPORTED;
  if (!a.b_mn)
    ok = operand_map(&a.tb, B, K, N, ldb, b_s1, b_s2, nb1, nb2, 64, BN, &a.b_bc1, &a.b_bc2);
  else
    ok = operand_map(&a.tb, B, N, K, ldb, b_s1, b_s2, nb1, nb2, 64, 64, &a.b_bc1, &a.b_bc2);
  if (!ok) return RSA_ERR_UNSUPPORTED;
  a.C = C;
  a.c_bf16 = c_dtype == RSA_BF16;
  const int esz = a.c_bf16 ? 2 : 4;
  a.vec_ok = aligned16(C) && (ldc * esz) % 16 == 0 && (c_s1 * esz) % 16 == 0 && (c_s2 * esz) % 16 == 0;
  a.ldc = ldc, a.c_s1 = c_s1, a.c_s2 = c_s2;
  a.alpha = alpha;
  a.accumulate = accumulate;
  const int batches = nb1 * nb2;
  if (BN == 64) return launch_tc<64>(a, batches, st);
  if (BN == 128) return launch_tc<128>(a, batches, st);
  return launch_tc<256>(a, batches, st);
}

int gemm_simt(int M, int N, int K, const void* A, int a_dtype, int64_t lda, int ta, int64_t a_s1, int64_t a_s2,
              const void* B, int b_dtype, int64_t ldb, int tb, int64_t b_s1, int64_t b_s2, void* C, int c_dtype,
              int64_t ldc, int64_t c_s1, int64_t c_s2, int nb1, int nb2, float alpha, int accumulate,
              cudaStream_t st) {
  if (int64_t(nb1) * nb2 * ((int64_t(M) + 127) / 128) * ((int64_t(N) + 63) / 64) > (int64_t(1) << 30))
    return fail(RSA_ERR_UNSUPPORTED, "gemm: too many tiles");
  SimtArgs p{M, N, K, A, lda, a_s1, a_s2, ta, B, ldb, b_s1, b_s2, tb, C, c_dtype == RSA_BF16, ldc, c_s1, c_s2,
             nb2, alpha, accumulate};
  dim3 grid((N + 15) / 16, (M + 15) / 16, nb1 * nb2);
  const bool abf = a_dtype == RSA_BF16, bbf = b_dtype == RSA_BF16;
  if (abf && bbf)
    gemm_simt_kernel<__nv_bfloat16, __nv_bfloat16><<<grid, 256, 0, st>>>(p);
  else if (abf)
    gemm_simt_kernel<__nv_bfloat16, float><<<grid, 256, 0, st>>>(p);
  else if (bbf)
    gemm_simt_kernel<float, __nv_bfloat16><<<grid, 256, 0, st>>>(p);
  else
    gemm_simt_kernel<float, float><<<grid, 256, 0, st>>>(p);
  return check_launch("gemm_simt_kernel");
}

}  // namespace
}  // namespace rsa

extern "C" {

int rsa_gemm_set_backend(int backend) {
  if (backend < 0 || backend > 2) return rsa::fail(RSA_ERR_INVALID, "backend must be 0, 1 or 2");
  rsa::g_backend = backend;
  return RSA_OK;
}

int rsa_gemm(int M, int N, int K, const void* A, int a_dtype, int64_t lda, int trans_a, int64_t a_s1, int64_t a_s2,
             const void* B, int b_dtype, int64_t ldb, int trans_b, int64_t b_s1, int64_t b_s2, void* C, int c_dtype,
             int64_t ldc, int64_t c_s1, int64_t c_s2, int nb1, int nb2, float alpha, int accumulate, void* stream) {
  using namespace rsa;
  if (M < 0 || N < 0 || K < 0 || nb1 < 1 || nb2 < 1) return fail(RSA_ERR_INVALID, "gemm: bad sizes");
  if (M == 0 || N == 0) return RSA_OK;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  if (K == 0) {
    // Empty contraction: C = 0 (or unchanged when accumulating).
    if (accumulate) return RSA_OK;
    const int esz = c_dtype == RSA_BF16 ? 2 : 4;
    for (int i1 = 0; i1 < nb1; ++i1)
      for (int i2 = 0; i2 < nb2; ++i2) {
        char* base = reinterpret_cast<char*>(C) + (int64_t(i1) * c_s1 + int64_t(i2) * c_s2) * esz;
        if (cudaMemset2DAsync(base, ldc * esz, 0, size_t(N) * esz, M, st) != cudaSuccess)
          return check_launch("gemm zero-fill");
      }
    return RSA_OK;
  }
  const bool tc_dtypes = a_dtype == RSA_BF16 && b_dtype == RSA_BF16;
  if (g_backend != 2 && tc_dtypes) {
    int r = gemm_tc(M, N, K, A, lda, trans_a, a_s1, a_s2, B, ldb, trans_b, b_s1, b_s2, C, c_dtype, ldc, c_s1, c_s2,
                    nb1, nb2, alpha, accumulate, st);
    if (r != RSA_ERR_UNSUPPORTED || g_backend == 1) return r;
  } else if (g_backend == 1) {
    return fail(RSA_ERR_UNSUPPORTED, "gemm: tcgen05 path needs bf16 operands");
  }
  return gemm_simt(M, N, K, A, a_dtype, lda, trans_a, a_s1, a_s2, B, b_dtype, ldb, trans_b, b_s1, b_s2, C, c_dtype,
                   ldc, c_s1, c_s2, nb1, nb2, alpha, accumulate, st);
}

}  // extern "C"

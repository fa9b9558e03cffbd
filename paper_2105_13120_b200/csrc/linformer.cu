// Linformer sequence-sharded K/V projection for sm_100a (ringseq/sparse_attention.py:111-123):
//   K' = sum_d E_d K_d,   V' = sum_d F_d V_d         (E_d, F_d: rank d's (Kp x c) column blocks)
// for every head at once.  The sum over the resident ranks is one contraction over the whole
// length L (ranks in ascending order, as the reference's ring-accumulate adds them when every
// rank is resident), so no per-rank partials reach HBM.
//
// Tile: 128 rows of E (M) x FOUR heads' 64 dimensions (N = 256) per tcgen05.mma, so each E
// tile staged in shared memory feeds four heads (the generic batched rsa_gemm re-reads E_d
// from L2 for every head).  The contraction over L is split over enough CTAs to fill the
// machine; each split's fp32 128 x 256 result is added into the fp32 output in L2 by TMA
// reduce-add (cp.reduce.async.bulk.tensor), and a small kernel casts to bf16 at the end.
//
// Warp roles (6 warps): 0 TMA producer, 1 MMA issuer (owns TMEM: two 256-column
// accumulators), 2..5 epilogue (warp w reads TMEM lanes 32 * (w % 4), stages 32 x 32 fp32
// chunks, issues the reduce).  Work item = (projection, 128-row block of Kp, group of four
// heads, split of L).
#include <algorithm>

#include "fused_common.cuh"

namespace rsa {
namespace {

constexpr int LP_HEADS = 4;                         // heads per N tile
constexpr int LP_KB = 64;                           // L positions per stage
constexpr int LP_ST = 4;                            // stages
constexpr uint32_t LP_A = TR * LP_KB * 2;           // 16 KB: 128 rows of E x 64 positions
constexpr uint32_t LP_BH = LP_KB * HD * 2;          // 8 KB: one head's 64 positions x 64 dims
constexpr uint32_t LP_STAGE = LP_A + LP_HEADS * LP_BH;  // 48 KB
constexpr uint32_t LP_OFF_STG = LP_ST * LP_STAGE;       // epilogue staging: [warp][2][32 rows][128 B]
constexpr uint32_t LP_OFF_BAR = LP_OFF_STG + 4 * 2 * 4096;
constexpr uint32_t LP_SMEM = LP_OFF_BAR + 256 + 1024;
constexpr int LP_THREADS = 32 * 6;
static_assert(LP_SMEM <= 232448, "linformer projection smem over the sm_100 per-CTA limit");

struct LpArgs {
  CUtensorMap ta[2], tb[2], to[2];  // per projection: E / F (Kp x L), K / V (heads), fp32 output
  int kp, BZ, Z, B;                 // Kp, heads, heads per batch, batch
  int c, n_org;                     // positions per origin chunk, resident origins
  int splits, stages_total, stages_per_split;
  int items;
};

__global__ void __launch_bounds__(LP_THREADS, 1) linformer_project_kernel(const __grid_constant__ LpArgs p) {
  uint8_t* smem = smem_base();
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + LP_OFF_BAR);
  uint64_t *full = bar, *empty = bar + LP_ST, *acc_full = empty + LP_ST, *acc_empty = acc_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);
  const uint32_t warp = warp_id(), lane = lane_id();
  const int mblocks = p.kp / TR, hgroups = p.BZ / LP_HEADS;
  const int per_origin = p.c / LP_KB;

  if (warp == 1) tmem_alloc(tmem_slot, 512);
  if (threadIdx.x == 0) {
    for (int s = 0; s < LP_ST; ++s) mbar_init(&full[s], 1), mbar_init(&empty[s], 1);
    for (int s = 0; s < 2; ++s) mbar_init(&acc_full[s], 1), mbar_init(&acc_empty[s], 4);
    fence_barrier_init();
    for (int j = 0; j < 2; ++j) tma_prefetch(&p.ta[j]), tma_prefetch(&p.tb[j]), tma_prefetch(&p.to[j]);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base(tmem_slot);

  // item -> (projection j, Kp block mb, head group hg, split ks); stage range [s0, s1)
  auto decode = [&](int item, int& j, int& mb, int& hg, int& s0, int& s1) {
    const int ks = item % p.splits;
    int rest = item / p.splits;
    hg = rest % hgroups, rest /= hgroups;
    mb = rest % mblocks, j = rest / mblocks;
    s0 = ks * p.stages_per_split;
    s1 = min(s0 + p.stages_per_split, p.stages_total);
  };

  if (warp == 0) {
    if (lane == 0) {
      Pos lq;
      for (int item = blockIdx.x; item < p.items; item += gridDim.x) {
        int j, mb, hg, s0, s1;
        decode(item, j, mb, hg, s0, s1);
        for (int st = s0; st < s1; ++st) {
          const uint32_t s = lq.slot(LP_ST);
          mbar_wait(&empty[s], lq.phase(LP_ST) ^ 1);
          mbar_arrive_expect_tx(&full[s], LP_STAGE);
          uint8_t* sa = smem + s * LP_STAGE;
          const int d = st / per_origin, row = (st % per_origin) * LP_KB;
          tma_load_2d(sa, &p.ta[j], &full[s], d * p.c + row, mb * TR);
#pragma unroll
          for (int h = 0; h < LP_HEADS; ++h) {
            const int bz = hg * LP_HEADS + h;
            tma_load_4d(sa + LP_A + h * LP_BH, &p.tb[j], &full[s], 0, row, bz % p.Z, d * p.B + bz / p.Z);
          }
          ++lq.i;
        }
      }
    }
  } else if (warp == 1) {
    // K-major A (E rows, positions contiguous), MN-major B (per head: positions x dims, dims
    // contiguous; the four heads' 64-dim blocks 8 KB apart): M = 128, N = 256
    const uint32_t idesc = idesc_bf16_f32(TR, LP_HEADS * HD, 0, 1);
    Pos lq;
    uint32_t it = 0;
    for (int item = blockIdx.x; item < p.items; item += gridDim.x, ++it) {
      int j, mb, hg, s0, s1;
      decode(item, j, mb, hg, s0, s1);
      const uint32_t ab = it & 1;
      mbar_wait(&acc_empty[ab], ((it >> 1) & 1) ^ 1);
      tc_fence_after();
      for (int st = s0; st < s1; ++st) {
        const uint32_t s = lq.slot(LP_ST);
        mbar_wait(&full[s], lq.phase(LP_ST));
        tc_fence_after();
        const uint32_t sa = smem_u32(smem + s * LP_STAGE), sb = sa + LP_A;
#pragma unroll
        for (int k = 0; k < LP_KB / 16; ++k)
          umma_bf16_ws(tmem + ab * 256, smem_desc_sw128(sa + k * 32, 0, 1024),
                       smem_desc_sw128(sb + k * 2048, LP_BH, 1024), idesc, (st > s0) || (k > 0));
        umma_commit_ws(&empty[s]);
        ++lq.i;
      }
      umma_commit_ws(&acc_full[ab]);
    }
  } else {
    // epilogue: warp w owns TMEM lanes 32 * (w % 4) = rows of the Kp block; 8 chunks of 32
    // columns (head h = chunk / 2, dims (chunk % 2) * 32 ..), each staged (SWIZZLE_128B) and
    // reduce-added into the fp32 output by TMA
    const uint32_t quad = warp & 3;
    const uint32_t lane_base = (quad * 32u) << 16;
    uint8_t* stg = smem + LP_OFF_STG + (warp - 2) * 8192;
    uint32_t it = 0;
    for (int item = blockIdx.x; item < p.items; item += gridDim.x, ++it) {
      int j, mb, hg, s0, s1;
      decode(item, j, mb, hg, s0, s1);
      const uint32_t ab = it & 1;
      mbar_wait(&acc_full[ab], (it >> 1) & 1);
      tc_fence_after();
#pragma unroll 1
      for (int ch = 0; ch < 2 * LP_HEADS; ++ch) {
        float v[32];
        __syncwarp();
        tmem_ld32(tmem + lane_base + ab * 256 + ch * 32, v);
        tmem_ld_wait();
        if (ch == 2 * LP_HEADS - 1) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&acc_empty[ab]);
        }
        uint8_t* buf = stg + (ch & 1) * 4096;
        if (lane == 0) tma_store_wait_read<1>();  // the reduce that used this buffer has read it
        __syncwarp();
        const uint32_t row = smem_u32(buf) + lane * 128;
#pragma unroll
        for (int q = 0; q < 8; ++q)
          st_shared_v4(row + ((q ^ (lane & 7)) << 4), __float_as_uint(v[4 * q]), __float_as_uint(v[4 * q + 1]),
                       __float_as_uint(v[4 * q + 2]), __float_as_uint(v[4 * q + 3]));
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          const int bz = hg * LP_HEADS + ch / 2;
          tma_reduce_add_4d(&p.to[j], buf, (ch & 1) * 32, mb * TR + int(quad) * 32, bz % p.Z, bz / p.Z);
          tma_store_commit();
        }
      }
    }
    if (lane == 0) tma_store_wait_all<0>();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, 512);
}

// ---------------------------------------------------------------- projection gradients
//
// dE[:, d-block] = sum_{b,z} dK'_{bz} K_{d,bz}^T (and dF from dV', V): for every rank d's
// c positions, a (Kp x c) block summed over the B*Z heads -- ringseq/sparse_attention.py's
// projections differentiated.  Tile: 128 rows of Kp (M) x 256
// positions (N); the contraction walks the heads, 64 dimensions each: A = dK'_{bz} rows
// (dims contiguous, K-major), B = K_{d,bz} positions (dims contiguous, K-major), so neither
// operand is transposed or copied.  The fp32 128 x 256 result leaves by TMA store.
constexpr int LG_N = 256;                           // positions per tile
constexpr uint32_t LG_A = TR * HD * 2;              // 16 KB
constexpr uint32_t LG_B = LG_N * HD * 2;            // 32 KB
constexpr uint32_t LG_STAGE = LG_A + LG_B;          // 48 KB (= LP_STAGE: same layout of stages)

struct LgArgs {
  CUtensorMap ta[2], tb[2], to[2];  // dK' / dV' ([b][z][Kp][64]), K / V (heads), fp32 dE / dF (Kp x L)
  int kp, BZ, Z, B, c, n_org;
  int nblocks;                      // 256-position blocks per origin chunk
  int items;
};

__global__ void __launch_bounds__(LP_THREADS, 1) linformer_grad_kernel(const __grid_constant__ LgArgs p) {
  uint8_t* smem = smem_base();
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + LP_OFF_BAR);
  uint64_t *full = bar, *empty = bar + LP_ST, *acc_full = empty + LP_ST, *acc_empty = acc_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);
  const uint32_t warp = warp_id(), lane = lane_id();
  const int mblocks = p.kp / TR;

  if (warp == 1) tmem_alloc(tmem_slot, 512);
  if (threadIdx.x == 0) {
    for (int s = 0; s < LP_ST; ++s) mbar_init(&full[s], 1), mbar_init(&empty[s], 1);
    for (int s = 0; s < 2; ++s) mbar_init(&acc_full[s], 1), mbar_init(&acc_empty[s], 4);
    fence_barrier_init();
    for (int j = 0; j < 2; ++j) tma_prefetch(&p.ta[j]), tma_prefetch(&p.tb[j]), tma_prefetch(&p.to[j]);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base(tmem_slot);

  // item -> (projection j, Kp block mb, origin d, position block nb)
  auto decode = [&](int item, int& j, int& mb, int& d, int& nb) {
    nb = item % p.nblocks;
    int rest = item / p.nblocks;
    d = rest % p.n_org, rest /= p.n_org;
    mb = rest % mblocks, j = rest / mblocks;
  };

  if (warp == 0) {
    if (lane == 0) {
      Pos lq;
      for (int item = blockIdx.x; item < p.items; item += gridDim.x) {
        int j, mb, d, nb;
        decode(item, j, mb, d, nb);
        for (int bz = 0; bz < p.BZ; ++bz) {
          const uint32_t s = lq.slot(LP_ST);
          mbar_wait(&empty[s], lq.phase(LP_ST) ^ 1);
          mbar_arrive_expect_tx(&full[s], LG_STAGE);
          uint8_t* sa = smem + s * LP_STAGE;
          tma_load_4d(sa, &p.ta[j], &full[s], 0, mb * TR, bz % p.Z, bz / p.Z);
          tma_load_4d(sa + LG_A, &p.tb[j], &full[s], 0, nb * LG_N, bz % p.Z, d * p.B + bz / p.Z);
          ++lq.i;
        }
      }
    }
  } else if (warp == 1) {
    const uint32_t idesc = idesc_bf16_f32(TR, LG_N, 0, 0);  // both K-major (head dims contiguous)
    Pos lq;
    uint32_t it = 0;
    for (int item = blockIdx.x; item < p.items; item += gridDim.x, ++it) {
      const uint32_t ab = it & 1;
      mbar_wait(&acc_empty[ab], ((it >> 1) & 1) ^ 1);
      tc_fence_after();
      for (int bz = 0; bz < p.BZ; ++bz) {
        const uint32_t s = lq.slot(LP_ST);
        mbar_wait(&full[s], lq.phase(LP_ST));
        tc_fence_after();
        const uint32_t sa = smem_u32(smem + s * LP_STAGE), sb = sa + LG_A;
#pragma unroll
        for (int k = 0; k < HD / 16; ++k)
          umma_bf16_ws(tmem + ab * 256, smem_desc_sw128(sa + k * 32, 0, 1024), smem_desc_sw128(sb + k * 32, 0, 1024),
                       idesc, (bz > 0) || (k > 0));
        umma_commit_ws(&empty[s]);
        ++lq.i;
      }
      umma_commit_ws(&acc_full[ab]);
    }
  } else {
    const uint32_t quad = warp & 3;
    const uint32_t lane_base = (quad * 32u) << 16;
    uint8_t* stg = smem + LP_OFF_STG + (warp - 2) * 8192;
    uint32_t it = 0;
    for (int item = blockIdx.x; item < p.items; item += gridDim.x, ++it) {
      int j, mb, d, nb;
      decode(item, j, mb, d, nb);
      const uint32_t ab = it & 1;
      mbar_wait(&acc_full[ab], (it >> 1) & 1);
      tc_fence_after();
#pragma unroll 1
      for (int ch = 0; ch < LG_N / 32; ++ch) {
        float v[32];
        __syncwarp();
        tmem_ld32(tmem + lane_base + ab * 256 + ch * 32, v);
        tmem_ld_wait();
        if (ch == LG_N / 32 - 1) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&acc_empty[ab]);
        }
        uint8_t* buf = stg + (ch & 1) * 4096;
        if (lane == 0) tma_store_wait_read<1>();
        __syncwarp();
        const uint32_t row = smem_u32(buf) + lane * 128;
#pragma unroll
        for (int q = 0; q < 8; ++q)
          st_shared_v4(row + ((q ^ (lane & 7)) << 4), __float_as_uint(v[4 * q]), __float_as_uint(v[4 * q + 1]),
                       __float_as_uint(v[4 * q + 2]), __float_as_uint(v[4 * q + 3]));
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          asm volatile(
              "cp.async.bulk.tensor.2d.global.shared::cta.tile.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                  reinterpret_cast<uint64_t>(&p.to[j])),
              "r"(smem_u32(buf)), "r"(d * p.c + nb * LG_N + ch * 32), "r"(mb * TR + int(quad) * 32)
              : "memory");
          tma_store_commit();
        }
      }
    }
    if (lane == 0) tma_store_wait_all<0>();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, 512);
}

// ------------------------------------------------------------ the projections' transposes
//
// dK_d = E_d^T dK', dV_d = F_d^T dV' (the Linformer backward's gradients of the keys and
// values) for every rank and head: tile = 128 positions (M) x four
// heads' 64 dimensions (N = 256), contraction over Kp in 64-row stages.  A = E read as
// MN-major (positions contiguous), B = the four heads' dK' blocks (dims contiguous), so the
// E tile staged for a position block feeds four heads; bf16 rows leave straight from TMEM
// (each thread one row's 32 dimensions per store pair).
struct LbArgs {
  CUtensorMap ta[2], tb[2];  // E / F (Kp x L), dK' / dV' ([b][z][Kp][64])
  OutView out[2];            // dK / dV: [origin][b][z][position][64] bf16
  int kp, BZ, Z, B, c, n_org, org_lo;
  int pblocks, items;
};

__global__ void __launch_bounds__(LP_THREADS, 1) linformer_back_kernel(const __grid_constant__ LbArgs p) {
  uint8_t* smem = smem_base();
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + LP_OFF_BAR);
  uint64_t *full = bar, *empty = bar + LP_ST, *acc_full = empty + LP_ST, *acc_empty = acc_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);
  const uint32_t warp = warp_id(), lane = lane_id();
  const int hgroups = p.BZ / LP_HEADS, kstages = p.kp / LP_KB;

  if (warp == 1) tmem_alloc(tmem_slot, 512);
  if (threadIdx.x == 0) {
    for (int s = 0; s < LP_ST; ++s) mbar_init(&full[s], 1), mbar_init(&empty[s], 1);
    for (int s = 0; s < 2; ++s) mbar_init(&acc_full[s], 1), mbar_init(&acc_empty[s], 4);
    fence_barrier_init();
    for (int j = 0; j < 2; ++j) tma_prefetch(&p.ta[j]), tma_prefetch(&p.tb[j]);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base(tmem_slot);

  // item -> (projection j, origin d, position block pb, head group hg): head groups fastest,
  // so consecutive items of a CTA reuse the E tile from L2
  auto decode = [&](int item, int& j, int& d, int& pb, int& hg) {
    hg = item % hgroups;
    int rest = item / hgroups;
    pb = rest % p.pblocks, rest /= p.pblocks;
    d = rest % p.n_org, j = rest / p.n_org;
  };

  if (warp == 0) {
    if (lane == 0) {
      Pos lq;
      for (int item = blockIdx.x; item < p.items; item += gridDim.x) {
        int j, d, pb, hg;
        decode(item, j, d, pb, hg);
        for (int ks = 0; ks < kstages; ++ks) {
          const uint32_t s = lq.slot(LP_ST);
          mbar_wait(&empty[s], lq.phase(LP_ST) ^ 1);
          mbar_arrive_expect_tx(&full[s], LP_STAGE);
          uint8_t* sa = smem + s * LP_STAGE;
          const int col = (p.org_lo + d) * p.c + pb * TR;
          tma_load_2d(sa, &p.ta[j], &full[s], col, ks * LP_KB);                  // positions col .. +63
          tma_load_2d(sa + LP_A / 2, &p.ta[j], &full[s], col + 64, ks * LP_KB);  // positions col + 64 .. +127
#pragma unroll
          for (int h = 0; h < LP_HEADS; ++h) {
            const int bz = hg * LP_HEADS + h;
            tma_load_4d(sa + LP_A + h * LP_BH, &p.tb[j], &full[s], 0, ks * LP_KB, bz % p.Z, bz / p.Z);
          }
          ++lq.i;
        }
      }
    }
  } else if (warp == 1) {
    // A: E^T (positions contiguous: MN-major, two 64-position atoms 8 KB apart); B: dK' blocks
    // (dims contiguous: MN-major, four 64-dim atoms 8 KB apart); 16 Kp rows (2 KB) per k step
    const uint32_t idesc = idesc_bf16_f32(TR, LP_HEADS * HD, 1, 1);
    Pos lq;
    uint32_t it = 0;
    for (int item = blockIdx.x; item < p.items; item += gridDim.x, ++it) {
      const uint32_t ab = it & 1;
      mbar_wait(&acc_empty[ab], ((it >> 1) & 1) ^ 1);
      tc_fence_after();
      for (int ks = 0; ks < kstages; ++ks) {
        const uint32_t s = lq.slot(LP_ST);
        mbar_wait(&full[s], lq.phase(LP_ST));
        tc_fence_after();
        const uint32_t sa = smem_u32(smem + s * LP_STAGE), sb = sa + LP_A;
#pragma unroll
        for (int k = 0; k < LP_KB / 16; ++k)
          umma_bf16_ws(tmem + ab * 256, smem_desc_sw128(sa + k * 2048, LP_A / 2, 1024),
                       smem_desc_sw128(sb + k * 2048, LP_BH, 1024), idesc, (ks > 0) || (k > 0));
        umma_commit_ws(&empty[s]);
        ++lq.i;
      }
      umma_commit_ws(&acc_full[ab]);
    }
  } else {
    const uint32_t quad = warp & 3;
    const uint32_t lane_base = (quad * 32u) << 16;
    uint32_t it = 0;
    for (int item = blockIdx.x; item < p.items; item += gridDim.x, ++it) {
      int j, d, pb, hg;
      decode(item, j, d, pb, hg);
      const uint32_t ab = it & 1;
      const int pos = pb * TR + int(quad) * 32 + int(lane);
      mbar_wait(&acc_full[ab], (it >> 1) & 1);
      tc_fence_after();
#pragma unroll 1
      for (int ch = 0; ch < 2 * LP_HEADS; ++ch) {
        float v[32];
        __syncwarp();
        tmem_ld32(tmem + lane_base + ab * 256 + ch * 32, v);
        tmem_ld_wait();
        if (ch == 2 * LP_HEADS - 1) {
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&acc_empty[ab]);
        }
        if (pos < p.c) {
          const int bz = hg * LP_HEADS + ch / 2;
          const OutView none{nullptr, 0, 0, 0, 0};
          store_row32(none, p.out[j], 0, d, bz / p.Z, bz % p.Z, pos, (ch & 1) * 32, v);
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, 512);
}

__global__ void cast_bf16_kernel(const float4* __restrict__ x, uint2* __restrict__ y, int64_t n4) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n4; i += int64_t(gridDim.x) * blockDim.x) {
    const float4 v = x[i];
    y[i] = make_uint2(pack_bf16(v.x, v.y), pack_bf16(v.z, v.w));
  }
}

}  // namespace
}  // namespace rsa

extern "C" {

int rsa_linformer_project(const rsa_geom* g, int proj_dim, const void* e, const void* f, int64_t ld_proj, rsa_view k,
                          rsa_view v, float* k_acc, float* v_acc, void* k_low, void* v_low, void* stream) {
  using namespace rsa;
  if (!g || g->head_dim != HD || g->chunk % LP_KB || proj_dim % TR || (g->batch * g->heads) % LP_HEADS ||
      g->n_org < 1 || g->org_lo < 0 || !e || !f || !k_acc || !v_acc || ld_proj < int64_t(g->org_lo + g->n_org) * g->chunk)
    return fail(RSA_ERR_INVALID, "rsa_linformer_project: unsupported geometry (A = 64, chunk %% 64, Kp %% 128, "
                                 "B*Z %% 4)");
  if (!aligned16(e) || !aligned16(f) || (ld_proj * 2) % 16 || !aligned16(k_acc) || !aligned16(v_acc))
    return fail(RSA_ERR_UNSUPPORTED, "rsa_linformer_project: projections / outputs not 16-byte aligned");
  LpArgs a{};
  const void* proj[2] = {e, f};
  const rsa_view x[2] = {k, v};
  float* acc[2] = {k_acc, v_acc};
  for (int j = 0; j < 2; ++j) {
    // E / F: (Kp x L) row-major, columns from org_lo * c on; 64-position x 128-row boxes
    const char* base = static_cast<const char*>(proj[j]) + int64_t(g->org_lo) * g->chunk * 2;
    uint64_t dims[2] = {uint64_t(g->n_org) * g->chunk, uint64_t(proj_dim)};
    uint64_t str[1] = {uint64_t(ld_proj) * 2};
    uint32_t box[2] = {LP_KB, TR};
    if (!encode_tmap(&a.ta[j], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, base, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B))
      return RSA_ERR_UNSUPPORTED;
    // K / V: [origin][b][z][row][a]; 64-row boxes (head_map's layout checks, then the box)
    if (!head_map(&a.tb[j], x[j], g, g->n_org)) return RSA_ERR_UNSUPPORTED;
    {
      uint64_t d4[4] = {uint64_t(HD), uint64_t(g->chunk), uint64_t(g->heads), uint64_t(g->batch) * g->n_org};
      const int64_t sb = (g->batch == 1 && g->n_org > 1) ? x[j].s_rank : x[j].s_b;
      uint64_t s4[3] = {uint64_t(x[j].s_row) * 2, uint64_t(x[j].s_z) * 2, uint64_t(sb) * 2};
      uint32_t b4[4] = {HD, LP_KB, 1, 1};
      if (!encode_tmap(&a.tb[j], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, x[j].ptr, d4, s4, b4, CU_TENSOR_MAP_SWIZZLE_128B))
        return RSA_ERR_UNSUPPORTED;
    }
    // fp32 output [b][z][Kp][a] (contiguous): 32-dim x 32-row boxes, SWIZZLE_128B
    uint64_t od[4] = {uint64_t(HD), uint64_t(proj_dim), uint64_t(g->heads), uint64_t(g->batch)};
    uint64_t os[3] = {uint64_t(HD) * 4, uint64_t(proj_dim) * HD * 4, uint64_t(g->heads) * proj_dim * HD * 4};
    uint32_t ob[4] = {32, 32, 1, 1};
    if (!encode_tmap(&a.to[j], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, acc[j], od, os, ob, CU_TENSOR_MAP_SWIZZLE_128B))
      return RSA_ERR_UNSUPPORTED;
  }
  a.kp = proj_dim, a.BZ = g->batch * g->heads, a.Z = g->heads, a.B = g->batch;
  a.c = g->chunk, a.n_org = g->n_org;
  a.stages_total = g->n_org * g->chunk / LP_KB;
  const int tiles = 2 * (proj_dim / TR) * (a.BZ / LP_HEADS);
  const int sms = num_sms();
  a.splits = std::max(1, std::min(sms / std::max(1, tiles), a.stages_total / 8));  // >= 8 stages per split
  a.stages_per_split = (a.stages_total + a.splits - 1) / a.splits;
  a.splits = (a.stages_total + a.stages_per_split - 1) / a.stages_per_split;
  a.items = tiles * a.splits;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const int64_t n_out = int64_t(a.BZ) * proj_dim * HD;
  if (cudaMemsetAsync(k_acc, 0, size_t(n_out) * 4, st) != cudaSuccess ||
      cudaMemsetAsync(v_acc, 0, size_t(n_out) * 4, st) != cudaSuccess)
    return check_launch("rsa_linformer_project: zero-fill");
  if (int rc = launch(linformer_project_kernel, a.items, LP_SMEM, a, stream, "linformer_project_kernel", LP_THREADS))
    return rc;
  void* lows[2] = {k_low, v_low};
  for (int j = 0; j < 2; ++j) {
    if (!lows[j]) continue;
    const int64_t n4 = n_out / 4;
    cast_bf16_kernel<<<int(std::min<int64_t>((n4 + 255) / 256, int64_t(sms) * 8)), 256, 0, st>>>(
        reinterpret_cast<const float4*>(acc[j]), static_cast<uint2*>(lows[j]), n4);
    if (int rc = check_launch("cast_bf16_kernel")) return rc;
  }
  return RSA_OK;
}

int rsa_linformer_proj_grad(const rsa_geom* g, int proj_dim, const void* dk_low, const void* dv_low, rsa_view k,
                            rsa_view v, float* grad_e, float* grad_f, int64_t ld_grad, void* stream) {
  using namespace rsa;
  if (!g || g->head_dim != HD || g->chunk % LG_N || proj_dim % TR || g->n_org < 1 || g->org_lo < 0 || !dk_low ||
      !dv_low || !grad_e || !grad_f || ld_grad < int64_t(g->org_lo + g->n_org) * g->chunk)
    return fail(RSA_ERR_INVALID, "rsa_linformer_proj_grad: unsupported geometry (A = 64, chunk %% 256, Kp %% 128)");
  if (!aligned16(dk_low) || !aligned16(dv_low) || !aligned16(grad_e) || !aligned16(grad_f) || (ld_grad * 4) % 16)
    return fail(RSA_ERR_UNSUPPORTED, "rsa_linformer_proj_grad: buffers not 16-byte aligned");
  LgArgs a{};
  const void* low[2] = {dk_low, dv_low};
  const rsa_view x[2] = {k, v};
  float* out[2] = {grad_e, grad_f};
  for (int j = 0; j < 2; ++j) {
    // dK' / dV': [b][z][Kp][64] bf16 contiguous; 64-dim x 128-row boxes
    uint64_t ad[4] = {uint64_t(HD), uint64_t(proj_dim), uint64_t(g->heads), uint64_t(g->batch)};
    uint64_t as[3] = {uint64_t(HD) * 2, uint64_t(proj_dim) * HD * 2, uint64_t(g->heads) * proj_dim * HD * 2};
    uint32_t ab[4] = {HD, TR, 1, 1};
    if (!encode_tmap(&a.ta[j], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, low[j], ad, as, ab, CU_TENSOR_MAP_SWIZZLE_128B))
      return RSA_ERR_UNSUPPORTED;
    // K / V: [origin][b][z][row][a]; 256-row boxes
    if (!head_map(&a.tb[j], x[j], g, g->n_org)) return RSA_ERR_UNSUPPORTED;
    {
      uint64_t d4[4] = {uint64_t(HD), uint64_t(g->chunk), uint64_t(g->heads), uint64_t(g->batch) * g->n_org};
      const int64_t sb = (g->batch == 1 && g->n_org > 1) ? x[j].s_rank : x[j].s_b;
      uint64_t s4[3] = {uint64_t(x[j].s_row) * 2, uint64_t(x[j].s_z) * 2, uint64_t(sb) * 2};
      uint32_t b4[4] = {HD, LG_N, 1, 1};
      if (!encode_tmap(&a.tb[j], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, x[j].ptr, d4, s4, b4, CU_TENSOR_MAP_SWIZZLE_128B))
        return RSA_ERR_UNSUPPORTED;
    }
    // fp32 dE / dF (Kp x L), columns from org_lo * c on: 32-column x 32-row boxes
    float* base = out[j] + int64_t(g->org_lo) * g->chunk;
    uint64_t od[2] = {uint64_t(g->n_org) * g->chunk, uint64_t(proj_dim)};
    uint64_t os[1] = {uint64_t(ld_grad) * 4};
    uint32_t ob[2] = {32, 32};
    if (!encode_tmap(&a.to[j], CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, base, od, os, ob, CU_TENSOR_MAP_SWIZZLE_128B))
      return RSA_ERR_UNSUPPORTED;
  }
  a.kp = proj_dim, a.BZ = g->batch * g->heads, a.Z = g->heads, a.B = g->batch;
  a.c = g->chunk, a.n_org = g->n_org;
  a.nblocks = g->chunk / LG_N;
  a.items = 2 * (proj_dim / TR) * g->n_org * a.nblocks;
  return launch(linformer_grad_kernel, a.items, LP_SMEM, a, stream, "linformer_grad_kernel", LP_THREADS);
}

int rsa_linformer_proj_back(const rsa_geom* g, int proj_dim, const void* e, const void* f, int64_t ld_proj,
                            const void* dk_low, const void* dv_low, rsa_view dk, rsa_view dv, void* stream) {
  using namespace rsa;
  if (!g || g->head_dim != HD || g->chunk % TR || proj_dim % LP_KB || (g->batch * g->heads) % LP_HEADS ||
      g->n_org < 1 || g->org_lo < 0 || !e || !f || !dk_low || !dv_low || !dk.ptr || !dv.ptr ||
      ld_proj < int64_t(g->org_lo + g->n_org) * g->chunk)
    return fail(RSA_ERR_INVALID, "rsa_linformer_proj_back: unsupported geometry (A = 64, chunk %% 128, Kp %% 64, "
                                 "B*Z %% 4)");
  if (!aligned16(e) || !aligned16(f) || (ld_proj * 2) % 16 || !aligned16(dk_low) || !aligned16(dv_low) ||
      !out_ok(dk, 2) || !out_ok(dv, 2))
    return fail(RSA_ERR_UNSUPPORTED, "rsa_linformer_proj_back: buffers not 16-byte aligned");
  LbArgs a{};
  const void* proj[2] = {e, f};
  const void* low[2] = {dk_low, dv_low};
  const rsa_view out[2] = {dk, dv};
  for (int j = 0; j < 2; ++j) {
    // E / F: (Kp x L) row-major; 64-position x 64-row boxes (positions contiguous)
    uint64_t dims[2] = {uint64_t(ld_proj), uint64_t(proj_dim)};
    uint64_t str[1] = {uint64_t(ld_proj) * 2};
    uint32_t box[2] = {64, LP_KB};
    if (!encode_tmap(&a.ta[j], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, proj[j], dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B))
      return RSA_ERR_UNSUPPORTED;
    // dK' / dV': [b][z][Kp][64] bf16 contiguous; 64-dim x 64-row boxes
    uint64_t bd[4] = {uint64_t(HD), uint64_t(proj_dim), uint64_t(g->heads), uint64_t(g->batch)};
    uint64_t bs[3] = {uint64_t(HD) * 2, uint64_t(proj_dim) * HD * 2, uint64_t(g->heads) * proj_dim * HD * 2};
    uint32_t bb[4] = {HD, LP_KB, 1, 1};
    if (!encode_tmap(&a.tb[j], CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, low[j], bd, bs, bb, CU_TENSOR_MAP_SWIZZLE_128B))
      return RSA_ERR_UNSUPPORTED;
    a.out[j] = to_out(out[j]);
  }
  a.kp = proj_dim, a.BZ = g->batch * g->heads, a.Z = g->heads, a.B = g->batch;
  a.c = g->chunk, a.n_org = g->n_org, a.org_lo = g->org_lo;
  a.pblocks = g->chunk / TR;
  a.items = 2 * g->n_org * a.pblocks * (a.BZ / LP_HEADS);
  return launch(linformer_back_kernel, a.items, LP_SMEM, a, stream, "linformer_back_kernel", LP_THREADS);
}

}  // extern "C"

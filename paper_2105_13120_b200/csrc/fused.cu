// Fused Ring Self-Attention kernels for sm_100a (head size A = 64).
//
// Tensor layout (all bf16 unless noted): per-head tensors are addressed as
// [rank][b][z][row][a] and probability / dS panels as [rank][b][z][row][col]
// with col = origin * c + key (ringseq/ring_attention.py:91-94: column block
// j of the panel belongs to origin j).  TMA moves 128-row x 64-column tiles
// (one 128-byte swizzle row per tile row); every tile lives in shared memory
// in the SWIZZLE_128B layout the UMMA descriptors read, and the same bytes are
// read as K-major or MN-major operands as each product needs.
//
// Each kernel is warp-specialised, 6 warps:
//   warp 0      TMA producer (one elected lane)
//   warp 1      tcgen05.mma issuer (one elected lane); owns TMEM alloc
//   warps 2..5  epilogue: warp w reads TMEM lanes 32*(w%4).. (= tile rows),
//               so every row-wise reduction is thread-local (no shuffles)
//
// rsa_fwd_stats    stage 1 (K ring): S = Q K_j^T per key tile, online row
//                  max / sum of exp2 kept in registers -> (m, l) per row.
// rsa_fwd_probs_pv stage 2 (V ring): S recomputed, P = 2^(S' - m) / l written
//                  once to the bf16 panel (TMA store) and fed from smem to a
//                  second UMMA, O += P V_j accumulating in TMEM.
// rsa_bwd_dkdv     V-ring half of the backward, one CTA per key tile of an
//                  origin: dP = dO V^T (TMEM), dS = P (dP - D) scale (smem +
//                  TMA store), dV += P^T dO and dK += dS^T Q (TMEM).
// rsa_bwd_dq       K-ring half: dQ += dS K_j.
#include "common.h"
#include "ptx.cuh"

namespace rsa {
namespace {

constexpr int HD = 64;                          // head size the fused kernels tile
constexpr int TR = 128;                         // rows per tile (UMMA M)
constexpr int TKEYS = 128;                      // keys per tile
constexpr uint32_t TILE = TR * HD * 2;          // 16 KB: 128 x 64 bf16
constexpr uint32_t PTILE = TR * TKEYS * 2;      // 32 KB: 128 x 128 bf16 (two 64-key atoms)
constexpr uint32_t ATOM = TR * 128;             // 16 KB: one 128-row x 128-byte swizzle atom column
constexpr float LOG2E = 1.4426950408889634f;
constexpr int NTHREADS = 192;

__device__ __forceinline__ void epi_bar() { asm volatile("bar.sync 1, 128;" ::: "memory"); }

// Write 32 consecutive fp32 values (key columns col0..col0+31 of row r) as
// bf16 into a [key atom][128 rows][128 B] SWIZZLE_128B tile.
__device__ __forceinline__ void st_row32_sw128(uint32_t tile_base, uint32_t r, int col0, const float* v) {
  const uint32_t atom = col0 >> 6;
  const uint32_t chunk0 = (col0 & 63) >> 3;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const uint32_t addr = tile_base + atom * ATOM + sw128_offset(r, chunk0 + q);
    st_shared_v4(addr, pack_bf16(v[8 * q], v[8 * q + 1]), pack_bf16(v[8 * q + 2], v[8 * q + 3]),
                 pack_bf16(v[8 * q + 4], v[8 * q + 5]), pack_bf16(v[8 * q + 6], v[8 * q + 7]));
  }
}

// Read 32 consecutive bf16 (columns col0..col0+31 of row r) from the same layout.
__device__ __forceinline__ void ld_row32_sw128(uint32_t tile_base, uint32_t r, int col0, float* v) {
  const uint32_t atom = col0 >> 6;
  const uint32_t chunk0 = (col0 & 63) >> 3;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    uint32_t w[4];
    ld_shared_v4(tile_base + atom * ATOM + sw128_offset(r, chunk0 + q), w[0], w[1], w[2], w[3]);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float2 f = __bfloat1622float2(*reinterpret_cast<__nv_bfloat162*>(&w[e]));
      v[8 * q + 2 * e] = f.x;
      v[8 * q + 2 * e + 1] = f.y;
    }
  }
}

struct OutView {  // generic strided output [rank][b][z][row][a]
  void* ptr;
  int64_t s_rank, s_b, s_z, s_row;
};

__device__ __forceinline__ int64_t out_off(const OutView& o, int rank, int b, int z, int row) {
  return int64_t(rank) * o.s_rank + int64_t(b) * o.s_b + int64_t(z) * o.s_z + int64_t(row) * o.s_row;
}

// Store 64 fp32 values of one row (fp32 accumulate and/or bf16 final).
__device__ __forceinline__ void store_row64(const OutView& acc, const OutView& fin, int accumulate, int rank, int b,
                                            int z, int row, float* v) {
  if (acc.ptr) {
    float* p = reinterpret_cast<float*>(acc.ptr) + out_off(acc, rank, b, z, row);
#pragma unroll
    for (int i = 0; i < 64; i += 4) {
      float4 o = make_float4(v[i], v[i + 1], v[i + 2], v[i + 3]);
      if (accumulate) {
        const float4 old = *reinterpret_cast<const float4*>(p + i);
        o.x += old.x, o.y += old.y, o.z += old.z, o.w += old.w;
        v[i] = o.x, v[i + 1] = o.y, v[i + 2] = o.z, v[i + 3] = o.w;
      }
      *reinterpret_cast<float4*>(p + i) = o;
    }
  }
  if (fin.ptr) {
    __nv_bfloat16* p = reinterpret_cast<__nv_bfloat16*>(fin.ptr) + out_off(fin, rank, b, z, row);
#pragma unroll
    for (int i = 0; i < 64; i += 8)
      *reinterpret_cast<uint4*>(p + i) = make_uint4(pack_bf16(v[i], v[i + 1]), pack_bf16(v[i + 2], v[i + 3]),
                                                    pack_bf16(v[i + 4], v[i + 5]), pack_bf16(v[i + 6], v[i + 7]));
  }
}

struct Geo {
  int n_rank, B, Z, c, L, org_lo, n_org;
  float scale;
};

// =================================================================== stats

struct StatsArgs {
  CUtensorMap tq, tk;
  Geo g;
  float sl;  // scale * log2(e)
  float2* stats;
  int64_t slot_off;
  int* flag;
};

constexpr int ST_STAGES = 4;
constexpr uint32_t ST_SMEM = TILE + ST_STAGES * TILE + 256 + 1024;

__global__ void __launch_bounds__(NTHREADS, 1) fwd_stats_kernel(const __grid_constant__ StatsArgs p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sq = smem;
  uint8_t* sk = smem + TILE;
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + TILE + ST_STAGES * TILE);
  uint64_t* q_full = bars;
  uint64_t* k_full = bars + 1;
  uint64_t* k_empty = k_full + ST_STAGES;
  uint64_t* s_full = k_empty + ST_STAGES;
  uint64_t* s_empty = s_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(s_empty + 2);

  const Geo& g = p.g;
  const int rt = blockIdx.x, bz = blockIdx.y, d = blockIdx.z;
  const int b = bz / g.Z, z = bz % g.Z;
  const int r0 = rt * TR;
  const int ntk = (g.c + TKEYS - 1) / TKEYS;
  const int T = g.n_org * ntk;
  const uint32_t warp = warp_id(), lane = lane_id();

  if (warp == 1) tmem_alloc(tmem_slot, 256);
  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    for (int s = 0; s < ST_STAGES; ++s) mbar_init(&k_full[s], 1), mbar_init(&k_empty[s], 1);
    for (int s = 0; s < 2; ++s) mbar_init(&s_full[s], 1), mbar_init(&s_empty[s], 4);
    fence_barrier_init();
    tma_prefetch(&p.tq);
    tma_prefetch(&p.tk);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      mbar_arrive_expect_tx(q_full, TILE);
      tma_load_4d(sq, &p.tq, q_full, 0, r0, z, d * g.B + b);
      for (int i = 0; i < T; ++i) {
        const int s = i % ST_STAGES;
        mbar_wait(&k_empty[s], ((i / ST_STAGES) & 1) ^ 1);
        mbar_arrive_expect_tx(&k_full[s], TILE);
        const int jo = i / ntk, k0 = (i % ntk) * TKEYS;
        tma_load_4d(sk + s * TILE, &p.tk, &k_full[s], 0, k0, z, jo * g.B + b);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t idesc = idesc_bf16_f32(TR, TKEYS, 0, 0);
      mbar_wait(q_full, 0);
      const uint32_t qa = smem_u32(sq);
      for (int i = 0; i < T; ++i) {
        const int s = i % ST_STAGES, buf = i & 1;
        mbar_wait(&k_full[s], (i / ST_STAGES) & 1);
        mbar_wait(&s_empty[buf], ((i >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t ka = smem_u32(sk + s * TILE);
#pragma unroll
        for (int k = 0; k < HD / 16; ++k)
          umma_bf16(tmem + buf * TKEYS, smem_desc_sw128(qa + k * 32, 0, 1024), smem_desc_sw128(ka + k * 32, 0, 1024),
                    idesc, k > 0);
        umma_commit(&k_empty[s]);
        umma_commit(&s_full[buf]);
      }
    }
  } else {
    const uint32_t quad = warp & 3;
    const int r = quad * 32 + lane;
    float m = -INFINITY, l = 0.f;
    bool bad = false;
    for (int i = 0; i < T; ++i) {
      const int buf = i & 1;
      mbar_wait(&s_full[buf], (i >> 1) & 1);
      tc_fence_after();
      const int nvalid = min(TKEYS, g.c - (i % ntk) * TKEYS);
#pragma unroll 1
      for (int cc = 0; cc < TKEYS / 32; ++cc) {
        float v[32];
        __syncwarp();
        tmem_ld32(tmem + ((quad * 32u) << 16) + buf * TKEYS + cc * 32, v);
        tmem_ld_wait();
        float cm = -INFINITY;
#pragma unroll
        for (int e = 0; e < 32; ++e) {
          const float t = __fmul_rn(v[e], p.sl);
          v[e] = (cc * 32 + e < nvalid) ? t : -INFINITY;
          bad |= !isfinite(t);
          cm = fmaxf(cm, v[e]);
        }
        if (cm > m) {
          l *= fast_exp2(m - cm);
          m = cm;
        }
#pragma unroll
        for (int e = 0; e < 32; ++e) l += fast_exp2(v[e] - m);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&s_empty[buf]);
    }
    const int row = r0 + r;
    if (row < g.c) {
      const int64_t idx = (int64_t(d * g.B + b) * g.Z + z) * g.c + row;
      p.stats[p.slot_off + idx] = make_float2(m, l);
      if (bad && p.flag) atomicExch(p.flag, 1);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, 256);
}

// ======================================================== probs + PV

struct PvArgs {
  CUtensorMap tq, tk, tv, tp;
  Geo g;
  float sl;
  const float2* stats;
  int n_slots;
  int64_t slot_stride;
  OutView o_acc, o_out;
  int accumulate;
};

constexpr int PV_STAGES = 3;
constexpr uint32_t PV_OFF_K = TILE;
constexpr uint32_t PV_OFF_V = PV_OFF_K + PV_STAGES * TILE;
constexpr uint32_t PV_OFF_P = PV_OFF_V + PV_STAGES * TILE;
constexpr uint32_t PV_OFF_BAR = PV_OFF_P + 2 * PTILE;
constexpr uint32_t PV_SMEM = PV_OFF_BAR + 256 + 1024;

__global__ void __launch_bounds__(NTHREADS, 1) fwd_pv_kernel(const __grid_constant__ PvArgs p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + PV_OFF_BAR);
  uint64_t* q_full = bars;
  uint64_t* kv_full = bars + 1;
  uint64_t* kv_empty = kv_full + PV_STAGES;
  uint64_t* s_full = kv_empty + PV_STAGES;
  uint64_t* s_empty = s_full + 2;
  uint64_t* p_full = s_empty + 2;
  uint64_t* p_empty = p_full + 2;
  uint64_t* o_full = p_empty + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_full + 1);

  const Geo& g = p.g;
  const int rt = blockIdx.x, bz = blockIdx.y, d = blockIdx.z;
  const int b = bz / g.Z, z = bz % g.Z;
  const int r0 = rt * TR;
  const int ntk = (g.c + TKEYS - 1) / TKEYS;
  const int T = g.n_org * ntk;
  const uint32_t warp = warp_id(), lane = lane_id();
  constexpr uint32_t O_COL = 2 * TKEYS;

  if (warp == 1) tmem_alloc(tmem_slot, 512);
  if (threadIdx.x == 0) {
    mbar_init(q_full, 1);
    for (int s = 0; s < PV_STAGES; ++s) mbar_init(&kv_full[s], 1), mbar_init(&kv_empty[s], 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&s_full[s], 1), mbar_init(&s_empty[s], 4);
      mbar_init(&p_full[s], 4), mbar_init(&p_empty[s], 1);
    }
    mbar_init(o_full, 1);
    fence_barrier_init();
    tma_prefetch(&p.tq);
    tma_prefetch(&p.tk);
    tma_prefetch(&p.tv);
    tma_prefetch(&p.tp);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      mbar_arrive_expect_tx(q_full, TILE);
      tma_load_4d(smem, &p.tq, q_full, 0, r0, z, d * g.B + b);
      for (int i = 0; i < T; ++i) {
        const int s = i % PV_STAGES;
        mbar_wait(&kv_empty[s], ((i / PV_STAGES) & 1) ^ 1);
        mbar_arrive_expect_tx(&kv_full[s], 2 * TILE);
        const int jo = i / ntk, k0 = (i % ntk) * TKEYS;
        tma_load_4d(smem + PV_OFF_K + s * TILE, &p.tk, &kv_full[s], 0, k0, z, jo * g.B + b);
        tma_load_4d(smem + PV_OFF_V + s * TILE, &p.tv, &kv_full[s], 0, k0, z, jo * g.B + b);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t idesc_s = idesc_bf16_f32(TR, TKEYS, 0, 0);
      const uint32_t idesc_o = idesc_bf16_f32(TR, HD, 0, 1);
      mbar_wait(q_full, 0);
      const uint32_t qa = smem_u32(smem);
      auto issue_s = [&](int i) {
        const int s = i % PV_STAGES, buf = i & 1;
        mbar_wait(&kv_full[s], (i / PV_STAGES) & 1);
        mbar_wait(&s_empty[buf], ((i >> 1) & 1) ^ 1);
        tc_fence_after();
        const uint32_t ka = smem_u32(smem + PV_OFF_K + s * TILE);
#pragma unroll
        for (int k = 0; k < HD / 16; ++k)
          umma_bf16(tmem + buf * TKEYS, smem_desc_sw128(qa + k * 32, 0, 1024), smem_desc_sw128(ka + k * 32, 0, 1024),
                    idesc_s, k > 0);
        umma_commit(&s_full[buf]);
      };
      auto issue_pv = [&](int i) {
        const int s = i % PV_STAGES, pb = i & 1;
        mbar_wait(&p_full[pb], (i >> 1) & 1);
        tc_fence_after();
        const uint32_t pa = smem_u32(smem + PV_OFF_P + pb * PTILE);
        const uint32_t va = smem_u32(smem + PV_OFF_V + s * TILE);
#pragma unroll
        for (int k = 0; k < TKEYS / 16; ++k)
          umma_bf16(tmem + O_COL, smem_desc_sw128(pa + (k >> 2) * ATOM + (k & 3) * 32, 0, 1024),
                    smem_desc_sw128(va + k * 2048, ATOM, 1024), idesc_o, (i | k) != 0);
        umma_commit(&kv_empty[s]);
        umma_commit(&p_empty[pb]);
      };
      if (T > 0) issue_s(0);
      for (int i = 0; i < T; ++i) {
        if (i + 1 < T) issue_s(i + 1);
        issue_pv(i);
      }
      umma_commit(o_full);
    }
  } else {
    const uint32_t quad = warp & 3;
    const int r = quad * 32 + lane;
    const int et = (warp - 2) * 32 + lane;
    const int row = r0 + r;
    const int head = (d * g.B + b) * g.Z + z;
    float m = 0.f, inv_l = 1.f;
    if (row < g.c) {
      const int64_t idx = int64_t(head) * g.c + row;
      float mm = -INFINITY, ll = 0.f;
      for (int s = 0; s < p.n_slots; ++s) {
        const float2 st = p.stats[s * p.slot_stride + idx];
        const float mn = fmaxf(mm, st.x);
        if (mn != -INFINITY) {
          ll = ll * fast_exp2(mm - mn) + st.y * fast_exp2(st.x - mn);
          mm = mn;
        }
      }
      m = mm;
      inv_l = 1.f / ll;
    }
    const uint32_t pbase = smem_u32(smem + PV_OFF_P);
    for (int i = 0; i < T; ++i) {
      const int buf = i & 1;
      const int jo = i / ntk, k0 = (i % ntk) * TKEYS;
      const int nvalid = min(TKEYS, g.c - k0);
      mbar_wait(&s_full[buf], (i >> 1) & 1);
      mbar_wait(&p_empty[buf], ((i >> 1) & 1) ^ 1);
      if (et == 0 && i >= 2) tma_store_wait_read<1>();
      epi_bar();
      tc_fence_after();
#pragma unroll 1
      for (int cc = 0; cc < TKEYS / 32; ++cc) {
        float v[32];
        __syncwarp();
        tmem_ld32(tmem + ((quad * 32u) << 16) + buf * TKEYS + cc * 32, v);
        tmem_ld_wait();
#pragma unroll
        for (int e = 0; e < 32; ++e)
          v[e] = (cc * 32 + e < nvalid) ? fast_exp2(__fmul_rn(v[e], p.sl) - m) * inv_l : 0.f;
        st_row32_sw128(pbase + buf * PTILE, r, cc * 32, v);
      }
      tc_fence_before();
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&s_empty[buf]);
        mbar_arrive(&p_full[buf]);
      }
      epi_bar();
      if (et == 0) {
        const int jg = g.org_lo + jo;
        tma_store_5d(&p.tp, smem + PV_OFF_P + buf * PTILE, k0, jg, r0, z, d * g.B + b);
        if (nvalid > 64) tma_store_5d(&p.tp, smem + PV_OFF_P + buf * PTILE + ATOM, k0 + 64, jg, r0, z, d * g.B + b);
        tma_store_commit();
      }
    }
    mbar_wait(o_full, 0);
    tc_fence_after();
    float v[64];
    __syncwarp();
    tmem_ld32(tmem + ((quad * 32u) << 16) + O_COL, v);
    tmem_ld32(tmem + ((quad * 32u) << 16) + O_COL + 32, v + 32);
    tmem_ld_wait();
    if (row < g.c) store_row64(p.o_acc, p.o_out, p.accumulate, d, b, z, row, v);
    if (et == 0) tma_store_wait_all<0>();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, 512);
}

// ================================================================ dK / dV

struct DkdvArgs {
  CUtensorMap tq, tv, tdo, tp, tds;
  Geo g;
  const float* dvec;
  OutView dk, dv;
  int dkv_bf16;
  int accumulate;
};

constexpr int BK_STAGES = 2;
constexpr uint32_t BK_STAGE = TILE /*dO*/ + TILE /*Q*/ + PTILE /*P*/;
constexpr uint32_t BK_OFF_ST = TILE;  // after V
constexpr uint32_t BK_OFF_DS = BK_OFF_ST + BK_STAGES * BK_STAGE;
constexpr uint32_t BK_OFF_BAR = BK_OFF_DS + 2 * PTILE;
constexpr uint32_t BK_SMEM = BK_OFF_BAR + 256 + 1024;

__global__ void __launch_bounds__(NTHREADS, 1) bwd_dkdv_kernel(const __grid_constant__ DkdvArgs p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + BK_OFF_BAR);
  uint64_t* v_full = bars;
  uint64_t* ld_full = bars + 1;
  uint64_t* ld_empty = ld_full + BK_STAGES;
  uint64_t* dp_full = ld_empty + BK_STAGES;
  uint64_t* dp_empty = dp_full + 2;
  uint64_t* ds_full = dp_empty + 2;
  uint64_t* ds_empty = ds_full + 2;
  uint64_t* acc_full = ds_empty + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_full + 1);

  const Geo& g = p.g;
  const int kt = blockIdx.x, bz = blockIdx.y, jo = blockIdx.z;
  const int b = bz / g.Z, z = bz % g.Z;
  const int k0 = kt * TKEYS;
  const int jg = g.org_lo + jo;
  const int nrt = (g.c + TR - 1) / TR;
  const int T = g.n_rank * nrt;
  const uint32_t warp = warp_id(), lane = lane_id();
  constexpr uint32_t DV_COL = 2 * TKEYS, DK_COL = 2 * TKEYS + HD;

  if (warp == 1) tmem_alloc(tmem_slot, 512);
  if (threadIdx.x == 0) {
    mbar_init(v_full, 1);
    for (int s = 0; s < BK_STAGES; ++s) mbar_init(&ld_full[s], 1), mbar_init(&ld_empty[s], 1 + 4);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&dp_full[s], 1), mbar_init(&dp_empty[s], 4);
      mbar_init(&ds_full[s], 4), mbar_init(&ds_empty[s], 1);
    }
    mbar_init(acc_full, 1);
    fence_barrier_init();
    tma_prefetch(&p.tq);
    tma_prefetch(&p.tv);
    tma_prefetch(&p.tdo);
    tma_prefetch(&p.tp);
    tma_prefetch(&p.tds);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      mbar_arrive_expect_tx(v_full, TILE);
      tma_load_4d(smem, &p.tv, v_full, 0, k0, z, jo * g.B + b);
      for (int i = 0; i < T; ++i) {
        const int s = i % BK_STAGES;
        const int d = i / nrt, r0 = (i % nrt) * TR;
        mbar_wait(&ld_empty[s], ((i / BK_STAGES) & 1) ^ 1);
        mbar_arrive_expect_tx(&ld_full[s], BK_STAGE);
        uint8_t* st = smem + BK_OFF_ST + s * BK_STAGE;
        tma_load_4d(st, &p.tdo, &ld_full[s], 0, r0, z, d * g.B + b);
        tma_load_4d(st + TILE, &p.tq, &ld_full[s], 0, r0, z, d * g.B + b);
        tma_load_5d(st + 2 * TILE, &p.tp, &ld_full[s], k0, jg, r0, z, d * g.B + b);
        tma_load_5d(st + 2 * TILE + ATOM, &p.tp, &ld_full[s], k0 + 64, jg, r0, z, d * g.B + b);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t idesc_dp = idesc_bf16_f32(TR, TKEYS, 0, 0);  // dO (K-major) x V (K-major)
      const uint32_t idesc_kv = idesc_bf16_f32(TKEYS, HD, 1, 1);  // P^T / dS^T (MN-major) x dO / Q (MN-major)
      mbar_wait(v_full, 0);
      const uint32_t va = smem_u32(smem);
      for (int i = 0; i < T; ++i) {
        const int s = i % BK_STAGES, buf = i & 1;
        const uint32_t st = smem_u32(smem + BK_OFF_ST + s * BK_STAGE);
        const uint32_t doa = st, qa = st + TILE, pa = st + 2 * TILE;
        const uint32_t dsa = smem_u32(smem + BK_OFF_DS + buf * PTILE);
        mbar_wait(&ld_full[s], (i / BK_STAGES) & 1);
        mbar_wait(&dp_empty[buf], ((i >> 1) & 1) ^ 1);
        tc_fence_after();
#pragma unroll
        for (int k = 0; k < HD / 16; ++k)
          umma_bf16(tmem + buf * TKEYS, smem_desc_sw128(doa + k * 32, 0, 1024), smem_desc_sw128(va + k * 32, 0, 1024),
                    idesc_dp, k > 0);
        umma_commit(&dp_full[buf]);
        // dV += P^T dO : contraction over the 128 query rows of this tile
#pragma unroll
        for (int k = 0; k < TR / 16; ++k)
          umma_bf16(tmem + DV_COL, smem_desc_sw128(pa + k * 2048, ATOM, 1024), smem_desc_sw128(doa + k * 2048, ATOM, 1024),
                    idesc_kv, (i | k) != 0);
        mbar_wait(&ds_full[buf], (i >> 1) & 1);
        tc_fence_after();
        // dK += dS^T Q
#pragma unroll
        for (int k = 0; k < TR / 16; ++k)
          umma_bf16(tmem + DK_COL, smem_desc_sw128(dsa + k * 2048, ATOM, 1024), smem_desc_sw128(qa + k * 2048, ATOM, 1024),
                    idesc_kv, (i | k) != 0);
        umma_commit(&ld_empty[s]);
        umma_commit(&ds_empty[buf]);
      }
      umma_commit(acc_full);
    }
  } else {
    const uint32_t quad = warp & 3;
    const int r = quad * 32 + lane;
    const int et = (warp - 2) * 32 + lane;
    const uint32_t dsbase = smem_u32(smem + BK_OFF_DS);
    for (int i = 0; i < T; ++i) {
      const int s = i % BK_STAGES, buf = i & 1;
      const int d = i / nrt, r0 = (i % nrt) * TR;
      const int row = r0 + r;
      const float dval = row < g.c ? p.dvec[(int64_t((d * g.B + b) * g.Z + z)) * g.c + row] : 0.f;
      const uint32_t pbase = smem_u32(smem + BK_OFF_ST + s * BK_STAGE + 2 * TILE);
      mbar_wait(&ld_full[s], (i / BK_STAGES) & 1);
      mbar_wait(&dp_full[buf], (i >> 1) & 1);
      mbar_wait(&ds_empty[buf], ((i >> 1) & 1) ^ 1);
      if (et == 0 && i >= 2) tma_store_wait_read<1>();
      epi_bar();
      tc_fence_after();
#pragma unroll 1
      for (int cc = 0; cc < TKEYS / 32; ++cc) {
        float v[32], pv[32];
        __syncwarp();
        tmem_ld32(tmem + ((quad * 32u) << 16) + buf * TKEYS + cc * 32, v);
        ld_row32_sw128(pbase, r, cc * 32, pv);
        tmem_ld_wait();
#pragma unroll
        for (int e = 0; e < 32; ++e) v[e] = pv[e] * (v[e] - dval) * g.scale;
        st_row32_sw128(dsbase + buf * PTILE, r, cc * 32, v);
      }
      tc_fence_before();
      fence_proxy_async_smem();
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(&dp_empty[buf]);
        mbar_arrive(&ld_empty[s]);
        mbar_arrive(&ds_full[buf]);
      }
      epi_bar();
      if (et == 0) {
        tma_store_5d(&p.tds, smem + BK_OFF_DS + buf * PTILE, k0, jg, r0, z, d * g.B + b);
        if (g.c - k0 > 64) tma_store_5d(&p.tds, smem + BK_OFF_DS + buf * PTILE + ATOM, k0 + 64, jg, r0, z, d * g.B + b);
        tma_store_commit();
      }
    }
    mbar_wait(acc_full, 0);
    tc_fence_after();
    const int key = k0 + r;
    float v[64];
    __syncwarp();
    tmem_ld32(tmem + ((quad * 32u) << 16) + DV_COL, v);
    tmem_ld32(tmem + ((quad * 32u) << 16) + DV_COL + 32, v + 32);
    tmem_ld_wait();
    const OutView none{nullptr, 0, 0, 0, 0};
    if (key < g.c) {
      if (p.dkv_bf16)
        store_row64(none, p.dv, 0, jo, b, z, key, v);
      else
        store_row64(p.dv, none, p.accumulate, jo, b, z, key, v);
    }
    __syncwarp();
    tmem_ld32(tmem + ((quad * 32u) << 16) + DK_COL, v);
    tmem_ld32(tmem + ((quad * 32u) << 16) + DK_COL + 32, v + 32);
    tmem_ld_wait();
    if (key < g.c) {
      if (p.dkv_bf16)
        store_row64(none, p.dk, 0, jo, b, z, key, v);
      else
        store_row64(p.dk, none, p.accumulate, jo, b, z, key, v);
    }
    if (et == 0) tma_store_wait_all<0>();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, 512);
}

// ===================================================================== dQ

struct DqArgs {
  CUtensorMap tds, tk;
  Geo g;
  OutView dq_acc, dq_out;
  int accumulate;
};

constexpr int DQ_STAGES = 4;
constexpr uint32_t DQ_STAGE = PTILE + TILE;
constexpr uint32_t DQ_OFF_BAR = DQ_STAGES * DQ_STAGE;
constexpr uint32_t DQ_SMEM = DQ_OFF_BAR + 256 + 1024;

__global__ void __launch_bounds__(NTHREADS, 1) bwd_dq_kernel(const __grid_constant__ DqArgs p) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t* bars = reinterpret_cast<uint64_t*>(smem + DQ_OFF_BAR);
  uint64_t* ld_full = bars;
  uint64_t* ld_empty = ld_full + DQ_STAGES;
  uint64_t* acc_full = ld_empty + DQ_STAGES;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_full + 1);

  const Geo& g = p.g;
  const int rt = blockIdx.x, bz = blockIdx.y, d = blockIdx.z;
  const int b = bz / g.Z, z = bz % g.Z;
  const int r0 = rt * TR;
  const int ntk = (g.c + TKEYS - 1) / TKEYS;
  const int T = g.n_org * ntk;
  const uint32_t warp = warp_id(), lane = lane_id();

  if (warp == 1) tmem_alloc(tmem_slot, 64);
  if (threadIdx.x == 0) {
    for (int s = 0; s < DQ_STAGES; ++s) mbar_init(&ld_full[s], 1), mbar_init(&ld_empty[s], 1);
    mbar_init(acc_full, 1);
    fence_barrier_init();
    tma_prefetch(&p.tds);
    tma_prefetch(&p.tk);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      for (int i = 0; i < T; ++i) {
        const int s = i % DQ_STAGES;
        const int jo = i / ntk, k0 = (i % ntk) * TKEYS;
        mbar_wait(&ld_empty[s], ((i / DQ_STAGES) & 1) ^ 1);
        mbar_arrive_expect_tx(&ld_full[s], DQ_STAGE);
        uint8_t* st = smem + s * DQ_STAGE;
        tma_load_5d(st, &p.tds, &ld_full[s], k0, g.org_lo + jo, r0, z, d * g.B + b);
        tma_load_5d(st + ATOM, &p.tds, &ld_full[s], k0 + 64, g.org_lo + jo, r0, z, d * g.B + b);
        tma_load_4d(st + PTILE, &p.tk, &ld_full[s], 0, k0, z, jo * g.B + b);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      const uint32_t idesc = idesc_bf16_f32(TR, HD, 0, 1);  // dS (K-major over keys) x K (MN-major)
      for (int i = 0; i < T; ++i) {
        const int s = i % DQ_STAGES;
        mbar_wait(&ld_full[s], (i / DQ_STAGES) & 1);
        tc_fence_after();
        const uint32_t dsa = smem_u32(smem + s * DQ_STAGE), ka = dsa + PTILE;
#pragma unroll
        for (int k = 0; k < TKEYS / 16; ++k)
          umma_bf16(tmem, smem_desc_sw128(dsa + (k >> 2) * ATOM + (k & 3) * 32, 0, 1024),
                    smem_desc_sw128(ka + k * 2048, ATOM, 1024), idesc, (i | k) != 0);
        umma_commit(&ld_empty[s]);
      }
      umma_commit(acc_full);
    }
  } else {
    const uint32_t quad = warp & 3;
    const int row = r0 + quad * 32 + lane;
    mbar_wait(acc_full, 0);
    tc_fence_after();
    float v[64];
    __syncwarp();
    tmem_ld32(tmem + ((quad * 32u) << 16), v);
    tmem_ld32(tmem + ((quad * 32u) << 16) + 32, v + 32);
    tmem_ld_wait();
    if (row < g.c) store_row64(p.dq_acc, p.dq_out, p.accumulate, d, b, z, row, v);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, 64);
}

// ================================================================== host

bool geom_ok(const rsa_geom* g) {
  return g && g->n_rank >= 1 && g->batch >= 1 && g->heads >= 1 && g->chunk >= 1 && g->head_dim == HD &&
         g->n_org >= 1 && g->org_lo >= 0 && g->seq_len % g->chunk == 0 && g->chunk % 8 == 0 &&
         g->org_lo + g->n_org <= g->seq_len / g->chunk && int64_t(g->batch) * g->heads <= 65535 &&
         g->n_rank <= 65535 && g->n_org <= 65535;
}

Geo to_geo(const rsa_geom* g) {
  return Geo{g->n_rank, g->batch, g->heads, g->chunk, g->seq_len, g->org_lo, g->n_org, g->scale};
}

// [rank][b][z][row][a] with a = 64 contiguous, `nrank` ranks merged into b.
bool head_map(CUtensorMap* m, const rsa_view& v, const rsa_geom* g, int nrank) {
  if (!v.ptr || !aligned16(v.ptr)) return fail(RSA_ERR_UNSUPPORTED, "fused: tensor not 16-byte aligned"), false;
  if (nrank > 1 && v.s_rank != int64_t(g->batch) * v.s_b && g->batch > 1)
    return fail(RSA_ERR_UNSUPPORTED, "fused: rank stride must equal B * batch stride"), false;
  const int64_t sb = (g->batch == 1 && nrank > 1) ? v.s_rank : v.s_b;
  if (!stride_ok(v.s_row * 2) || !stride_ok(v.s_z * 2) || !stride_ok(sb * 2))
    return fail(RSA_ERR_UNSUPPORTED, "fused: strides must be multiples of 8 elements"), false;
  uint64_t dims[4] = {uint64_t(HD), uint64_t(g->chunk), uint64_t(g->heads), uint64_t(g->batch) * nrank};
  uint64_t str[3] = {uint64_t(v.s_row) * 2, uint64_t(v.s_z) * 2, uint64_t(sb) * 2};
  uint32_t box[4] = {64, TR, 1, 1};
  return encode_tmap(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, v.ptr, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B);
}

// [rank][b][z][row][col], col = blk * c + key: 5-D (key, blk, row, z, b*rank).
bool panel_map(CUtensorMap* m, const rsa_view& v, const rsa_geom* g, int nrank) {
  if (!v.ptr || !aligned16(v.ptr)) return fail(RSA_ERR_UNSUPPORTED, "fused: panel not 16-byte aligned"), false;
  if (nrank > 1 && v.s_rank != int64_t(g->batch) * v.s_b && g->batch > 1)
    return fail(RSA_ERR_UNSUPPORTED, "fused: panel rank stride must equal B * batch stride"), false;
  const int64_t sb = (g->batch == 1 && nrank > 1) ? v.s_rank : v.s_b;
  if (!stride_ok(v.s_row * 2) || !stride_ok(v.s_z * 2) || !stride_ok(sb * 2))
    return fail(RSA_ERR_UNSUPPORTED, "fused: panel strides must be multiples of 8 elements"), false;
  const int nblk = g->seq_len / g->chunk;
  uint64_t dims[5] = {uint64_t(g->chunk), uint64_t(nblk), uint64_t(g->chunk), uint64_t(g->heads),
                      uint64_t(g->batch) * nrank};
  uint64_t str[4] = {uint64_t(g->chunk) * 2, uint64_t(v.s_row) * 2, uint64_t(v.s_z) * 2, uint64_t(sb) * 2};
  uint32_t box[5] = {64, 1, TR, 1, 1};
  return encode_tmap(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, v.ptr, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B);
}

OutView to_out(const rsa_view& v) { return OutView{v.ptr, v.s_rank, v.s_b, v.s_z, v.s_row}; }

bool out_ok(const rsa_view& v, int esz) {
  if (!v.ptr) return true;
  return aligned16(v.ptr) && (v.s_row * esz) % 16 == 0 && (v.s_z * esz) % 16 == 0 && (v.s_b * esz) % 16 == 0 &&
         (v.s_rank * esz) % 16 == 0;
}

template <typename K, typename A>
int launch(K kernel, dim3 grid, uint32_t smem, const A& args, void* stream, const char* name) {
  cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  kernel<<<grid, NTHREADS, smem, reinterpret_cast<cudaStream_t>(stream)>>>(args);
  return check_launch(name);
}

}  // namespace
}  // namespace rsa

extern "C" {

int rsa_fused_supported(const rsa_geom* g) { return rsa::geom_ok(g) ? 1 : 0; }

int rsa_fwd_stats(const rsa_geom* g, rsa_view q, rsa_view k, float* stats, int slot, int* nonfinite_flag,
                  void* stream) {
  using namespace rsa;
  if (!geom_ok(g) || !stats || slot < 0) return fail(RSA_ERR_INVALID, "rsa_fwd_stats: unsupported geometry");
  StatsArgs a{};
  if (!head_map(&a.tq, q, g, g->n_rank) || !head_map(&a.tk, k, g, g->n_org)) return RSA_ERR_UNSUPPORTED;
  a.g = to_geo(g);
  a.sl = g->scale * LOG2E;
  a.stats = reinterpret_cast<float2*>(stats);
  a.slot_off = int64_t(slot) * g->n_rank * g->batch * g->heads * g->chunk;
  a.flag = nonfinite_flag;
  dim3 grid((g->chunk + TR - 1) / TR, g->batch * g->heads, g->n_rank);
  return launch(fwd_stats_kernel, grid, ST_SMEM, a, stream, "fwd_stats_kernel");
}

int rsa_fwd_probs_pv(const rsa_geom* g, rsa_view q, rsa_view k, rsa_view v, const float* stats, int n_slots,
                     rsa_view panel, rsa_view o_acc, int accumulate, rsa_view o_out, void* stream) {
  using namespace rsa;
  if (!geom_ok(g) || !stats || n_slots < 1) return fail(RSA_ERR_INVALID, "rsa_fwd_probs_pv: unsupported geometry");
  if (!out_ok(o_acc, 4) || !out_ok(o_out, 2)) return fail(RSA_ERR_UNSUPPORTED, "rsa_fwd_probs_pv: output alignment");
  PvArgs a{};
  if (!head_map(&a.tq, q, g, g->n_rank) || !head_map(&a.tk, k, g, g->n_org) || !head_map(&a.tv, v, g, g->n_org) ||
      !panel_map(&a.tp, panel, g, g->n_rank))
    return RSA_ERR_UNSUPPORTED;
  a.g = to_geo(g);
  a.sl = g->scale * LOG2E;
  a.stats = reinterpret_cast<const float2*>(stats);
  a.n_slots = n_slots;
  a.slot_stride = int64_t(g->n_rank) * g->batch * g->heads * g->chunk;
  a.o_acc = to_out(o_acc);
  a.o_out = to_out(o_out);
  a.accumulate = accumulate;
  dim3 grid((g->chunk + TR - 1) / TR, g->batch * g->heads, g->n_rank);
  return launch(fwd_pv_kernel, grid, PV_SMEM, a, stream, "fwd_pv_kernel");
}

int rsa_bwd_dkdv(const rsa_geom* g, rsa_view q, rsa_view v, rsa_view dout, rsa_view panel, const float* dvec,
                 rsa_view ds_panel, rsa_view dk, rsa_view dv, int dkv_dtype, int accumulate, void* stream) {
  using namespace rsa;
  if (!geom_ok(g) || !dvec) return fail(RSA_ERR_INVALID, "rsa_bwd_dkdv: unsupported geometry");
  const int esz = dkv_dtype == RSA_BF16 ? 2 : 4;
  if (!dk.ptr || !dv.ptr || !out_ok(dk, esz) || !out_ok(dv, esz))
    return fail(RSA_ERR_UNSUPPORTED, "rsa_bwd_dkdv: output alignment");
  DkdvArgs a{};
  if (!head_map(&a.tq, q, g, g->n_rank) || !head_map(&a.tdo, dout, g, g->n_rank) || !head_map(&a.tv, v, g, g->n_org) ||
      !panel_map(&a.tp, panel, g, g->n_rank) || !panel_map(&a.tds, ds_panel, g, g->n_rank))
    return RSA_ERR_UNSUPPORTED;
  a.g = to_geo(g);
  a.dvec = dvec;
  a.dk = to_out(dk);
  a.dv = to_out(dv);
  a.dkv_bf16 = dkv_dtype == RSA_BF16;
  a.accumulate = accumulate;
  dim3 grid((g->chunk + TKEYS - 1) / TKEYS, g->batch * g->heads, g->n_org);
  return launch(bwd_dkdv_kernel, grid, BK_SMEM, a, stream, "bwd_dkdv_kernel");
}

int rsa_bwd_dq(const rsa_geom* g, rsa_view ds_panel, rsa_view k, rsa_view dq_acc, int accumulate, rsa_view dq_out,
               void* stream) {
  using namespace rsa;
  if (!geom_ok(g)) return fail(RSA_ERR_INVALID, "rsa_bwd_dq: unsupported geometry");
  if (!out_ok(dq_acc, 4) || !out_ok(dq_out, 2)) return fail(RSA_ERR_UNSUPPORTED, "rsa_bwd_dq: output alignment");
  DqArgs a{};
  if (!panel_map(&a.tds, ds_panel, g, g->n_rank) || !head_map(&a.tk, k, g, g->n_org)) return RSA_ERR_UNSUPPORTED;
  a.g = to_geo(g);
  a.dq_acc = to_out(dq_acc);
  a.dq_out = to_out(dq_out);
  a.accumulate = accumulate;
  dim3 grid((g->chunk + TR - 1) / TR, g->batch * g->heads, g->n_rank);
  return launch(bwd_dq_kernel, grid, DQ_SMEM, a, stream, "bwd_dq_kernel");
}

}  // extern "C"

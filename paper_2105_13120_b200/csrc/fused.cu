// Fused Ring Self-Attention kernels for sm_100a (head size A = 64).
//
// Tensor layout (bf16 unless noted): per-head tensors are [rank][b][z][row][a];
// probability panels are [rank][b][z][row][col] with col = origin * c + key
// (ringseq/ring_attention.py:91-94: column block j of a panel is origin j).
// TMA moves 128-row x 64-column tiles (one 128-byte swizzle row per tile
// row).  In shared memory every tile uses the SWIZZLE_128B layout the UMMA
// descriptors read, and the same bytes serve as K-major or MN-major
// operands as each product needs (P is K-major A of P.V and MN-major A of
// P^T.dO; dO is K-major A of dO.V^T and MN-major B of P^T.dO; ...).
//
// All kernels are persistent (one CTA per SM walking a static work list)
// and warp-specialised, 10 warps:
//   warp 0      TMA producer (one lane)
//   warp 1      tcgen05.mma issuer (one lane); owns the TMEM allocation
//   warps 2..9  epilogue: warp w reads TMEM lanes 32*(w%4).. (tile rows) and
//               the column half (w-2)/4 of each 128-column tile, so row
//               reductions are thread-local plus one smem exchange.
// Accumulators and smem tiles are double-buffered, so the MMAs of tile i+1
// and the TMA loads of the next work item overlap the epilogue of tile i.
//
// rsa_fwd          K ring stage (pass A: S = Q K^T, running row max / sum of
//                  exp2) and V ring stage (pass B: S recomputed, P = 2^(S'-m)/l
//                  to smem -> TMA store to the bf16 panel and UMMA O += P V).
//                  Passes A+B in one launch when every key is resident.
// rsa_bwd_dkdv     per key tile: dP = dO V^T, dS = P (dP - D) scale (smem
//                  only), dV += P^T dO, dK += dS^T Q over all query rows.
// rsa_bwd_dq       per query row tile: dP, dS recomputed the same way,
//                  dQ += dS K.  dS never goes to HBM.
#include "fused_common.cuh"

namespace rsa {
namespace {

// ================================================================ forward

struct FwdArgs {
  CUtensorMap tq, tk, tv, tp;
  Geo g;
  int mode;
  float sl;  // scale * log2(e)
  float2* stats;
  int slot;
  int n_slots;
  int64_t slot_stride;
  int* flag;
  OutView o_acc, o_out;
  int accumulate;
};

constexpr int FK_ST = 3, FV_ST = 2;
constexpr uint32_t F_OFF_Q = 0;
constexpr uint32_t F_OFF_K = F_OFF_Q + 2 * TILE;
constexpr uint32_t F_OFF_V = F_OFF_K + FK_ST * TILE;
constexpr uint32_t F_OFF_P = F_OFF_V + FV_ST * TILE;
constexpr uint32_t F_OFF_X = F_OFF_P + 2 * PTILE;         // (m, l) exchange, 256 x float2
constexpr uint32_t F_OFF_BAR = F_OFF_X + EPI_THREADS * 8;
constexpr uint32_t F_SMEM = F_OFF_BAR + 512 + 1024;

__global__ void __launch_bounds__(NTHREADS, 1) fwd_kernel(const __grid_constant__ FwdArgs p) {
  uint8_t* smem = smem_base();
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + F_OFF_BAR);
  uint64_t *q_full = bar, *q_empty = bar + 2, *k_full = bar + 4, *k_empty = k_full + FK_ST;
  uint64_t *v_full = k_empty + FK_ST, *v_empty = v_full + FV_ST;
  uint64_t *s_full = v_empty + FV_ST, *s_empty = s_full + 2, *p_full = s_empty + 2, *p_empty = p_full + 2;
  uint64_t *o_full = p_empty + 2, *o_empty = o_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_empty + 2);

  const Geo& g = p.g;
  const bool pass_a = p.mode & MODE_PASS_A, pass_b = p.mode & MODE_PASS_B;
  const int ntk = (g.c + TK - 1) / TK, nrt = (g.c + TR - 1) / TR;
  const int T = g.n_org * ntk;
  const int BZ = g.B * g.Z;
  const int items = g.n_rank * BZ * nrt;
  const uint32_t warp = warp_id(), lane = lane_id();

  if (warp == 1) tmem_alloc(tmem_slot, 512);
  if (threadIdx.x == 0) {
    for (int s = 0; s < 2; ++s) {
      mbar_init(&q_full[s], 1), mbar_init(&q_empty[s], 1);
      mbar_init(&s_full[s], 1), mbar_init(&s_empty[s], EPI_WARPS);
      mbar_init(&p_full[s], EPI_WARPS), mbar_init(&p_empty[s], 1);
      mbar_init(&o_full[s], 1), mbar_init(&o_empty[s], EPI_WARPS);
    }
    for (int s = 0; s < FK_ST; ++s) mbar_init(&k_full[s], 1), mbar_init(&k_empty[s], 1);
    for (int s = 0; s < FV_ST; ++s) mbar_init(&v_full[s], 1), mbar_init(&v_empty[s], 1);
    fence_barrier_init();
    tma_prefetch(&p.tq);
    tma_prefetch(&p.tk);
    if (pass_b) tma_prefetch(&p.tv), tma_prefetch(&p.tp);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base(tmem_slot);

  if (warp == 0) {
    if (lane == 0) {
      Pos kq, vq;
      uint32_t it = 0;
      for (int item = blockIdx.x; item < items; item += gridDim.x, ++it) {
        const int rt = item % nrt, bz = (item / nrt) % BZ, d = item / (nrt * BZ);
        const int b = bz / g.Z, z = bz % g.Z;
        const int qb = it & 1;
        mbar_wait(&q_empty[qb], ((it >> 1) & 1) ^ 1);
        mbar_arrive_expect_tx(&q_full[qb], TILE);
        tma_load_4d(smem + F_OFF_Q + qb * TILE, &p.tq, &q_full[qb], 0, rt * TR, z, d * g.B + b);
        for (int pass = 0; pass < 2; ++pass) {
          if ((pass == 0 && !pass_a) || (pass == 1 && !pass_b)) continue;
          for (int t = 0, jo = 0, k0 = 0; t < T; ++t, k0 = k0 + TK >= ntk * TK ? (++jo, 0) : k0 + TK) {
            const uint32_t ks = kq.slot(FK_ST);
            mbar_wait(&k_empty[ks], kq.phase(FK_ST) ^ 1);
            mbar_arrive_expect_tx(&k_full[ks], TILE);
            tma_load_4d(smem + F_OFF_K + ks * TILE, &p.tk, &k_full[ks], 0, k0, z, jo * g.B + b);
            ++kq.i;
            if (pass == 1) {
              const uint32_t vs = vq.slot(FV_ST);
              mbar_wait(&v_empty[vs], vq.phase(FV_ST) ^ 1);
              mbar_arrive_expect_tx(&v_full[vs], TILE);
              tma_load_4d(smem + F_OFF_V + vs * TILE, &p.tv, &v_full[vs], 0, k0, z, jo * g.B + b);
              ++vq.i;
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    {  // whole warp; elect.sync inside the _ws issue helpers
      const uint32_t idesc_s = idesc_bf16_f32(TR, TK, 0, 0);
      const uint32_t idesc_o = idesc_bf16_f32(TR, HD, 0, 1);
      Pos kq, vq, sq, pq;
      uint32_t it = 0;
      for (int item = blockIdx.x; item < items; item += gridDim.x, ++it) {
        const int qb = it & 1;
        mbar_wait(&q_full[qb], (it >> 1) & 1);
        const uint32_t qa = smem_u32(smem + F_OFF_Q + qb * TILE);
        auto issue_s = [&]() {
          const uint32_t ks = kq.slot(FK_ST), sb = sq.slot(2);
          mbar_wait(&k_full[ks], kq.phase(FK_ST));
          mbar_wait(&s_empty[sb], sq.phase(2) ^ 1);
          tc_fence_after();
          const uint32_t ka = smem_u32(smem + F_OFF_K + ks * TILE);
#pragma unroll
          for (int k = 0; k < HD / 16; ++k)
            umma_bf16_ws(tmem + sb * TK, smem_desc_sw128(qa + k * 32, 0, 1024), smem_desc_sw128(ka + k * 32, 0, 1024),
                      idesc_s, k > 0);
          umma_commit_ws(&k_empty[ks]);
          umma_commit_ws(&s_full[sb]);
          ++kq.i, ++sq.i;
        };
        if (pass_a)
          for (int t = 0; t < T; ++t) issue_s();
        if (pass_b) {
          const uint32_t ob = it & 1;
          mbar_wait(&o_empty[ob], ((it >> 1) & 1) ^ 1);
          if (T > 0) issue_s();
          for (int t = 0; t < T; ++t) {
            if (t + 1 < T) issue_s();
            const uint32_t pb = pq.slot(2), vs = vq.slot(FV_ST);
            mbar_wait(&p_full[pb], pq.phase(2));
            mbar_wait(&v_full[vs], vq.phase(FV_ST));
            tc_fence_after();
            const uint32_t pa = smem_u32(smem + F_OFF_P + pb * PTILE);
            const uint32_t va = smem_u32(smem + F_OFF_V + vs * TILE);
#pragma unroll
            for (int k = 0; k < TK / 16; ++k)
              umma_bf16_ws(tmem + 2 * TK + ob * HD, smem_desc_sw128(pa + (k >> 2) * ATOM + (k & 3) * 32, 0, 1024),
                        smem_desc_sw128(va + k * 2048, ATOM, 1024), idesc_o, (t | k) != 0);
            umma_commit_ws(&v_empty[vs]);
            umma_commit_ws(&p_empty[pb]);
            ++pq.i, ++vq.i;
          }
          umma_commit_ws(&o_full[ob]);
        }
        umma_commit_ws(&q_empty[qb]);
      }
    }
  } else {
    const uint32_t quad = warp & 3;
    const int half = (warp - 2) >> 2;  // which 64-column half of each S tile
    const int r = quad * 32 + lane;
    const int et = threadIdx.x - 64;   // 0..255
    const bool storer = (lane == 0) && (quad == 2);  // first warp of each half issues its TMA stores
    const uint32_t lane_base = (quad * 32u) << 16;
    const uint32_t xbase = smem_u32(smem + F_OFF_X);
    const uint32_t pbase = smem_u32(smem + F_OFF_P);
    const float sl = p.sl;
    Pos sq, pq;
    uint32_t it = 0;
    bool bad = false;
    auto load_s = [&](float* v) {  // this thread's 64 columns of the next S tile, then free the buffer
      const uint32_t sb = sq.slot(2);
      mbar_wait(&s_full[sb], sq.phase(2));
      tc_fence_after();
      __syncwarp();
      tmem_ld32(tmem + lane_base + sb * TK + half * 64, v);
      tmem_ld32(tmem + lane_base + sb * TK + half * 64 + 32, v + 32);
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&s_empty[sb]);
      ++sq.i;
    };
    for (int item = blockIdx.x; item < items; item += gridDim.x, ++it) {
      const int rt = item % nrt, bz = (item / nrt) % BZ, d = item / (nrt * BZ);
      const int b = bz / g.Z, z = bz % g.Z;
      const int row = rt * TR + r;
      const int64_t sidx = (int64_t(d * g.B + b) * g.Z + z) * g.c + row;
      float bias = 0.f;  // pass B computes p = 2^(s*sl - bias), bias = m*sl + log2(l)
      if (pass_a) {
        float m = -INFINITY, l = 0.f;  // m: raw (unscaled) row max; l = sum 2^((s - m) * sl)
        int k0 = 0;
        for (int t = 0; t < T; ++t) {
          float v[64];
          load_s(v);
          const int nvalid = min(TK, g.c - k0) - half * 64;
          k0 = k0 + TK >= g.c ? 0 : k0 + TK;
          if (nvalid <= 0) continue;
          float cmax, cmin;
          if (nvalid >= 64) {
            float mx[8], mi[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) mx[e] = mi[e] = v[e];
#pragma unroll
            for (int e = 8; e < 64; ++e) mx[e & 7] = max_nan(mx[e & 7], v[e]), mi[e & 7] = min_nan(mi[e & 7], v[e]);
#pragma unroll
            for (int w = 4; w; w >>= 1)
#pragma unroll
              for (int e = 0; e < w; ++e) mx[e] = max_nan(mx[e], mx[e + w]), mi[e] = min_nan(mi[e], mi[e + w]);
            cmax = mx[0], cmin = mi[0];
          } else {
            cmax = -INFINITY, cmin = INFINITY;
#pragma unroll
            for (int e = 0; e < 64; ++e)
              if (e < nvalid) cmax = max_nan(cmax, v[e]), cmin = min_nan(cmin, v[e]);
          }
          bad |= !(fabsf(cmax) <= 3.402823466e38f) || !(fabsf(cmin) <= 3.402823466e38f);
          const float mn = fmaxf(m, cmax);
          if (mn > m) {
            l *= fast_exp2((m - mn) * sl);
            m = mn;
          }
          const float msl = m * sl;
          float acc[4] = {0.f, 0.f, 0.f, 0.f};
          if (nvalid >= 64) {
#pragma unroll
            for (int e = 0; e < 64; ++e) {
              const float x = fmaf(v[e], sl, -msl);
              acc[e & 3] += (e & 3) == 3 ? exp2_poly<4>(x) : fast_exp2(x);
            }
          } else {
#pragma unroll
            for (int e = 0; e < 64; ++e)
              if (e < nvalid) acc[e & 3] += fast_exp2(fmaf(v[e], sl, -msl));
          }
          l += (acc[0] + acc[1]) + (acc[2] + acc[3]);
        }
        // combine the two column halves of each row through shared memory
        st_shared_f2(xbase + et * 8, m, l);
        bar_epi();
        const float2 o = ld_shared_f2(xbase + ((et + 128) & 255) * 8);
        bar_epi();
        const float mn = fmaxf(m, o.x);
        if (mn != -INFINITY) {
          l = l * fast_exp2((m - mn) * sl) + o.y * fast_exp2((o.x - mn) * sl);
          m = mn;
        }
        if ((p.mode & MODE_WRITE_STATS) && half == 0 && row < g.c)
          p.stats[int64_t(p.slot) * p.slot_stride + sidx] = make_float2(m * sl, l);
        bias = (row < g.c && l > 0.f) ? m * sl + __log2f(l) : 0.f;
      }
      if (!pass_b) continue;
      if (p.mode & MODE_EXT_STATS) {  // stats slots hold (scaled max, sum), base 2
        float msl = -INFINITY, l = 0.f;
        if (row < g.c)
          for (int s = 0; s < p.n_slots; ++s) {
            const float2 st = p.stats[int64_t(s) * p.slot_stride + sidx];
            const float mn = fmaxf(msl, st.x);
            if (mn != -INFINITY) {
              l = l * fast_exp2(msl - mn) + st.y * fast_exp2(st.x - mn);
              msl = mn;
            }
          }
        bias = (row < g.c && l > 0.f) ? msl + __log2f(l) : 0.f;  // padded rows: finite garbage, never stored
      }
      int jo = 0, k0 = 0;
      for (int t = 0; t < T; ++t) {
        const uint32_t pb = pq.slot(2);
        const int nvalid = min(TK, g.c - k0) - half * 64;
        float v[64];
        load_s(v);
        if (nvalid >= 64) {
#pragma unroll
          for (int e = 0; e < 64; ++e) {
            const float x = fmaf(v[e], sl, -bias);
            v[e] = (e & 3) == 3 ? exp2_poly<3>(x) : fast_exp2(x);
          }
        } else {
#pragma unroll
          for (int e = 0; e < 64; ++e) v[e] = e < nvalid ? fast_exp2(fmaf(v[e], sl, -bias)) : 0.f;
        }
        mbar_wait(&p_empty[pb], pq.phase(2) ^ 1);
        if (storer && pq.i >= 2) tma_store_wait_read<1>();
        bar_half(half);
        const uint32_t ptile = pbase + pb * PTILE;
        st_row32_sw128(ptile, r, half * 64, v);
        st_row32_sw128(ptile, r, half * 64 + 32, v + 32);
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&p_full[pb]);
        bar_half(half);
        if (storer) {
          if (nvalid > 0)
            tma_store_5d(&p.tp, smem + F_OFF_P + pb * PTILE + half * ATOM, k0 + half * 64, g.org_lo + jo, rt * TR,
                         z, d * g.B + b);
          tma_store_commit();
        }
        ++pq.i;
        if (k0 + TK >= g.c) k0 = 0, ++jo;
        else k0 += TK;
      }
      const uint32_t ob = it & 1;
      mbar_wait(&o_full[ob], (it >> 1) & 1);
      tc_fence_after();
      float o[32];
      __syncwarp();
      tmem_ld32(tmem + lane_base + 2 * TK + ob * HD + half * 32, o);
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&o_empty[ob]);
      if (row < g.c) store_row32(p.o_acc, p.o_out, p.accumulate, d, b, z, row, half * 32, o);
    }
    if (bad && p.flag) atomicExch(p.flag, 1);
    if (storer) tma_store_wait_all<0>();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, 512);
}

// ============================================================== dK / dV

struct DkdvArgs {
  CUtensorMap tq, tv, tdo, tp;
  Geo g;
  const float* dvec;
  OutView dk, dv;
  int dkv_bf16;
  int accumulate;
};

// A stage holds dO, Q and the P tile; the epilogue overwrites P with dS in
// place (each thread rewrites exactly the elements it read, after the
// P^T dO product that also reads P has completed), so 3 stages fit.
constexpr int BK_ST = 3;
constexpr uint32_t BK_STAGE = TILE /*dO*/ + TILE /*Q*/ + PTILE /*P, then dS*/;
constexpr uint32_t BK_OFF_V = 0;
constexpr uint32_t BK_OFF_ST = TILE;
constexpr uint32_t BK_OFF_BAR = BK_OFF_ST + BK_ST * BK_STAGE;
constexpr uint32_t BK_SMEM = BK_OFF_BAR + 512 + 1024;

__global__ void __launch_bounds__(NTHREADS, 1) bwd_dkdv_kernel(const __grid_constant__ DkdvArgs p) {
  uint8_t* smem = smem_base();
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + BK_OFF_BAR);
  uint64_t *v_full = bar, *v_empty = bar + 1, *ld_full = bar + 2, *ld_empty = ld_full + BK_ST;
  uint64_t *dp_full = ld_empty + BK_ST, *dp_empty = dp_full + 2, *ds_full = dp_empty + 2, *ds_empty = ds_full + 2;
  uint64_t *acc_full = ds_empty + 2, *acc_empty = acc_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

  const Geo& g = p.g;
  const int ntk = (g.c + TK - 1) / TK, nrt = (g.c + TR - 1) / TR;
  const int T = g.n_rank * nrt;  // query row tiles walked per key tile
  const int BZ = g.B * g.Z;
  const int items = g.n_org * BZ * ntk;
  const uint32_t warp = warp_id(), lane = lane_id();
  constexpr uint32_t ACC_COL = 2 * TK;  // [dV | dK] x 2 buffers, 128 columns each

  if (warp == 1) tmem_alloc(tmem_slot, 512);
  if (threadIdx.x == 0) {
    mbar_init(v_full, 1), mbar_init(v_empty, 1);
    for (int s = 0; s < BK_ST; ++s) mbar_init(&ld_full[s], 1), mbar_init(&ld_empty[s], 1);
    for (int s = 0; s < 2; ++s) {
      mbar_init(&dp_full[s], 1), mbar_init(&dp_empty[s], EPI_WARPS);
      mbar_init(&ds_full[s], EPI_WARPS), mbar_init(&ds_empty[s], 1);
      mbar_init(&acc_full[s], 1), mbar_init(&acc_empty[s], EPI_WARPS);
    }
    fence_barrier_init();
    tma_prefetch(&p.tq), tma_prefetch(&p.tv), tma_prefetch(&p.tdo), tma_prefetch(&p.tp);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base(tmem_slot);

  if (warp == 0) {
    if (lane == 0) {
      Pos lq;
      uint32_t it = 0;
      const uint64_t pol = l2_evict_first();  // the panel streams through once
      for (int item = blockIdx.x; item < items; item += gridDim.x, ++it) {
        const int kt = item % ntk, bz = (item / ntk) % BZ, jo = item / (ntk * BZ);
        const int b = bz / g.Z, z = bz % g.Z, k0 = kt * TK, jg = g.org_lo + jo;
        mbar_wait(v_empty, (it & 1) ^ 1);
        mbar_arrive_expect_tx(v_full, TILE);
        tma_load_4d(smem + BK_OFF_V, &p.tv, v_full, 0, k0, z, jo * g.B + b);
        for (int t = 0, d = 0, r0 = 0; t < T; ++t, r0 = r0 + TR >= nrt * TR ? (++d, 0) : r0 + TR) {
          const uint32_t s = lq.slot(BK_ST);
          mbar_wait(&ld_empty[s], lq.phase(BK_ST) ^ 1);
          mbar_arrive_expect_tx(&ld_full[s], BK_STAGE);
          uint8_t* st = smem + BK_OFF_ST + s * BK_STAGE;
          tma_load_4d(st, &p.tdo, &ld_full[s], 0, r0, z, d * g.B + b);
          tma_load_4d(st + TILE, &p.tq, &ld_full[s], 0, r0, z, d * g.B + b);
          tma_load_5d_hint(st + 2 * TILE, &p.tp, &ld_full[s], k0, jg, r0, z, d * g.B + b, pol);
          tma_load_5d_hint(st + 2 * TILE + ATOM, &p.tp, &ld_full[s], k0 + 64, jg, r0, z, d * g.B + b, pol);
          ++lq.i;
        }
      }
    }
  } else if (warp == 1) {
    {  // whole warp; elect.sync inside the _ws issue helpers
      const uint32_t idesc_dp = idesc_bf16_f32(TR, TK, 0, 0);  // dO (K-major) x V (K-major)
      const uint32_t idesc_kv = idesc_bf16_f32(TK, HD, 1, 1);  // P^T / dS^T (MN-major) x dO / Q (MN-major)
      const uint32_t va = smem_u32(smem + BK_OFF_V);
      Pos lq_a, dq_a, lq_b, dq_b;  // "a": dP/dV issue (runs one tile ahead), "b": dK issue
      uint32_t it = 0;
      for (int item = blockIdx.x; item < items; item += gridDim.x, ++it) {
        const uint32_t ab = it & 1;
        const uint32_t dv_col = ACC_COL + ab * 128, dk_col = dv_col + HD;
        mbar_wait(v_full, it & 1);
        mbar_wait(&acc_empty[ab], ((it >> 1) & 1) ^ 1);
        // dP(t) = dO V^T and dV += P^T dO need only the loaded stage; issuing
        // them one tile ahead of dK(t) (which waits for the epilogue's dS)
        // keeps the epilogue fed.
        auto issue_dp = [&](int t) {
          const uint32_t s = lq_a.slot(BK_ST), db = dq_a.slot(2);
          const uint32_t st = smem_u32(smem + BK_OFF_ST + s * BK_STAGE);
          const uint32_t doa = st, pa = st + 2 * TILE;
          mbar_wait(&ld_full[s], lq_a.phase(BK_ST));
          mbar_wait(&dp_empty[db], dq_a.phase(2) ^ 1);
          tc_fence_after();
#pragma unroll
          for (int k = 0; k < HD / 16; ++k)
            umma_bf16_ws(tmem + db * TK, smem_desc_sw128(doa + k * 32, 0, 1024), smem_desc_sw128(va + k * 32, 0, 1024),
                      idesc_dp, k > 0);
          if (t == T - 1) umma_commit_ws(v_empty);  // last read of V for this item
#pragma unroll
          for (int k = 0; k < TR / 16; ++k)
            umma_bf16_ws(tmem + dv_col, smem_desc_sw128(pa + k * 2048, ATOM, 1024),
                      smem_desc_sw128(doa + k * 2048, ATOM, 1024), idesc_kv, (t | k) != 0);
          // dp_full also certifies that P^T dO has finished reading P, so the
          // epilogue may overwrite P with dS in place.
          umma_commit_ws(&dp_full[db]);
          ++lq_a.i, ++dq_a.i;
        };
        if (T > 0) issue_dp(0);
        for (int t = 0; t < T; ++t) {
          if (t + 1 < T) issue_dp(t + 1);
          const uint32_t s = lq_b.slot(BK_ST), db = dq_b.slot(2);
          const uint32_t qa = smem_u32(smem + BK_OFF_ST + s * BK_STAGE) + TILE;
          const uint32_t dsa = qa + TILE;  // dS, written over P
          mbar_wait(&ds_full[db], dq_b.phase(2));
          tc_fence_after();
#pragma unroll
          for (int k = 0; k < TR / 16; ++k)
            umma_bf16_ws(tmem + dk_col, smem_desc_sw128(dsa + k * 2048, ATOM, 1024),
                      smem_desc_sw128(qa + k * 2048, ATOM, 1024), idesc_kv, (t | k) != 0);
          umma_commit_ws(&ld_empty[s]);
          ++lq_b.i, ++dq_b.i;
        }
        umma_commit_ws(&acc_full[ab]);
      }
    }
  } else {
    const uint32_t quad = warp & 3;
    const int half = (warp - 2) >> 2;
    const int r = quad * 32 + lane;
    const uint32_t lane_base = (quad * 32u) << 16;
    Pos lq, dq_;
    uint32_t it = 0;
    for (int item = blockIdx.x; item < items; item += gridDim.x, ++it) {
      const int kt = item % ntk, bz = (item / ntk) % BZ, jo = item / (ntk * BZ);
      const int b = bz / g.Z, z = bz % g.Z, k0 = kt * TK;
      int d = 0, r0 = 0;
      float dnext = r < g.c ? p.dvec[(int64_t(b) * g.Z + z) * g.c + r] : 0.f;
      for (int t = 0; t < T; ++t) {
        const uint32_t s = lq.slot(BK_ST), db = dq_.slot(2);
        const float dval = dnext;
        if (r0 + TR >= g.c) r0 = 0, ++d;
        else r0 += TR;
        if (t + 1 < T) {  // next step's D now: its load latency hides behind this step
          const int nrow = r0 + r;
          dnext = nrow < g.c ? p.dvec[(int64_t(d * g.B + b) * g.Z + z) * g.c + nrow] : 0.f;
        }
        const uint32_t pt = smem_u32(smem + BK_OFF_ST + s * BK_STAGE + 2 * TILE);
        const uint32_t dst = pt;  // dS overwrites P in place
        mbar_wait(&ld_full[s], lq.phase(BK_ST));
        mbar_wait(&dp_full[db], dq_.phase(2));
        tc_fence_after();
        const uint64_t nd = neg_pair(dval);
#pragma unroll
        for (int cc = 0; cc < 2; ++cc) {
          float v[32];
          const int col = half * 64 + cc * 32;
          __syncwarp();
          tmem_ld32(tmem + lane_base + db * TK + col, v);
          tmem_ld_wait();
          // dS' = P (dP - D) in place; the 1/sqrt(A) scale is applied to dK once, at the end
          ds_row32_inplace(dst, r, col, v, nd);
        }
        tc_fence_before();
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&dp_empty[db]);
          mbar_arrive(&ds_full[db]);
        }
        ++lq.i, ++dq_.i;
      }
      const uint32_t ab = it & 1;
      mbar_wait(&acc_full[ab], (it >> 1) & 1);
      tc_fence_after();
      float dvv[32], dkv[32];
      __syncwarp();
      tmem_ld32(tmem + lane_base + ACC_COL + ab * 128 + half * 32, dvv);
      tmem_ld32(tmem + lane_base + ACC_COL + ab * 128 + HD + half * 32, dkv);
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[ab]);
#pragma unroll
      for (int e = 0; e < 32; ++e) dkv[e] *= g.scale;
      const int key = k0 + r;
      if (key < g.c) {
        const OutView none{nullptr, 0, 0, 0, 0};
        if (p.dkv_bf16) {
          store_row32(none, p.dv, 0, jo, b, z, key, half * 32, dvv);
          store_row32(none, p.dk, 0, jo, b, z, key, half * 32, dkv);
        } else {
          store_row32(p.dv, none, p.accumulate, jo, b, z, key, half * 32, dvv);
          store_row32(p.dk, none, p.accumulate, jo, b, z, key, half * 32, dkv);
        }
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, 512);
}

// =================================================================== dQ

struct DqArgs {
  CUtensorMap tdo, tk, tv, tp;
  Geo g;
  const float* dvec;
  OutView dq_acc, dq_out;
  int accumulate;
};

constexpr int DQ_ST = 3;  // dS overwrites P inside the stage, as in bwd_dkdv
constexpr uint32_t DQ_STAGE = TILE /*V*/ + TILE /*K*/ + PTILE /*P, then dS*/;
constexpr uint32_t DQ_OFF_DO = 0;
constexpr uint32_t DQ_OFF_ST = 2 * TILE;
constexpr uint32_t DQ_OFF_BAR = DQ_OFF_ST + DQ_ST * DQ_STAGE;
constexpr uint32_t DQ_SMEM = DQ_OFF_BAR + 512 + 1024;

__global__ void __launch_bounds__(NTHREADS, 1) bwd_dq_kernel(const __grid_constant__ DqArgs p) {
  uint8_t* smem = smem_base();
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + DQ_OFF_BAR);
  uint64_t *do_full = bar, *do_empty = bar + 2, *ld_full = bar + 4, *ld_empty = ld_full + DQ_ST;
  uint64_t *dp_full = ld_empty + DQ_ST, *dp_empty = dp_full + 2, *ds_full = dp_empty + 2, *ds_empty = ds_full + 2;
  uint64_t *acc_full = ds_empty + 2, *acc_empty = acc_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

  const Geo& g = p.g;
  const int ntk = (g.c + TK - 1) / TK, nrt = (g.c + TR - 1) / TR;
  const int T = g.n_org * ntk;
  const int BZ = g.B * g.Z;
  const int items = g.n_rank * BZ * nrt;
  const uint32_t warp = warp_id(), lane = lane_id();
  constexpr uint32_t ACC_COL = 2 * TK;

  if (warp == 1) tmem_alloc(tmem_slot, 512);
  if (threadIdx.x == 0) {
    for (int s = 0; s < 2; ++s) {
      mbar_init(&do_full[s], 1), mbar_init(&do_empty[s], 1);
      mbar_init(&dp_full[s], 1), mbar_init(&dp_empty[s], EPI_WARPS);
      mbar_init(&ds_full[s], EPI_WARPS), mbar_init(&ds_empty[s], 1);
      mbar_init(&acc_full[s], 1), mbar_init(&acc_empty[s], EPI_WARPS);
    }
    for (int s = 0; s < DQ_ST; ++s) mbar_init(&ld_full[s], 1), mbar_init(&ld_empty[s], 1);
    fence_barrier_init();
    tma_prefetch(&p.tdo), tma_prefetch(&p.tk), tma_prefetch(&p.tv), tma_prefetch(&p.tp);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base(tmem_slot);

  if (warp == 0) {
    if (lane == 0) {
      Pos lq;
      uint32_t it = 0;
      const uint64_t pol = l2_evict_first();  // the panel streams through once
      for (int item = blockIdx.x; item < items; item += gridDim.x, ++it) {
        const int rt = item % nrt, bz = (item / nrt) % BZ, d = item / (nrt * BZ);
        const int b = bz / g.Z, z = bz % g.Z, r0 = rt * TR;
        const uint32_t ob = it & 1;
        mbar_wait(&do_empty[ob], ((it >> 1) & 1) ^ 1);
        mbar_arrive_expect_tx(&do_full[ob], TILE);
        tma_load_4d(smem + DQ_OFF_DO + ob * TILE, &p.tdo, &do_full[ob], 0, r0, z, d * g.B + b);
        for (int t = 0, jo = 0, k0 = 0; t < T; ++t, k0 = k0 + TK >= ntk * TK ? (++jo, 0) : k0 + TK) {
          const uint32_t s = lq.slot(DQ_ST);
          mbar_wait(&ld_empty[s], lq.phase(DQ_ST) ^ 1);
          mbar_arrive_expect_tx(&ld_full[s], DQ_STAGE);
          uint8_t* st = smem + DQ_OFF_ST + s * DQ_STAGE;
          tma_load_4d(st, &p.tv, &ld_full[s], 0, k0, z, jo * g.B + b);
          tma_load_4d(st + TILE, &p.tk, &ld_full[s], 0, k0, z, jo * g.B + b);
          tma_load_5d_hint(st + 2 * TILE, &p.tp, &ld_full[s], k0, g.org_lo + jo, r0, z, d * g.B + b, pol);
          tma_load_5d_hint(st + 2 * TILE + ATOM, &p.tp, &ld_full[s], k0 + 64, g.org_lo + jo, r0, z, d * g.B + b, pol);
          ++lq.i;
        }
      }
    }
  } else if (warp == 1) {
    {  // whole warp; elect.sync inside the _ws issue helpers
      const uint32_t idesc_dp = idesc_bf16_f32(TR, TK, 0, 0);  // dO x V^T
      const uint32_t idesc_dq = idesc_bf16_f32(TR, HD, 0, 1);  // dS (K-major over keys) x K (MN-major)
      Pos lq_a, dq_a, lq_b, dq_b;  // "a": dP issue (one tile ahead), "b": dQ issue
      uint32_t it = 0;
      for (int item = blockIdx.x; item < items; item += gridDim.x, ++it) {
        const uint32_t ob = it & 1;
        const uint32_t doa = smem_u32(smem + DQ_OFF_DO + ob * TILE);
        mbar_wait(&do_full[ob], (it >> 1) & 1);
        mbar_wait(&acc_empty[ob], ((it >> 1) & 1) ^ 1);
        auto issue_dp = [&](int t) {
          const uint32_t s = lq_a.slot(DQ_ST), db = dq_a.slot(2);
          const uint32_t va = smem_u32(smem + DQ_OFF_ST + s * DQ_STAGE);
          mbar_wait(&ld_full[s], lq_a.phase(DQ_ST));
          mbar_wait(&dp_empty[db], dq_a.phase(2) ^ 1);
          tc_fence_after();
#pragma unroll
          for (int k = 0; k < HD / 16; ++k)
            umma_bf16_ws(tmem + db * TK, smem_desc_sw128(doa + k * 32, 0, 1024), smem_desc_sw128(va + k * 32, 0, 1024),
                      idesc_dp, k > 0);
          umma_commit_ws(&dp_full[db]);
          if (t == T - 1) umma_commit_ws(&do_empty[ob]);
          ++lq_a.i, ++dq_a.i;
        };
        if (T > 0) issue_dp(0);
        for (int t = 0; t < T; ++t) {
          if (t + 1 < T) issue_dp(t + 1);
          const uint32_t s = lq_b.slot(DQ_ST), db = dq_b.slot(2);
          const uint32_t ka = smem_u32(smem + DQ_OFF_ST + s * DQ_STAGE) + TILE;
          const uint32_t dsa = ka + TILE;  // dS, written over P
          mbar_wait(&ds_full[db], dq_b.phase(2));
          tc_fence_after();
#pragma unroll
          for (int k = 0; k < TK / 16; ++k)
            umma_bf16_ws(tmem + ACC_COL + ob * HD, smem_desc_sw128(dsa + (k >> 2) * ATOM + (k & 3) * 32, 0, 1024),
                      smem_desc_sw128(ka + k * 2048, ATOM, 1024), idesc_dq, (t | k) != 0);
          umma_commit_ws(&ld_empty[s]);
          ++lq_b.i, ++dq_b.i;
        }
        umma_commit_ws(&acc_full[ob]);
      }
    }
  } else {
    const uint32_t quad = warp & 3;
    const int half = (warp - 2) >> 2;
    const int r = quad * 32 + lane;
    const uint32_t lane_base = (quad * 32u) << 16;
    Pos lq, dq_;
    uint32_t it = 0;
    for (int item = blockIdx.x; item < items; item += gridDim.x, ++it) {
      const int rt = item % nrt, bz = (item / nrt) % BZ, d = item / (nrt * BZ);
      const int b = bz / g.Z, z = bz % g.Z, row = rt * TR + r;
      const float dval = row < g.c ? p.dvec[(int64_t(d * g.B + b) * g.Z + z) * g.c + row] : 0.f;
      for (int t = 0; t < T; ++t) {
        const uint32_t s = lq.slot(DQ_ST), db = dq_.slot(2);
        const uint32_t pt = smem_u32(smem + DQ_OFF_ST + s * DQ_STAGE + 2 * TILE);
        const uint32_t dst = pt;  // dS overwrites P in place (no MMA reads this P tile)
        mbar_wait(&ld_full[s], lq.phase(DQ_ST));
        mbar_wait(&dp_full[db], dq_.phase(2));
        tc_fence_after();
        const uint64_t nd = neg_pair(dval);
#pragma unroll
        for (int cc = 0; cc < 2; ++cc) {
          float v[32];
          const int col = half * 64 + cc * 32;
          __syncwarp();
          tmem_ld32(tmem + lane_base + db * TK + col, v);
          tmem_ld_wait();
          ds_row32_inplace(dst, r, col, v, nd);  // dS' = P (dP - D); scale applied to dQ
        }
        tc_fence_before();
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          mbar_arrive(&dp_empty[db]);
          mbar_arrive(&ds_full[db]);
        }
        ++lq.i, ++dq_.i;
      }
      const uint32_t ob = it & 1;
      mbar_wait(&acc_full[ob], (it >> 1) & 1);
      tc_fence_after();
      float o[32];
      __syncwarp();
      tmem_ld32(tmem + lane_base + ACC_COL + ob * HD + half * 32, o);
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[ob]);
#pragma unroll
      for (int e = 0; e < 32; ++e) o[e] *= g.scale;
      if (row < g.c) store_row32(p.dq_acc, p.dq_out, p.accumulate, d, b, z, row, half * 32, o);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, 512);
}

// ================================================================== host

int fwd_launch(const rsa_geom* g, int mode, rsa_view q, rsa_view k, rsa_view v, float* stats, int slot, int n_slots,
               rsa_view panel, rsa_view o_acc, int accumulate, rsa_view o_out, int* flag, void* stream) {
  if (!geom_ok(g)) return fail(RSA_ERR_INVALID, "rsa_fwd: unsupported geometry");
  if ((mode & (MODE_WRITE_STATS | MODE_EXT_STATS)) && !stats) return fail(RSA_ERR_INVALID, "rsa_fwd: stats missing");
  if (!out_ok(o_acc, 4) || !out_ok(o_out, 2)) return fail(RSA_ERR_UNSUPPORTED, "rsa_fwd: output alignment");
  FwdArgs a{};
  if (!head_map(&a.tq, q, g, g->n_rank) || !head_map(&a.tk, k, g, g->n_org)) return RSA_ERR_UNSUPPORTED;
  if (mode & MODE_PASS_B) {
    if (!head_map(&a.tv, v, g, g->n_org) || !panel_map(&a.tp, panel, g, g->n_rank)) return RSA_ERR_UNSUPPORTED;
  }
  a.g = to_geo(g);
  a.mode = mode;
  a.sl = g->scale * LOG2E;
  a.stats = reinterpret_cast<float2*>(stats);
  a.slot = slot;
  a.n_slots = n_slots;
  a.slot_stride = int64_t(g->n_rank) * g->batch * g->heads * g->chunk;
  a.flag = flag;
  a.o_acc = to_out(o_acc);
  a.o_out = to_out(o_out);
  a.accumulate = accumulate;
  const int items = g->n_rank * g->batch * g->heads * ((g->chunk + TR - 1) / TR);
  return launch(fwd_kernel, items, F_SMEM, a, stream, "fwd_kernel");
}

}  // namespace
}  // namespace rsa

extern "C" {

int rsa_fused_supported(const rsa_geom* g) { return rsa::geom_ok(g) ? 1 : 0; }

int rsa_fwd_resident(const rsa_geom* g, rsa_view q, rsa_view k, rsa_view v, rsa_view panel, rsa_view o_out,
                     int* nonfinite_flag, void* stream) {
  using namespace rsa;
  const rsa_view none{nullptr, 0, 0, 0, 0};
  return fwd_launch(g, MODE_PASS_A | MODE_PASS_B, q, k, v, nullptr, 0, 0, panel, none, 0, o_out, nonfinite_flag,
                    stream);
}

int rsa_fwd_stats(const rsa_geom* g, rsa_view q, rsa_view k, float* stats, int slot, int* nonfinite_flag,
                  void* stream) {
  using namespace rsa;
  const rsa_view none{nullptr, 0, 0, 0, 0};
  if (slot < 0) return fail(RSA_ERR_INVALID, "rsa_fwd_stats: bad slot");
  return fwd_launch(g, MODE_PASS_A | MODE_WRITE_STATS, q, k, none, stats, slot, 0, none, none, 0, none,
                    nonfinite_flag, stream);
}

int rsa_fwd_probs_pv(const rsa_geom* g, rsa_view q, rsa_view k, rsa_view v, const float* stats, int n_slots,
                     rsa_view panel, rsa_view o_acc, int accumulate, rsa_view o_out, void* stream) {
  using namespace rsa;
  if (n_slots < 1) return fail(RSA_ERR_INVALID, "rsa_fwd_probs_pv: n_slots must be >= 1");
  return fwd_launch(g, MODE_PASS_B | MODE_EXT_STATS, q, k, v, const_cast<float*>(stats), 0, n_slots, panel, o_acc,
                    accumulate, o_out, nullptr, stream);
}

int rsa_bwd_dkdv(const rsa_geom* g, rsa_view q, rsa_view v, rsa_view dout, rsa_view panel, const float* dvec,
                 rsa_view dk, rsa_view dv, int dkv_dtype, int accumulate, void* stream) {
  using namespace rsa;
  if (!geom_ok(g) || !dvec) return fail(RSA_ERR_INVALID, "rsa_bwd_dkdv: unsupported geometry");
  const int esz = dkv_dtype == RSA_BF16 ? 2 : 4;
  if (!dk.ptr || !dv.ptr || !out_ok(dk, esz) || !out_ok(dv, esz))
    return fail(RSA_ERR_UNSUPPORTED, "rsa_bwd_dkdv: output alignment");
  DkdvArgs a{};
  if (!head_map(&a.tq, q, g, g->n_rank) || !head_map(&a.tdo, dout, g, g->n_rank) || !head_map(&a.tv, v, g, g->n_org) ||
      !panel_map(&a.tp, panel, g, g->n_rank))
    return RSA_ERR_UNSUPPORTED;
  a.g = to_geo(g);
  a.dvec = dvec;
  a.dk = to_out(dk);
  a.dv = to_out(dv);
  a.dkv_bf16 = dkv_dtype == RSA_BF16;
  a.accumulate = accumulate;
  const int items = g->n_org * g->batch * g->heads * ((g->chunk + TK - 1) / TK);
  return launch(bwd_dkdv_kernel, items, BK_SMEM, a, stream, "bwd_dkdv_kernel");
}

int rsa_bwd_dq(const rsa_geom* g, rsa_view dout, rsa_view k, rsa_view v, rsa_view panel, const float* dvec,
               rsa_view dq_acc, int accumulate, rsa_view dq_out, void* stream) {
  using namespace rsa;
  if (!geom_ok(g) || !dvec) return fail(RSA_ERR_INVALID, "rsa_bwd_dq: unsupported geometry");
  if (!out_ok(dq_acc, 4) || !out_ok(dq_out, 2)) return fail(RSA_ERR_UNSUPPORTED, "rsa_bwd_dq: output alignment");
  DqArgs a{};
  if (!head_map(&a.tdo, dout, g, g->n_rank) || !head_map(&a.tk, k, g, g->n_org) || !head_map(&a.tv, v, g, g->n_org) ||
      !panel_map(&a.tp, panel, g, g->n_rank))
    return RSA_ERR_UNSUPPORTED;
  a.g = to_geo(g);
  a.dvec = dvec;
  a.dq_acc = to_out(dq_acc);
  a.dq_out = to_out(dq_out);
  a.accumulate = accumulate;
  const int items = g->n_rank * g->batch * g->heads * ((g->chunk + TR - 1) / TR);
  return launch(bwd_dq_kernel, items, DQ_SMEM, a, stream, "bwd_dq_kernel");
}

}  // extern "C"

// Single-pass RSA backward for sm_100a (head size A = 64): dQ, dK and dV of a
// head from ONE read of its probability panel.
//
// Replaces the V-ring / K-ring pair of ringseq/ring_attention.py:168-209:
//   dP = dO V_j^T                       (V ring, :181-184)
//   dS = P (dP - rowsum(dP P)) scale    (:186-189; rowsum(dP P) = rowsum(dO O) = D, supplied)
//   dQ = sum_j dS_j K_j                 (K ring, :192-196)
//   dK_j = dS_j^T Q,  dV_j = P_j^T dO   (full-length partials, :198-205)
// for every (query tile, key tile) pair of one head inside one CTA, so the
// panel tile P(qt, kt) is loaded once and dS never leaves shared memory.
//
// A CTA owns a whole head (b, z): the outer loop walks key tiles kt (any
// number: all resident origins), the inner loop the head's query tiles qt
// (at most 4 -- n_rank * ceil(c / 128) <= 4, e.g. L <= 512 resident, or
// c <= 512 per ring hop).  TMEM (512 columns) holds
//   [  0,128)  dP of the current step
//   [128,192)  dV of the current key tile      (M = keys)
//   [192,256)  dK of the current key tile
//   [256,512)  dQ of each query tile, 64 columns per tile, live for the head
// so dK/dV are final when a key tile's inner loop ends and dQ when the last
// key tile has been applied -- every sum is accumulated in TMEM in a fixed
// order (deterministic, no atomics).
//
// Warp roles (10 warps): warp 0 TMA producer, warp 1 tcgen05.mma issuer
// (owns TMEM), warps 2..9 epilogue (warp w reads TMEM lanes 32*(w%4)..,
// column half (w-2)/4).  Rings: K, dO, Q tiles 2 deep each, V 1 deep, panel
// tiles 3 deep (the only HBM stream that matters; dO/Q re-reads are L2 hits).  dS overwrites P in place once P^T dO has consumed it.
#include <cstdio>
#include <cstdlib>
#include <cstring>

#include "fused_common.cuh"

namespace rsa {
namespace {

constexpr int MAX_QT = 4;  // query tiles per head that fit the dQ columns of TMEM

struct BwdArgs {
  CUtensorMap tq, tk, tv, tdo, tp, tdk, tdv, tdq;
  int dq_tma;  // bf16 dQ only: each query tile staged (BF_OFF_DQS) and TMA-stored
  int kv_tma;  // bf16, non-accumulating dK/dV: staged in the retiring P slot and TMA-stored
  int peer;    // K / V of origin j from pm.k[j] / pm.v[j] (rsa_bwd_fused_peer)
  PeerMaps pm;
  Geo g;
  const float* dvec;
  OutView dq_acc, dq_out, dk, dv;
  int accumulate_dq;
  int dkv_bf16;
  int accumulate_dkv;
  long long* trace;  // RSA_BF_TRACE: per-warp (event, clock) log of CTA 0 (timeline experiments)
};

#define BF_TRACE(ev)                                                                                          \
  do {                                                                                                        \
    if (p.trace && blockIdx.x == 0 && (threadIdx.x & 31) == 0 && tr_i < 4095)                                 \
      p.trace[(threadIdx.x >> 5) * 4096 + tr_i++] = ((long long)(ev) << 48) | (long long)(clock64() - tr0); \
  } while (0)

// Ring depths.  Each operand is released as soon as its last MMA has read it
// (dO after P^T dO, V after the key tile's last dO V^T, Q / P / K after the
// dS products), so the producer runs 1-2 steps ahead of the tensor pipe.
#ifndef BF_RDO  // ring depths (experiments: -DBF_RDO=.. -DBF_RQ=.. -DBF_RP=.. -DBF_RK=.. -DBF_RV=..)
#define BF_RDO 2
#endif
#ifndef BF_RQ
#define BF_RQ 2
#endif
#ifndef BF_RP
#define BF_RP 3
#endif
#ifndef BF_RK
#define BF_RK 2
#endif
#ifndef BF_RV
#define BF_RV 1  // one V tile: V is read by one product per step (dO V^T), and a second slot measured +-0
#endif
constexpr int BF_DO = BF_RDO, BF_Q = BF_RQ, BF_P = BF_RP, BF_K = BF_RK, BF_V = BF_RV;
constexpr uint32_t BF_OFF_DO = 0;
constexpr uint32_t BF_OFF_Q = BF_OFF_DO + BF_DO * TILE;
constexpr uint32_t BF_OFF_K = BF_OFF_Q + BF_Q * TILE;
constexpr uint32_t BF_OFF_V = BF_OFF_K + BF_K * TILE;
constexpr uint32_t BF_OFF_P = BF_OFF_V + BF_V * TILE;  // [slot] P, then dS in place
constexpr uint32_t BF_OFF_DQS = BF_OFF_P + BF_P * PTILE;  // dQ staging: 2 KB per epilogue warp (32 x 32 bf16, SWIZZLE_64B)
constexpr uint32_t BF_OFF_BAR = BF_OFF_DQS + TILE;
constexpr uint32_t BF_SMEM = BF_OFF_BAR + 512 + 1024;
static_assert(BF_SMEM <= 232448, "bwd_fused smem over the sm_100 per-CTA limit");

constexpr uint32_t COL_DP = 0, COL_DV = 128, COL_DK = 192, COL_DQ = 256;

struct Ring {  // full/empty barrier pair array of one operand ring
  uint64_t *full, *empty;
};

__global__ void __launch_bounds__(NTHREADS, 1) bwd_fused_kernel(const __grid_constant__ BwdArgs p) {
  uint8_t* smem = smem_base();
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + BF_OFF_BAR);
  const Ring rdo{bar, bar + BF_DO};
  const Ring rq{rdo.empty + BF_DO, rdo.empty + BF_DO + BF_Q};
  const Ring rk{rq.empty + BF_Q, rq.empty + BF_Q + BF_K};
  const Ring rv{rk.empty + BF_K, rk.empty + BF_K + BF_V};
  const Ring rp{rv.empty + BF_V, rv.empty + BF_V + BF_P};
  uint64_t* ds_full = rp.empty + BF_P;
  uint64_t* p_read = ds_full + BF_P;  // P^T dO has consumed the P slot (dS may overwrite it)
  uint64_t *dp_full = p_read + BF_P, *dp_empty = dp_full + 1, *acc_full = dp_empty + 1, *acc_empty = acc_full + 1;
  uint64_t *dq_full = acc_empty + 1, *dq_empty = dq_full + MAX_QT;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(dq_empty + MAX_QT);

  const Geo& g = p.g;
  const int nrt = (g.c + TR - 1) / TR, ntk = (g.c + TK - 1) / TK;
  const int NQ = g.n_rank * nrt;  // query tiles of a head (<= MAX_QT)
  const int NK = g.n_org * ntk;   // key tiles of a head
  const int T = NQ * NK;
  const int items = g.B * g.Z;
  const uint32_t warp = warp_id(), lane = lane_id();

  if (warp == 1) tmem_alloc(tmem_slot, 512);
  if (threadIdx.x == 0) {
    auto init = [](const Ring& r, int n) {
      for (int s = 0; s < n; ++s) mbar_init(&r.full[s], 1), mbar_init(&r.empty[s], 1);
    };
    init(rdo, BF_DO), init(rq, BF_Q), init(rk, BF_K), init(rv, BF_V), init(rp, BF_P);
    for (int s = 0; s < BF_P; ++s) mbar_init(&ds_full[s], EPI_WARPS), mbar_init(&p_read[s], 1);
    mbar_init(dp_full, 1), mbar_init(dp_empty, EPI_WARPS);
    mbar_init(acc_full, 1), mbar_init(acc_empty, EPI_WARPS);
    for (int s = 0; s < MAX_QT; ++s) mbar_init(&dq_full[s], 1), mbar_init(&dq_empty[s], EPI_WARPS);
    fence_barrier_init();
    tma_prefetch(&p.tq), tma_prefetch(&p.tk), tma_prefetch(&p.tv), tma_prefetch(&p.tdo), tma_prefetch(&p.tp);
    if (p.kv_tma) tma_prefetch(&p.tdk), tma_prefetch(&p.tdv);
    if (p.dq_tma) tma_prefetch(&p.tdq);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base(tmem_slot);
  const long long tr0 = clock64();
  int tr_i = 0;

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      const uint64_t pol = l2_evict_first();
      Pos dq_, qq, kq, vq, pq;
      // one 16 KB head tile (rows r0.. of rank/origin `blk`) into ring slot
      auto load_tile = [&](const Ring& r, Pos& pos, int depth, uint32_t off, const CUtensorMap* map, int r0, int z,
                           int blk) {
        const uint32_t s = pos.slot(depth);
        mbar_wait(&r.empty[s], pos.phase(depth) ^ 1);
        mbar_arrive_expect_tx(&r.full[s], TILE);
        tma_load_4d(smem + off + s * TILE, map, &r.full[s], 0, r0, z, blk);
        ++pos.i;
      };
      // V and K tiles of (head item, key tile kk); issued one key tile ahead of use
      auto load_vk = [&](int item, int kk) {
        const int b = item / g.Z, z = item % g.Z;
        const int jo = kk / ntk, k0 = (kk % ntk) * TK;
        load_tile(rv, vq, BF_V, BF_OFF_V, p.peer ? &p.pm.v[jo] : &p.tv, k0, z, p.peer ? b : jo * g.B + b);
        load_tile(rk, kq, BF_K, BF_OFF_K, p.peer ? &p.pm.k[jo] : &p.tk, k0, z, p.peer ? b : jo * g.B + b);
      };
      if (blockIdx.x < items) load_vk(blockIdx.x, 0);
      for (int item = blockIdx.x; item < items; item += gridDim.x) {
        const int b = item / g.Z, z = item % g.Z;
        // (origin, key offset) and (rank, row offset) advance by counters: no integer
        // division by a runtime count in any per-step path
        for (int kk = 0, jo = 0, k0 = 0; kk < NK; ++kk, k0 = k0 + TK >= ntk * TK ? (++jo, 0) : k0 + TK) {
          for (int qt = 0, d = 0, r0 = 0; qt < NQ; ++qt, r0 = r0 + TR >= nrt * TR ? (++d, 0) : r0 + TR) {
            load_tile(rdo, dq_, BF_DO, BF_OFF_DO, &p.tdo, r0, z, d * g.B + b);
            const uint32_t s = pq.slot(BF_P);
            mbar_wait(&rp.empty[s], pq.phase(BF_P) ^ 1);
            mbar_arrive_expect_tx(&rp.full[s], PTILE);
            uint8_t* pt = smem + BF_OFF_P + s * PTILE;
            // the panel streams through once: evict it first, keep dO / Q / K / V tiles in L2
            tma_load_5d_hint(pt, &p.tp, &rp.full[s], k0, g.org_lo + jo, r0, z, d * g.B + b, pol);
            tma_load_5d_hint(pt + ATOM, &p.tp, &rp.full[s], k0 + 64, g.org_lo + jo, r0, z, d * g.B + b, pol);
            BF_TRACE(1);
            ++pq.i;
            load_tile(rq, qq, BF_Q, BF_OFF_Q, &p.tq, r0, z, d * g.B + b);
            // the next key tile's V / K after this key tile's last step: their slots (key tile
            // kk - 1) have retired by now, and they arrive a step earlier than in step order
            if (qt == NQ - 1) {
              if (kk + 1 < NK) load_vk(item, kk + 1);
              else if (item + int(gridDim.x) < items) load_vk(item + gridDim.x, 0);
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------- MMA issuer
    // The whole warp runs this loop (warp-uniform state); elect.sync inside
    // umma_bf16_ws / umma_commit_ws picks the issuing lane.
    {
      const uint32_t idesc_dp = idesc_bf16_f32(TR, TK, 0, 0);  // dO (K-major) x V (K-major)     -> 128 x 128
      const uint32_t idesc_kv = idesc_bf16_f32(TK, HD, 1, 1);  // P^T / dS^T (MN) x dO / Q (MN) -> 128 x 64
      const uint32_t idesc_dq = idesc_bf16_f32(TR, HD, 0, 1);  // dS (K-major) x K (MN-major)   -> 128 x 64
      Pos v_a, do_a, p_a, k_b, q_b, p_b, dpq, accq;
      uint32_t head_it = 0;
      for (int item = blockIdx.x; item < items; item += gridDim.x, ++head_it) {
        // dP(t) = dO V^T into the single dP buffer (after the epilogue has read dP(t-1))
        auto issue_dp = [&](int qt) {
          const uint32_t vs = v_a.slot(BF_V), ds = do_a.slot(BF_DO);
          if (qt == 0) mbar_wait(&rv.full[vs], v_a.phase(BF_V));
          mbar_wait(&rdo.full[ds], do_a.phase(BF_DO));
          mbar_wait(dp_empty, dpq.phase(1) ^ 1);
          tc_fence_after();
          const uint64_t da = smem_desc_sw128(smem_u32(smem + BF_OFF_DO + ds * TILE), 0, 1024);
          const uint64_t db = smem_desc_sw128(smem_u32(smem + BF_OFF_V + vs * TILE), 0, 1024);
          umma_ss_x4<2, 2>(tmem + COL_DP, da, db, idesc_dp, 0);  // K-major: +32 B per 16-wide k step
          if (qt == NQ - 1) {
            umma_commit_ws(&rv.empty[vs]);
            ++v_a.i;
          }
          umma_commit_ws(dp_full);
          BF_TRACE(10);
          ++dpq.i;
        };
        // dV += P^T dO; p_read certifies P has been consumed, so dS may overwrite it
        auto issue_dv = [&](int qt) {
          const uint32_t ds = do_a.slot(BF_DO), ps = p_a.slot(BF_P);
          if (qt == 0) mbar_wait(acc_empty, accq.phase(1) ^ 1);
          mbar_wait(&rp.full[ps], p_a.phase(BF_P));
          tc_fence_after();
          const uint64_t da = smem_desc_sw128(smem_u32(smem + BF_OFF_P + ps * PTILE), ATOM, 1024);
          const uint64_t db = smem_desc_sw128(smem_u32(smem + BF_OFF_DO + ds * TILE), ATOM, 1024);
          umma_ss_x4<128, 128>(tmem + COL_DV, da, db, idesc_kv, qt != 0);  // MN-major: +16 rows (2048 B) per k step
          umma_ss_x4<128, 128>(tmem + COL_DV, da + 512, db + 512, idesc_kv, 1);
          umma_commit_ws(&rdo.empty[ds]);
          umma_commit_ws(&p_read[ps]);
          BF_TRACE(11);
          ++do_a.i, ++p_a.i;
          if (qt == NQ - 1) ++accq.i;
        };
        // dK += dS^T Q and dQ(qt) += dS K once the epilogue has written dS(t)
        auto issue_b = [&](int kk, int qt) {
          const uint32_t ks = k_b.slot(BF_K), qs = q_b.slot(BF_Q), ps = p_b.slot(BF_P);
          if (qt == 0) mbar_wait(&rk.full[ks], k_b.phase(BF_K));
          mbar_wait(&rq.full[qs], q_b.phase(BF_Q));
          mbar_wait(&ds_full[ps], p_b.phase(BF_P));
          tc_fence_after();
          const uint32_t dsa = smem_u32(smem + BF_OFF_P + ps * PTILE);
          const uint64_t dmn = smem_desc_sw128(dsa, ATOM, 1024);  // dS^T: MN-major A
          const uint64_t dkm = smem_desc_sw128(dsa, 0, 1024);     // dS: K-major A
          const uint64_t qd = smem_desc_sw128(smem_u32(smem + BF_OFF_Q + qs * TILE), ATOM, 1024);
          const uint64_t kd = smem_desc_sw128(smem_u32(smem + BF_OFF_K + ks * TILE), ATOM, 1024);
          umma_ss_x4<128, 128>(tmem + COL_DK, dmn, qd, idesc_kv, qt != 0);
          umma_ss_x4<128, 128>(tmem + COL_DK, dmn + 512, qd + 512, idesc_kv, 1);
          if (kk == 0) {
            mbar_wait(&dq_empty[qt], (head_it & 1) ^ 1);
            tc_fence_after();
          }
          // dS K-major over keys: 64-key atoms ATOM apart, +32 B per k
          umma_ss_x4<2, 128>(tmem + COL_DQ + qt * HD, dkm, kd, idesc_dq, kk != 0);
          umma_ss_x4<2, 128>(tmem + COL_DQ + qt * HD, dkm + (ATOM >> 4), kd + 512, idesc_dq, 1);
          if (!(p.kv_tma && qt == NQ - 1)) umma_commit_ws(&rp.empty[ps]);  // else the epilogue frees it
          umma_commit_ws(&rq.empty[qs]);
          if (qt == NQ - 1) {
            umma_commit_ws(acc_full);
            umma_commit_ws(&rk.empty[ks]);
            ++k_b.i;
          }
          if (kk == NK - 1) umma_commit_ws(&dq_full[qt]);
          BF_TRACE(12);
          ++q_b.i, ++p_b.i;
        };
        issue_dp(0);
        issue_dv(0);
        for (int t = 0, kk = 0, qt = 0; t < T; ++t) {
          const bool next = t + 1 < T;
          const int nqt = qt + 1 == NQ ? 0 : qt + 1;
          const bool new_kt = next && nqt == 0;
          if (next && !new_kt) issue_dp(nqt), issue_dv(nqt);
          issue_b(kk, qt);
          // key-tile boundary: the finished tile's dK products go first, so the epilogue's
          // dK/dV readout (which frees the accumulators for the next dV) waits the least
          if (new_kt) issue_dp(nqt), issue_dv(nqt);
          kk += nqt == 0, qt = nqt;
        }
      }
    }
  } else {
    // ------------------------------------------------------------ epilogue
    // Readouts of finished accumulators are deferred by one step: a key
    // tile's dK/dV are read while the next step's dS is in registers (before
    // its P slot is overwritten, since the next P^T dO waits for them), and a
    // query tile's dQ after the next step's dS is stored.  So the epilogue
    // never waits on the MMAs its own dS has just enabled.
    const uint32_t quad = warp & 3;
    const int half = (warp - 2) >> 2;
    const int r = quad * 32 + lane;
    const uint32_t lane_base = (quad * 32u) << 16;
    Pos pq, dpq, accq;
    uint32_t head_it = 0;
    // pending readouts: key tile (jo, k0) of head (kb, kz); query tile qqt of head (qb, qz)
    bool kv_on = false, q_on = false;
    uint32_t kslot = 0;  // P slot of the pending key tile's last step
    bool rel_pending = false;
    uint32_t rel_slot = 0;
    int kjo = 0, kk0 = 0, kb = 0, kz = 0, qqt = 0, qd = 0, qrow = 0, qb = 0, qz = 0;
    uint32_t qphase = 0;
    auto read_kv = [&](float* dvv, float* dkv) {
      mbar_wait(acc_full, accq.phase(1));
      tc_fence_after();
      __syncwarp();
      tmem_ld32(tmem + lane_base + COL_DV + half * 32, dvv);
      tmem_ld32(tmem + lane_base + COL_DK + half * 32, dkv);
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(acc_empty);
      ++accq.i;
    };
    auto store_kv = [&](float* dvv, float* dkv) {
#pragma unroll
      for (int e = 0; e < 32; ++e) dkv[e] *= g.scale;
      if (p.kv_tma) {
        // dV -> atom 0, dK -> atom 1 of the key tile's last P slot (its products are done:
        // read_kv waited for them), two TMA stores, then the slot goes back to the producer
        const uint32_t st = smem_u32(smem + BF_OFF_P + kslot * PTILE);
        st_row32_sw128(st, r, half * 32, dvv);
        st_row32_sw128(st, r, 64 + half * 32, dkv);
        fence_proxy_async_smem();
        bar_epi();
        if (threadIdx.x == 64) {
          tma_store_4d(&p.tdv, smem + BF_OFF_P + kslot * PTILE, 0, kk0, kz, kjo * g.B + kb);
          tma_store_4d(&p.tdk, smem + BF_OFF_P + kslot * PTILE + ATOM, 0, kk0, kz, kjo * g.B + kb);
          tma_store_commit();
        }
        rel_pending = true, rel_slot = kslot;  // slot returns to the producer once the stores have read it
        kv_on = false;
        return;
      }
      const int key = kk0 + r;
      if (key < g.c) {
        const OutView none{nullptr, 0, 0, 0, 0};
        if (p.dkv_bf16) {
          store_row32(none, p.dv, 0, kjo, kb, kz, key, half * 32, dvv);
          store_row32(none, p.dk, 0, kjo, kb, kz, key, half * 32, dkv);
        } else {
          store_row32(p.dv, none, p.accumulate_dkv, kjo, kb, kz, key, half * 32, dvv);
          store_row32(p.dk, none, p.accumulate_dkv, kjo, kb, kz, key, half * 32, dkv);
        }
      }
      kv_on = false;
    };
    auto flush_q = [&]() {
      float o[32];
      mbar_wait(&dq_full[qqt], qphase);
      tc_fence_after();
      __syncwarp();
      tmem_ld32(tmem + lane_base + COL_DQ + qqt * HD + half * 32, o);
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&dq_empty[qqt]);
#pragma unroll
      for (int e = 0; e < 32; ++e) o[e] *= g.scale;
      q_on = false;
      if (p.dq_tma) {  // this warp's 32 rows x 32 columns through its own 2 KB of staging: one TMA store
        uint8_t* stg = smem + BF_OFF_DQS + (warp - 2) * 2048;
        const uint32_t srow = smem_u32(stg) + lane * 64, sw = (lane >> 1) & 3;
        if (lane == 0) tma_store_wait_read<0>();  // this warp's previous dQ store has read it
        __syncwarp();
#pragma unroll
        for (int j = 0; j < 4; ++j)
          st_shared_v4(srow + ((j ^ sw) << 4), pack_bf16(o[8 * j], o[8 * j + 1]), pack_bf16(o[8 * j + 2], o[8 * j + 3]),
                       pack_bf16(o[8 * j + 4], o[8 * j + 5]), pack_bf16(o[8 * j + 6], o[8 * j + 7]));
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          tma_store_4d(&p.tdq, stg, half * 32, qrow - int(lane), qz, qd * g.B + qb);
          tma_store_commit();
        }
        return;
      }
      if (qrow < g.c) store_row32(p.dq_acc, p.dq_out, p.accumulate_dq, qd, qb, qz, qrow, half * 32, o);
    };
    auto load_d = [&](int it, float* out) {  // D of this thread's rows of head `it`
      const int hb = it / g.Z, hz = it % g.Z;
#pragma unroll
      for (int j = 0; j < MAX_QT; ++j) {
        const int rj = (j % nrt) * TR + r;
        out[j] = (it < items && j < NQ && rj < g.c)
                     ? __ldg(p.dvec + (int64_t((j / nrt) * g.B + hb) * g.Z + hz) * g.c + rj)
                     : 0.f;
      }
    };
    float dn[MAX_QT];
    load_d(blockIdx.x, dn);
    for (int item = blockIdx.x; item < items; item += gridDim.x, ++head_it) {
      const int b = item / g.Z, z = item % g.Z;
      // D of this thread's row in each query tile of the head: loaded once per head (every
      // key tile revisits the same rows), and a whole head ahead, so its load latency never
      // sits at a head boundary
      float dh[MAX_QT];
#pragma unroll
      for (int j = 0; j < MAX_QT; ++j) dh[j] = dn[j];
      load_d(item + int(gridDim.x), dn);
      for (int t = 0, kk = 0, qt = 0, d = 0, r0 = 0, jo = 0, k0 = 0; t < T; ++t) {
        const int row = r0 + r;
        const float dval = qt == 0 ? dh[0] : qt == 1 ? dh[1] : qt == 2 ? dh[2] : dh[3];
        const uint32_t ps = pq.slot(BF_P);
        const uint32_t pt = smem_u32(smem + BF_OFF_P + ps * PTILE);
        BF_TRACE(20);
        if (kv_on) {  // the finished key tile's dK / dV first: frees the accumulators for this step's P^T dO
          float dvv[32], dkv[32];
          read_kv(dvv, dkv);
          store_kv(dvv, dkv);
        }
        float dp[64];
        mbar_wait(&rp.full[ps], pq.phase(BF_P));
        BF_TRACE(21);
        mbar_wait(dp_full, dpq.phase(1));
        BF_TRACE(22);
        tc_fence_after();
        __syncwarp();
        tmem_ld32(tmem + lane_base + COL_DP + half * 64, dp);
        tmem_ld32(tmem + lane_base + COL_DP + half * 64 + 32, dp + 32);
        tmem_ld_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(dp_empty);
        ++dpq.i;
        // dS' = P (dP - D) as packed bf16 (the 1/sqrt(A) scale is applied to dQ / dK at the end)
        uint32_t dsw[32];
        uint64_t nd;
        asm("mov.b64 %0, {%1, %1};" : "=l"(nd) : "f"(-dval));
#pragma unroll
        for (int cc = 0; cc < 2; ++cc) {
          const uint32_t atom = (half * 64 + cc * 32) >> 6, chunk0 = ((half * 64 + cc * 32) & 63) >> 3;
#pragma unroll
          for (int q4 = 0; q4 < 4; ++q4) {
            uint32_t w[4];
            ld_shared_v4(pt + atom * ATOM + sw128_offset(r, chunk0 + q4), w[0], w[1], w[2], w[3]);
#pragma unroll
            for (int e = 0; e < 4; ++e)
              dsw[cc * 16 + q4 * 4 + e] = ds_pair(w[e], dp[cc * 32 + q4 * 8 + 2 * e], dp[cc * 32 + q4 * 8 + 2 * e + 1], nd);
          }
        }
        BF_TRACE(23);
        mbar_wait(&p_read[ps], pq.phase(BF_P));
        BF_TRACE(24);
#pragma unroll
        for (int cc = 0; cc < 2; ++cc) {
          const uint32_t atom = (half * 64 + cc * 32) >> 6, chunk0 = ((half * 64 + cc * 32) & 63) >> 3;
#pragma unroll
          for (int q4 = 0; q4 < 4; ++q4)
            st_shared_v4(pt + atom * ATOM + sw128_offset(r, chunk0 + q4), dsw[cc * 16 + q4 * 4],
                         dsw[cc * 16 + q4 * 4 + 1], dsw[cc * 16 + q4 * 4 + 2], dsw[cc * 16 + q4 * 4 + 3]);
        }
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) mbar_arrive(&ds_full[ps]);
        BF_TRACE(25);
        ++pq.i;
        if (rel_pending) {
          if (threadIdx.x == 64) tma_store_wait_read<0>(), mbar_arrive(&rp.empty[rel_slot]);
          rel_pending = false;
        }
        if (q_on) flush_q();
        if (qt == NQ - 1) kv_on = true, kjo = jo, kk0 = k0, kb = b, kz = z, kslot = ps;
        if (kk == NK - 1) q_on = true, qqt = qt, qd = d, qrow = row, qb = b, qz = z, qphase = head_it & 1;
        if (++qt == NQ) {  // advance (query tile, rank, row) and, after the last query tile, the key tile
          qt = 0, d = 0, r0 = 0, ++kk;
          if (k0 + TK >= ntk * TK) k0 = 0, ++jo;
          else k0 += TK;
        } else if (r0 + TR >= nrt * TR) {
          r0 = 0, ++d;
        } else {
          r0 += TR;
        }
      }
    }
    if (kv_on) {
      float dvv[32], dkv[32];
      read_kv(dvv, dkv);
      store_kv(dvv, dkv);
    }
    if (rel_pending && threadIdx.x == 64) mbar_arrive(&rp.empty[rel_slot]);
    if (p.kv_tma && threadIdx.x == 64) tma_store_wait_all<0>();
    if (q_on) flush_q();
    if (p.dq_tma && lane == 0) tma_store_wait_all<0>();  // this warp's dQ stores have left shared memory
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, 512);
}

bool bwd_fused_geom_ok(const rsa_geom* g) {
  return geom_ok(g) && g->n_rank * ((g->chunk + TR - 1) / TR) <= MAX_QT;
}

}  // namespace
}  // namespace rsa

extern "C" {

int rsa_bwd_fused_supported(const rsa_geom* g) { return rsa::bwd_fused_geom_ok(g) ? 1 : 0; }

int rsa_bwd_fused(const rsa_geom* g, rsa_view q, rsa_view k, rsa_view v, rsa_view dout, rsa_view panel,
                  const float* dvec, rsa_view dq_acc, int accumulate_dq, rsa_view dq_out, rsa_view dk, rsa_view dv,
                  int dkv_dtype, int accumulate_dkv, void* stream) {
  using namespace rsa;
  if (!bwd_fused_geom_ok(g) || !dvec)
    return fail(RSA_ERR_INVALID, "rsa_bwd_fused: unsupported geometry (need A=64, c%%8==0, n_rank*ceil(c/128)<=4)");
  const int esz = dkv_dtype == RSA_BF16 ? 2 : 4;
  if (!dk.ptr || !dv.ptr || !out_ok(dk, esz) || !out_ok(dv, esz) || !out_ok(dq_acc, 4) || !out_ok(dq_out, 2) ||
      (!dq_acc.ptr && !dq_out.ptr))
    return fail(RSA_ERR_UNSUPPORTED, "rsa_bwd_fused: output views missing or misaligned");
  BwdArgs a{};
  if (!head_map(&a.tq, q, g, g->n_rank) || !head_map(&a.tdo, dout, g, g->n_rank) ||
      !head_map(&a.tk, k, g, g->n_org) || !head_map(&a.tv, v, g, g->n_org) || !panel_map(&a.tp, panel, g, g->n_rank))
    return RSA_ERR_UNSUPPORTED;
  a.g = to_geo(g);
  a.dvec = dvec;
  a.dq_acc = to_out(dq_acc);
  a.dq_out = to_out(dq_out);
  a.dk = to_out(dk);
  a.dv = to_out(dv);
  a.accumulate_dq = accumulate_dq;
  a.dkv_bf16 = dkv_dtype == RSA_BF16;
  a.accumulate_dkv = accumulate_dkv;
  a.kv_tma = dkv_dtype == RSA_BF16 && head_map(&a.tdk, dk, g, g->n_org) && head_map(&a.tdv, dv, g, g->n_org);
  // (the layouts head_map_w32 accepts, checked first so a fallback leaves no error message)
  a.dq_tma = !dq_acc.ptr && dq_out.ptr &&
             !(g->n_rank > 1 && g->batch > 1 && dq_out.s_rank != int64_t(g->batch) * dq_out.s_b) &&
             head_map_w32(&a.tdq, dq_out, g, g->n_rank);
  static long long* trace_buf = nullptr;
  const char* trace_path = getenv("RSA_BF_TRACE");
  if (trace_path) {
    if (!trace_buf) cudaMalloc(&trace_buf, 10 * 4096 * sizeof(long long));
    cudaMemset(trace_buf, 0, 10 * 4096 * sizeof(long long));
    a.trace = trace_buf;
  }
  const int rc = launch(bwd_fused_kernel, g->batch * g->heads, BF_SMEM, a, stream, "bwd_fused_kernel");
  if (trace_path) {
    static long long host[10 * 4096];
    cudaMemcpy(host, trace_buf, sizeof(host), cudaMemcpyDeviceToHost);
    if (FILE* f = fopen(trace_path, "wb")) fwrite(host, sizeof(host), 1, f), fclose(f);
  }
  return rc;
}

int rsa_bwd_fused_peer(const rsa_geom* g, rsa_view q, const rsa_view* k_origin, const rsa_view* v_origin,
                       rsa_view dout, rsa_view panel, const float* dvec, rsa_view dq_out, rsa_view dk_part,
                       rsa_view dv_part, void* stream) {
  using namespace rsa;
  if (!bwd_fused_geom_ok(g) || !dvec || !k_origin || !v_origin)
    return fail(RSA_ERR_INVALID, "rsa_bwd_fused_peer: unsupported geometry (need A=64, c%%8==0, ceil(c/128)<=4)");
  if (g->n_rank != 1 || g->org_lo != 0 || g->n_org != g->seq_len / g->chunk)
    return fail(RSA_ERR_INVALID, "rsa_bwd_fused_peer: need n_rank = 1, org_lo = 0, n_org = L / c");
  if (!dk_part.ptr || !dv_part.ptr || !out_ok(dk_part, 4) || !out_ok(dv_part, 4) || !dq_out.ptr || !out_ok(dq_out, 2))
    return fail(RSA_ERR_UNSUPPORTED, "rsa_bwd_fused_peer: output views missing or misaligned");
  BwdArgs a{};
  a.peer = 1;
  if (!peer_maps(&a.pm, k_origin, v_origin, g) || !head_map(&a.tq, q, g, 1) || !head_map(&a.tdo, dout, g, 1) ||
      !panel_map(&a.tp, panel, g, 1))
    return RSA_ERR_UNSUPPORTED;
  a.g = to_geo(g);
  a.dvec = dvec;
  a.dq_out = to_out(dq_out);
  a.dk = to_out(dk_part);
  a.dv = to_out(dv_part);
  a.dkv_bf16 = 0;  // fp32 partials of every origin, reduce-scattered by the caller
  return launch(bwd_fused_kernel, g->batch * g->heads, BF_SMEM, a, stream, "bwd_fused_kernel");
}

}  // extern "C"

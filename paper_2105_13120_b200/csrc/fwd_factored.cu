// Factored-panel RSA forward for sm_100a (head size A = 64, every origin
// resident), ONE pass over the scores: the probability panel is saved as
//   P~[row, k] = 2^(s*sl - m_ref[row])   (bf16),   r[row] = 1 / sum_k P~[row, k]   (fp32)
// so the reference's probs are P = r * P~ (ringseq/ring_attention.py:89-94,
// ringseq/tensor_ops.py:75-84) and its output is O = P V = r * (P~ V)
// (ringseq/ring_attention.py:97-103).  sl = scale * log2(e).
//
// Why factored and single-pass.  A normalised panel needs the full row max
// AND sum before the first probability can be written, i.e. a second pass
// over S = Q K^T: another GEMM, another tcgen05.ld of every fp32 score (a
// per-warp latency chain: tools/membench/tmem_ld measures 53 B/clk per SM for
// 4 warps with one load in flight, 467 B/clk for 16 warps with four) and
// another exp2 per element.  Softmax is invariant to
// the reference point, so any per-row m_ref works as long as 2^(s*sl - m_ref)
// neither overflows nor flushes the row: here m_ref is the max of the row's
// FIRST key tile (exact, read once), and every later tile reuses it.  The row
// sum is taken over exactly the rounded bf16 values written to the panel, so
// r * P~ sums to one.  A row whose true max exceeds m_ref by more
// than 2^FF_HEADROOM (never for real attention logits: that is a probability
// ratio of 2^96 between the first tile's best key and the row's best key)
// sets bit 1 of *flag and the caller recomputes with the two-pass kernel
// (rsa_fwd_resident); non-finite scores set bit 0 (NumericError).
//
// A CTA work unit is a PAIR of 128-row query tiles of one head (b, z), so
// each K / V tile brought into shared memory feeds 256 query rows; CTAs walk
// contiguous unit ranges so consecutive units mostly share the head and K
// stays resident when a row's T <= FF_KST key tiles fit.  18 warps:
//   warp 0        TMA producer (one lane)
//   warp 1        tcgen05.mma issuer of S = Q K^T (elect.sync); owns the TMEM allocation
//   warp 18       tcgen05.mma issuer of O~ += P~ [V | 1]
//   warps 2..17   two epilogue groups of 8 warps, group g = (w - 2) / 8 owns
//                 query tile g of the unit; warp w reads TMEM lanes
//                 32 * (w % 4).. (its tile rows) and column half ((w-2)/4) % 2
// TMEM: group g owns columns [256g, 256g + 256): S at +0 (128 columns; the
// epilogue moves it to registers at once, so one buffer suffices) and the
// O~ accumulator at +128 (64 columns).
#include <cstdio>
#include <algorithm>
#include <cstdlib>

#include "fused_common.cuh"

namespace rsa {
namespace {

struct FfArgs {
  CUtensorMap tq, tk, tv, tp, to;  // tp: 64 keys x 32 rows boxes (one per epilogue warp)
  Geo g;
  float sl;  // scale * log2(e)
  int* flag;
  float* rowscale;   // [rank][b][z][c]
  long long* trace;  // RSA_FF_TRACE: per-warp (event, clock) log of CTA 0 (timeline experiments)
  int peer;          // K / V of origin j from pm.k[j] / pm.v[j] (rsa_fwd_factored_peer)
  PeerMaps pm;
  // rsa_fwd_factored_ex options (all zero: rsa_fwd_factored with the panel written)
  int no_panel;             // stream mode: P~ stays on chip
  float* rowmax;            // out: the reference point m (scaled base 2) per row
  const float* rowmax_in;   // in: reference points (stride rm_stride floats)
  int rm_stride, rm_exact;  // rm_exact: true row maxima, no headroom check
  OutView o_acc;            // ring hops: fp32 running O~ (ptr NULL: single launch)
  float* l_acc;             //            fp32 running l
  int acc_in, final_hop;
  int ck;                   // keys per origin chunk (key_chunk; == c for RSA)
};

constexpr int FF_GROUPS = 2;
constexpr int FF_EPI_WARPS = 8 * FF_GROUPS;
constexpr int FF_PV_WARP = 2 + FF_EPI_WARPS;            // 18: issues the P~ V products
constexpr int FF_THREADS = 32 * (FF_PV_WARP + 1);       // 608
#ifndef FF_ONES
#define FF_ONES 1  // row sums from the tensor core (ones block next to V) instead of FADDs
#endif
#ifndef FF_ABSMAX
#define FF_ABSMAX 1  // tiles after the first: max|s| only (finite check + headroom bound)
#endif
#ifndef FF_QST
#define FF_QST 1  // Q tiles per group (2: the next unit's Q loads during this unit)
#endif
#ifndef FF_TS_LD2
#define FF_TS_LD2 1  // TS form: load all 64 columns of S before the first exp2 (frees S sooner)
#endif
#ifndef FF_PANEL_TS
#define FF_PANEL_TS 1  // panel forward: P~V from a TMEM copy of P~ (TS form); the smem tile only feeds the store
#endif
#ifndef FF_DEFER
#define FF_DEFER 1  // a unit's O readout deferred into the next unit's first step (unit_end)
#endif
#ifndef FF_KSTAGES
#define FF_KSTAGES 4
#endif
#ifndef FF_VSTAGES
#define FF_VSTAGES (FF_ONES ? 2 : 3)
#endif
constexpr int FF_KST = FF_KSTAGES, FF_VST = FF_VSTAGES;
constexpr int PV_N = FF_ONES ? HD + 16 : HD;  // O columns (+ 16 row-sum columns)
constexpr uint32_t TS_COL_P = 256, TS_COL_O = 320;  // TS form: shared P~ buffer, O~ of group g at +80 g
static_assert(TS_COL_O + FF_GROUPS * PV_N <= 512, "TS-form TMEM layout over 512 columns");
constexpr float FF_HEADROOM = 96.f;
    // max (row max - m_ref) * sl before the two-pass fallback
constexpr uint32_t FF_OFF_Q = 0;                                  // one tile per group
constexpr uint32_t FF_OFF_K = FF_OFF_Q + FF_GROUPS * FF_QST * TILE;
constexpr uint32_t FF_OFF_V = FF_OFF_K + FF_KST * TILE;
constexpr uint32_t FF_OFF_ONES = FF_OFF_V + FF_VST * TILE;        // 128 rows x 128 B of bf16 1.0 (FF_ONES)
constexpr uint32_t FF_OFF_P = FF_OFF_ONES + (FF_ONES ? TILE : 0);  // one P~ tile per group
constexpr uint32_t FF_OFF_X = FF_OFF_P + FF_GROUPS * PTILE;       // m_ref [group][parity][256], l [group][256]
constexpr uint32_t FF_OFF_BAR = FF_OFF_X + FF_GROUPS * 3 * 256 * 4;
constexpr uint32_t FF_SMEM = FF_OFF_BAR + 512 + 1024;
static_assert(FF_SMEM <= 232448, "fwd_factored smem over the sm_100 per-CTA limit");

__device__ __forceinline__ void bar_named(uint32_t id, uint32_t count) {
  asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(count) : "memory");
}

#define FF_TRACE(ev)                                                                                          \
  do {                                                                                                        \
    if (p.trace && blockIdx.x == 0 && (threadIdx.x & 31) == 0 && tr_i < 4095)                                 \
      p.trace[(threadIdx.x >> 5) * 4096 + tr_i++] = ((long long)(ev) << 48) | (long long)(clock64() - tr0); \
  } while (0)

struct Unit {  // work unit u: head bz, query tiles qi0 = 2p and qi0 + 1 (when it exists)
  int bz, qi0, n;
};

__device__ __forceinline__ Unit unit_of(int u, int units_per_head, int nq) {
  Unit r;
  r.bz = u / units_per_head;
  r.qi0 = 2 * (u % units_per_head);
  r.n = min(2, nq - r.qi0);
  return r;
}

// 96 registers: 19 warps put 5 warps on three SM sub-partitions, each with a 16K-register file.
// EXT: the rsa_fwd_factored_ex features (stream mode, given reference points, ring-hop
// accumulation, key_chunk != chunk); the plain instantiation is the hot forward.
//
// TS (stream mode, no panel written): P~ never touches shared memory.  The epilogue
// writes it to TMEM as packed bf16 pairs (tcgen05.st) and O~ += P~ [V | 1] runs as a
// TS-form product (A from TMEM, B from shared memory), which removes the P~ stores
// and the A-operand reads (64 + 64 KB per 256 x 128 step) from the shared-memory port
// and the store -> proxy fence -> barrier chain from the epilogue.  TMEM: S of group g
// at 128 g, ONE P~ buffer (64 columns) at 256 that the two groups take in turn (P~V of
// one group frees it for the next), O~ of group g at 320 + 80 g: 480 columns.
template <bool EXT, bool TS>
__global__ void __maxnreg__(96) fwd_factored_kernel(const __grid_constant__ FfArgs p) {
  // stream mode (TS with EXT): no per-score check after the first key tile, the row sum
  // bounds the rest; the panel forward in TS form keeps the max|s| check
  constexpr bool LCHK = TS && EXT;
  constexpr bool NOPANEL = TS && EXT;  // ff_launch picks <true, true> exactly for p.no_panel
  // Q stages per group: stream mode has no panel to stage, so the second half of each group's
  // P~ tile holds a second Q stage -- the next unit's Q loads while this unit runs (the O
  // staging moves to the first half).  A Q tile from a busy HBM takes ~7 k clk, which a unit
  // of few key tiles (Linformer's K' = 256 keys: two) does not cover.
  constexpr int QS = NOPANEL ? 2 : FF_QST;
  auto q_off = [](int qx) -> uint32_t {  // qx = group * QS + stage
    if (QS == FF_QST) return FF_OFF_Q + qx * TILE;
    const int gq = qx / QS, sq = qx % QS;
    return sq < FF_QST ? FF_OFF_Q + (gq * FF_QST + sq) * TILE : FF_OFF_P + gq * PTILE + ATOM;
  };
  uint8_t* smem = smem_base();
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + FF_OFF_BAR);
  uint64_t *q_full = bar, *q_empty = q_full + 2 * QS;  // [group][stage]
  uint64_t *k_full = q_empty + 2 * QS, *k_empty = k_full + FF_KST;
  uint64_t *v_full = k_empty + FF_KST, *v_empty = v_full + FF_VST;
  uint64_t *s_full = v_empty + FF_VST, *s_empty = s_full + 2;
  uint64_t *p_full = s_empty + 2, *p_empty = p_full + 2;
  uint64_t *o_full = p_empty + 2, *o_empty = o_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_empty + 2);

  const Geo& g = p.g;
  const int ck = EXT ? p.ck : g.c;
  const int ntk = (ck + TK - 1) / TK, nrt = (g.c + TR - 1) / TR;
  const int T = g.n_org * ntk;    // key tiles per row
  const int NQ = g.n_rank * nrt;  // query tiles per head
  const int UH = (NQ + 1) / 2;    // units per head
  const int units = g.B * g.Z * UH;
  const uint32_t warp = warp_id(), lane = lane_id();
  const int u_begin = int(int64_t(blockIdx.x) * units / gridDim.x);
  const int u_end = int(int64_t(blockIdx.x + 1) * units / gridDim.x);
  const bool kres = T <= FF_KST;  // K tile t stays in slot t while the head is unchanged

#if FF_ONES
  {  // constant B-operand block of ones (read by the async proxy)
    uint4* ones = reinterpret_cast<uint4*>(smem + FF_OFF_ONES);
    for (uint32_t i = threadIdx.x; i < TILE / 16; i += FF_THREADS)
      ones[i] = make_uint4(0x3F803F80u, 0x3F803F80u, 0x3F803F80u, 0x3F803F80u);
    fence_proxy_async_smem();
  }
#endif
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  if (threadIdx.x == 0) {
    for (int s = 0; s < 2; ++s) {
      for (int q = 0; q < QS; ++q) mbar_init(&q_full[s * QS + q], 1), mbar_init(&q_empty[s * QS + q], 1);
      mbar_init(&s_full[s], 1), mbar_init(&s_empty[s], 8);
      mbar_init(&p_full[s], 8), mbar_init(&p_empty[s], 1);
      mbar_init(&o_full[s], 1), mbar_init(&o_empty[s], 8);
    }
    if (TS) mbar_arrive(&p_empty[0]);  // group 0's first use of the shared P~ buffer has no predecessor
    for (int s = 0; s < FF_KST; ++s) mbar_init(&k_full[s], 1), mbar_init(&k_empty[s], 1);
    for (int s = 0; s < FF_VST; ++s) mbar_init(&v_full[s], 1), mbar_init(&v_empty[s], 1);
    fence_barrier_init();
    tma_prefetch(&p.tq), tma_prefetch(&p.tk), tma_prefetch(&p.tv), tma_prefetch(&p.tp), tma_prefetch(&p.to);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base(tmem_slot);
  const long long tr0 = clock64();
  int tr_i = 0;

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    if (TS && lane == 31 && p.trace && blockIdx.x == 0) {
      // timeline experiments (RSA_FF_TRACE): completion times of group 0's S (event 50) and
      // of every P~V (event 51), observed from a lane that is otherwise idle
      uint32_t ns = 0, np0 = 0, np1 = 0;
      for (int i = 0; i < 4000 && tr_i < 4000; ++i) {
        if (mbar_try_wait(&s_full[0], ns & 1)) {
          p.trace[tr_i++] = (50ll << 48) | (clock64() - tr0), ++ns;
        }
        if (mbar_try_wait(&p_empty[1], np1 & 1)) {  // P~V of group 0 done (frees P~ for group 1)
          p.trace[tr_i++] = (51ll << 48) | (clock64() - tr0), ++np1;
        }
        if (mbar_try_wait(&p_empty[0], np0 & 1)) {  // phase 0 is the pre-arrive; then P~V of group 1
          if (np0) p.trace[tr_i++] = (52ll << 48) | (clock64() - tr0);
          ++np0;
        }
      }
    }
    if (lane == 0) {
      Pos kq, vq;
      uint32_t qn[2] = {0, 0}, kgen = 0;
      int prev_bz = -1;
      for (int u = u_begin; u < u_end; ++u) {
        const Unit un = unit_of(u, UH, NQ);
        const int b = un.bz / g.Z, z = un.bz % g.Z;
        for (int gi = 0; gi < un.n; ++gi) {
          const int qi = un.qi0 + gi, d = qi / nrt, rt = qi % nrt;
          const int qx = gi * QS + int(qn[gi] % QS);
          mbar_wait(&q_empty[qx], ((qn[gi] / QS) & 1) ^ 1);
          mbar_arrive_expect_tx(&q_full[qx], TILE);
          tma_load_4d(smem + q_off(qx), &p.tq, &q_full[qx], 0, rt * TR, z, d * g.B + b);
          ++qn[gi];
        }
        if (kres && un.bz != prev_bz) {
          for (int t = 0, jo = 0, k0 = 0; t < T; ++t, k0 = k0 + TK >= ntk * TK ? (++jo, 0) : k0 + TK) {
            mbar_wait(&k_empty[t], (kgen & 1) ^ 1);
            mbar_arrive_expect_tx(&k_full[t], TILE);
            tma_load_4d(smem + FF_OFF_K + t * TILE, p.peer ? &p.pm.k[jo] : &p.tk, &k_full[t], 0, k0, z,
                        p.peer ? b : jo * g.B + b);
          }
          ++kgen;
        }
        prev_bz = un.bz;
        for (int t = 0, jo = 0, k0 = 0; t < T; ++t, k0 = k0 + TK >= ntk * TK ? (++jo, 0) : k0 + TK) {
          if (!kres) {
            const uint32_t ks = kq.slot(FF_KST);
            mbar_wait(&k_empty[ks], kq.phase(FF_KST) ^ 1);
            mbar_arrive_expect_tx(&k_full[ks], TILE);
            tma_load_4d(smem + FF_OFF_K + ks * TILE, p.peer ? &p.pm.k[jo] : &p.tk, &k_full[ks], 0, k0, z,
                        p.peer ? b : jo * g.B + b);
            ++kq.i;
          }
          const uint32_t vs = vq.slot(FF_VST);
          mbar_wait(&v_empty[vs], vq.phase(FF_VST) ^ 1);
          mbar_arrive_expect_tx(&v_full[vs], TILE);
          tma_load_4d(smem + FF_OFF_V + vs * TILE, p.peer ? &p.pm.v[jo] : &p.tv, &v_full[vs], 0, k0, z,
                      p.peer ? b : jo * g.B + b);
          ++vq.i;
        }
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------- MMA issuer
    const uint32_t idesc_s = idesc_bf16_f32(TR, TK, 0, 0);
    Pos kq;
    uint32_t qn[2] = {0, 0}, sn[2] = {0, 0}, kgen = 0;
    int prev_bz = -1;
    for (int u = u_begin; u < u_end; ++u) {
      const Unit un = unit_of(u, UH, NQ);
      if (kres && un.bz != prev_bz) ++kgen;
      prev_bz = un.bz;
      // resident K: release the slots after the unit's last S unless the next unit reuses them
      const bool k_release = kres && u + 1 < u_end && unit_of(u + 1, UH, NQ).bz != un.bz;
      for (int gi = 0; gi < un.n; ++gi)
        mbar_wait(&q_full[gi * QS + qn[gi] % QS], (qn[gi] / QS) & 1);
      // S(g) = Q_g K_t^T for both query tiles of the unit from one K tile
      auto issue_s = [&](int t) {
        const bool last = t + 1 == T;
        const uint32_t ks = kres ? uint32_t(t) : kq.slot(FF_KST);
        mbar_wait(&k_full[ks], kres ? (kgen - 1) & 1 : kq.phase(FF_KST));
        const uint32_t ka = smem_u32(smem + FF_OFF_K + ks * TILE);
        for (int gi = 0; gi < un.n; ++gi) {
          mbar_wait(&s_empty[gi], (sn[gi] & 1) ^ 1);
          tc_fence_after();
          const uint32_t qa = smem_u32(smem + q_off(gi * QS + qn[gi] % QS));
#pragma unroll
          for (int k = 0; k < HD / 16; ++k)
            umma_bf16_ws(tmem + gi * (TS ? 128 : 256), smem_desc_sw128(qa + k * 32, 0, 1024),
                         smem_desc_sw128(ka + k * 32, 0, 1024), idesc_s, k > 0);
          umma_commit_ws(&s_full[gi]);
          FF_TRACE(10 + gi);
          if (last) umma_commit_ws(&q_empty[gi * QS + qn[gi] % QS]), ++qn[gi];
          ++sn[gi];
        }
        if (!kres) umma_commit_ws(&k_empty[ks]), ++kq.i;
        else if (last && k_release)
          for (int j = 0; j < T; ++j) umma_commit_ws(&k_empty[j]);
      };
      for (int t = 0; t < T; ++t) issue_s(t);
    }
  } else if (warp == FF_PV_WARP) {
    // ------------------------------------------- P~ V issuer (second MMA thread)
    // A separate issuing thread, so S(t+1) never queues behind the other group's
    // P~ V; tcgen05.commit tracks each thread's own MMAs, so the barriers stay exact.
    const uint32_t idesc_o = idesc_bf16_f32(TR, PV_N, 0, 1);
    Pos vq;
    uint32_t pn[2] = {0, 0}, on[2] = {0, 0};
    for (int u = u_begin; u < u_end; ++u) {
      const Unit un = unit_of(u, UH, NQ);
      for (int t = 0; t < T; ++t) {  // O~ += P~ [V | 1]
        const uint32_t vs = vq.slot(FF_VST);
        mbar_wait(&v_full[vs], vq.phase(FF_VST));
        const uint32_t va = smem_u32(smem + FF_OFF_V + vs * TILE);
        // N = 80: the second 64-column B atom is the ones block (its offset is the LBO)
        const uint32_t lbo = FF_ONES ? FF_OFF_ONES - (FF_OFF_V + vs * TILE) : ATOM;
        for (int gi = 0; gi < un.n; ++gi) {
          if (t == 0) mbar_wait(&o_empty[gi], (on[gi] & 1) ^ 1);
          mbar_wait(&p_full[gi], pn[gi] & 1);
          tc_fence_after();
          if (TS) {
#pragma unroll
            for (int k = 0; k < TK / 16; ++k)  // A: 8 TMEM columns (16 keys as bf16 pairs) per k step
              umma_bf16_ts_ws(tmem + TS_COL_O + gi * PV_N, tmem + TS_COL_P + 8 * k,
                              smem_desc_sw128(va + k * 2048, lbo, 1024), idesc_o, (t | k) != 0);
            // the shared P~ buffer passes to the next user: the other group, or group 0 of the next step
            umma_commit_ws(&p_empty[gi + 1 < un.n ? gi + 1 : 0]);
          } else {
            const uint32_t pa = smem_u32(smem + FF_OFF_P + gi * PTILE);
#pragma unroll
            for (int k = 0; k < TK / 16; ++k)
              umma_bf16_ws(tmem + gi * 256 + 128, smem_desc_sw128(pa + (k >> 2) * ATOM + (k & 3) * 32, 0, 1024),
                           smem_desc_sw128(va + k * 2048, lbo, 1024), idesc_o, (t | k) != 0);
            umma_commit_ws(&p_empty[gi]);
          }
          FF_TRACE(12 + gi);
          ++pn[gi];
        }
        umma_commit_ws(&v_empty[vs]);
        ++vq.i;
      }
      for (int gi = 0; gi < un.n; ++gi) umma_commit_ws(&o_full[gi]), ++on[gi];
    }
  } else if (warp < FF_PV_WARP) {
    // ------------------------------------------------------------ epilogue
    const uint32_t gi = (warp - 2) >> 3;
    const uint32_t quad = warp & 3;
    const int half = ((warp - 2) >> 2) & 1;
    const int r = quad * 32 + lane;
    const int et = (threadIdx.x - 64) & 255;         // thread index within the group
    const uint32_t lane_base = (quad * 32u) << 16;
    const uint32_t t_s = tmem + lane_base + gi * (TS ? 128 : 256) + half * 64;
    const uint32_t t_o = tmem + lane_base + (TS ? TS_COL_O + gi * PV_N : gi * 256 + 128);
    const uint32_t xbase = smem_u32(smem + FF_OFF_X) + gi * 3 * 256 * 4;
    const uint32_t ptile = smem_u32(smem + FF_OFF_P + gi * PTILE);
    uint8_t* ptile_gen = smem + FF_OFF_P + gi * PTILE + half * ATOM;
    const uint32_t bar_rows_id = 6 + gi * 4 + quad;
    const float sl = p.sl;
    uint32_t sn = 0, pn = 0, un_n = 0;
    bool bad = false, redo = false;
    const uint64_t pol = l2_evict_first();
    // DEFER (TS form, row sums from the ones block): the previous unit's end waits for the
    // next unit's first exp2 (unit_end)
    constexpr bool DEFER = TS && FF_DEFER;
    bool pend = false;
    int pd_ = 0, pb_ = 0, pz_ = 0, prt_ = 0;
    float pmsl_ = 0.f, plsum_ = 0.f;  // plsum_: the pending unit's row-sum share (FF_ONES = 0)
    uint32_t ux = 0;  // units begun: parity of the row-max exchange slot
    // A unit's end: O = O~ / l and r = 1 / l once its last P~ V has landed (o_full), then the
    // per-warp O store.  DEFER: run during the NEXT unit's first step, after that step's
    // exp2 and before its P~ store (which frees O~ for the next unit), so the epilogue does
    // not sit idle while the last P~ V products of the unit drain.
    auto unit_end = [&](int d, int b, int z, int rt, float msl, float lsum) {
      const int row = rt * TR + r;
      // ---- O = O~ / l, r = 1 / l (l >= 1 unless the row needs the fallback)
      mbar_wait(&o_full[gi], un_n & 1);
      FF_TRACE(7);
      tc_fence_after();
      float o[32];
      __syncwarp();
      tmem_ld32(t_o + half * 32, o);
#if FF_ONES
      uint32_t lraw;
      asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(lraw) : "r"(t_o + HD));
#endif
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&o_empty[gi]);
      float l;
#if FF_ONES
      l = __uint_as_float(lraw);
#else
      {  // the row sum: this half's share plus the other half's
        const uint32_t slot = xbase + 2 * 256 * 4;
        asm volatile("st.shared.f32 [%0], %1;" ::"r"(slot + et * 4), "f"(lsum) : "memory");
        bar_named(bar_rows_id, 64);
        float o2;
        asm volatile("ld.shared.f32 %0, [%1];" : "=f"(o2) : "r"(slot + ((et + 128) & 255) * 4) : "memory");
        l = lsum + o2;
      }
#endif
      ++un_n;
      const int64_t ridx = (int64_t(d * g.B + b) * g.Z + z) * g.c + row;
      if (EXT && p.acc_in && row < g.c) {  // ring hops: add the running O~ and l of earlier origins
        const float* oa = reinterpret_cast<const float*>(p.o_acc.ptr) + out_off(p.o_acc, d, b, z, row) + half * 32;
#pragma unroll
        for (int e = 0; e < 32; e += 4) {
          const float4 x = *reinterpret_cast<const float4*>(oa + e);
          o[e] += x.x, o[e + 1] += x.y, o[e + 2] += x.z, o[e + 3] += x.w;
        }
        l += p.l_acc[ridx];
      }
      if (EXT && !p.final_hop) {  // not the last hop: hand O~ and l to the next launch
        if (row < g.c) {
          float* oa = reinterpret_cast<float*>(p.o_acc.ptr) + out_off(p.o_acc, d, b, z, row) + half * 32;
#pragma unroll
          for (int e = 0; e < 32; e += 4) *reinterpret_cast<float4*>(oa + e) = make_float4(o[e], o[e + 1], o[e + 2], o[e + 3]);
          if (half == 0) {
            p.l_acc[ridx] = l;
            if (EXT && p.rowmax && !p.rowmax_in) p.rowmax[ridx] = msl;
          }
        }
        FF_TRACE(21);
        return;
      }
      const float rinv = 1.f / l;
      // TS: l >= every P~ of the row, so l <= 2^FF_HEADROOM is the headroom check (conservative)
      redo |= !(l >= 1.f && l <= (LCHK && !p.rm_exact ? 7.9228162514e28f : 3.402823466e38f));
      // O -> this warp's 32 rows x 32 columns, staged in the first 2 KB of its own P~ rows
      // (64-byte rows, SWIZZLE_64B) -> one TMA store per warp: no group barrier.  The region's
      // only other user is this warp's own P~ store (waited for here), and the P~V products
      // that read it (non-TS form) are complete: o_full.
      if (lane == 0) tma_store_wait_read<0>();
      __syncwarp();
      {
        // (stream mode: the first half of the P~ tile, 2 KB per warp; the second half is a Q stage)
        uint8_t* ostg = NOPANEL ? smem + FF_OFF_P + gi * PTILE + (half * 4 + quad) * 2048 : ptile_gen + quad * 4096;
        const uint32_t orow = smem_u32(ostg) + lane * 64, osw = (lane >> 1) & 3;
#pragma unroll
        for (int q4 = 0; q4 < 4; ++q4)
          st_shared_v4(orow + ((q4 ^ osw) << 4), pack_bf16(o[8 * q4] * rinv, o[8 * q4 + 1] * rinv),
                       pack_bf16(o[8 * q4 + 2] * rinv, o[8 * q4 + 3] * rinv),
                       pack_bf16(o[8 * q4 + 4] * rinv, o[8 * q4 + 5] * rinv),
                       pack_bf16(o[8 * q4 + 6] * rinv, o[8 * q4 + 7] * rinv));
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          tma_store_4d(&p.to, ostg, half * 32, rt * TR + int(quad) * 32, z, d * g.B + b);
          tma_store_commit();
        }
      }
      if (row < g.c && half == 0) {
        p.rowscale[ridx] = rinv;
        if (EXT && p.rowmax && !p.rowmax_in) p.rowmax[ridx] = msl;
      }
      FF_TRACE(21);
    };
    for (int u = u_begin; u < u_end; ++u) {
      const Unit un = unit_of(u, UH, NQ);
      if (int(gi) >= un.n) continue;
      const int b = un.bz / g.Z, z = un.bz % g.Z;
      const int qi = un.qi0 + gi, d = qi / nrt, rt = qi % nrt;
      const int row = rt * TR + r;
      FF_TRACE(1);
      // tile 0: raw max and min (the reference point); later tiles: max |s| only, which
      // bounds the row max (headroom check) and is finite iff every score is
      float m = -INFINITY, mi = INFINITY, am = 0.f, msl = 0.f;
      if (EXT && p.rowmax_in)
        msl = row < g.c ? __ldg(p.rowmax_in + ((int64_t(d * g.B + b) * g.Z + z) * g.c + row) * p.rm_stride) : 0.f;
#if !FF_ONES
      float lsum = 0.f;  // this thread's share of sum_k P~[row, k] over the bf16 values stored
#endif
      int jo = 0, k0 = 0;
      for (int t = 0; t < T; ++t) {
        const int nvalid = min(TK, ck - k0) - half * 64;
        uint32_t w[32];
        mbar_wait(&s_full[gi], sn & 1);
        FF_TRACE(3);
        tc_fence_after();
        __syncwarp();
        if (t == 0 && !(EXT && p.rowmax_in)) {  // first key tile: its row max is the reference
          float v[64];
          tmem_ld32(t_s, v);
          tmem_ld32(t_s + 32, v + 32);
          tmem_ld_wait();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&s_empty[gi]);
          minmax32(v, nvalid, m, mi);
          minmax32(v + 32, nvalid - 32, m, mi);
          const uint32_t slot = xbase + (ux & 1) * 256 * 4;  // combine the two column halves
          asm volatile("st.shared.f32 [%0], %1;" ::"r"(slot + et * 4), "f"(m) : "memory");
          bar_named(bar_rows_id, 64);
          float o;
          asm volatile("ld.shared.f32 %0, [%1];" : "=f"(o) : "r"(slot + ((et + 128) & 255) * 4) : "memory");
          const float mref = fmaxf(m, o);
          msl = (mref == -INFINITY || !(fabsf(mref) <= 3.402823466e38f)) ? 0.f : mref * sl;
          exp2_pack32(v, nvalid, sl, msl, w);
          exp2_pack32(v + 32, nvalid - 32, sl, msl, w + 16);
        } else if (LCHK && FF_TS_LD2) {  // both chunks in flight, then S is free before any exp2
          float v[64];
          tmem_ld32(t_s, v);
          tmem_ld32(t_s + 32, v + 32);
          tmem_ld_wait();
          FF_TRACE(40);
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&s_empty[gi]);
          FF_TRACE(41);
#pragma unroll
          for (int cc = 0; cc < 2; ++cc) {
            // no per-score check: the row sum l bounds every P~ (headroom) and is non-finite
            // iff a score is +inf / NaN; -inf scores come only from non-finite keys, which
            // rsa_fwd_factored_ex scans for before the launch (k_scan_kernel)
            exp2_pack32(v + cc * 32, nvalid - cc * 32, sl, msl, w + cc * 16);
          }
        } else {
#pragma unroll
          for (int cc = 0; cc < 2; ++cc) {  // two 32-column chunks (register budget of 18 warps)
            float v[32];
            tmem_ld32(t_s + cc * 32, v);
            tmem_ld_wait();
            FF_TRACE(40 + cc);
            if (cc == 1) {  // both chunks are in registers: free S for the next key tile
              tc_fence_before();
              __syncwarp();
              if (lane == 0) mbar_arrive(&s_empty[gi]);
            }
            if (FF_ABSMAX) absmax32(v, nvalid - cc * 32, am);
            else minmax32(v, nvalid - cc * 32, m, mi);
            exp2_pack32(v, nvalid - cc * 32, sl, msl, w + cc * 16);
          }
        }
        ++sn;
#if !FF_ONES
#pragma unroll
        for (int e = 0; e < 32; ++e) lsum += __uint_as_float(w[e] << 16) + __uint_as_float(w[e] & 0xFFFF0000u);
#endif
        FF_TRACE(4);
        if (DEFER && t == 0 && pend) {  // the previous unit's O~ is read out before this P~ V can overwrite it
          pend = false;
          unit_end(pd_, pb_, pz_, prt_, pmsl_, plsum_);
        }
        if (TS) {  // P~ -> the shared TMEM buffer once the previous user's P~ V has read it
          mbar_wait(&p_empty[gi], pn & 1);
          FF_TRACE(5);
          tc_fence_after();
          tmem_st32(tmem + lane_base + TS_COL_P + half * 32, w);
          tmem_st_wait();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&p_full[gi]);
          FF_TRACE(6);
          ++pn;
          if (NOPANEL) {
            if (k0 + TK >= ck) k0 = 0, ++jo;
            else k0 += TK;
            continue;
          }
        } else {
          mbar_wait(&p_empty[gi], (pn & 1) ^ 1);  // the previous P~ V product has read the tile
          FF_TRACE(5);
        }
        // Each warp stores its own 32 rows x 64 keys (4 KB, 1024-byte aligned, so the
        // 128-byte swizzle pattern is the tile's): no cross-warp barrier on this path.
        if (lane == 0) tma_store_wait_read<0>();  // this warp's previous store has read its rows
        __syncwarp();
#pragma unroll
        for (int q4 = 0; q4 < 8; ++q4)
          st_shared_v4(ptile + half * ATOM + sw128_offset(r, q4), w[4 * q4], w[4 * q4 + 1], w[4 * q4 + 2],
                       w[4 * q4 + 3]);
        fence_proxy_async_smem();
        __syncwarp();
        if (lane == 0) {
          if (!TS) mbar_arrive(&p_full[gi]);  // TS: the P~V product reads TMEM, the tile only feeds the store
          if (nvalid > 0 && !NOPANEL)  // the panel is read back only by the backward: evict-first in L2
            tma_store_5d_hint(&p.tp, ptile_gen + quad * 4096, k0 + half * 64, g.org_lo + jo, rt * TR + quad * 32, z,
                              d * g.B + b, pol);
          tma_store_commit();
        }
        FF_TRACE(6);
        if (!TS) ++pn;
        if (k0 + TK >= ck) k0 = 0, ++jo;
        else k0 += TK;
      }
      if (!(m == -INFINITY && mi == INFINITY))  // this thread saw at least one valid key in tile 0
        bad |= !(fabsf(m) <= 3.402823466e38f) || !(fabsf(mi) <= 3.402823466e38f);
      bad |= !(am <= 3.402823466e38f);
      if (!LCHK && !(EXT && p.rm_exact)) redo |= (FF_ABSMAX ? am : m) * sl - msl > FF_HEADROOM;  // |s| >= s: conservative
      ++ux;
      if (DEFER) {
        pend = true, pd_ = d, pb_ = b, pz_ = z, prt_ = rt, pmsl_ = msl;
#if !FF_ONES
        plsum_ = lsum;
#endif
      } else {
#if FF_ONES
        unit_end(d, b, z, rt, msl, 0.f);
#else
        unit_end(d, b, z, rt, msl, lsum);
#endif
      }
    }
    if (DEFER && pend) unit_end(pd_, pb_, pz_, prt_, pmsl_, plsum_);
    if (p.flag && (bad || redo)) atomicOr(p.flag, (bad ? 1 : 0) | (redo ? 2 : 0));
    if (lane == 0) tma_store_wait_all<0>();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, 512);
}

}  // namespace
}  // namespace rsa

namespace rsa {
namespace {

// Any non-finite bf16 among the keys [org][b][z][row][64] (16-byte chunks, strided rows) ->
// bit 0 of *flag (NumericError), as the reference's softmax_rows would raise on the scores.
// grid (row blocks, heads): no index division per element.
__global__ void __launch_bounds__(256) k_scan_kernel(const uint4* __restrict__ k, int64_t s_org, int64_t s_b,
                                                     int64_t s_z, int64_t s_row, int B, int Z, int ck, int* flag) {
  const int h = blockIdx.y, z = h % Z, ob = h / Z, b = ob % B, o = ob / B;
  const uint4* base = k + (o * s_org + b * s_b + z * s_z) / 8;
  const int chunks = ck * (HD / 8);
  bool bad = false;
  for (int i = blockIdx.x * 1024 + threadIdx.x, e = 0; e < 4; ++e, i += 256) {
    if (i >= chunks) break;
    const uint4 x = __ldg(base + ((i >> 3) * s_row) / 8 + (i & 7));
    const uint32_t w[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
    for (int j = 0; j < 4; ++j)
      bad |= (w[j] & 0x7F80u) == 0x7F80u || (w[j] & 0x7F800000u) == 0x7F800000u;
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 1);
}

int ff_launch(FfArgs& a, const rsa_geom* g, rsa_view q, rsa_view panel, rsa_view o_out, float* rowscale, int* flag,
              void* stream) {
  const bool final_hop = !a.o_acc.ptr || a.final_hop;
  a.final_hop = final_hop;
  if (!flag || (final_hop && (!rowscale || !o_out.ptr || !out_ok(o_out, 2))))
    return fail(RSA_ERR_UNSUPPORTED, "rsa_fwd_factored: output / row-scale / flag buffers missing or misaligned");
  if (a.o_acc.ptr && (!a.l_acc || !out_ok(rsa_view{a.o_acc.ptr, a.o_acc.s_rank, a.o_acc.s_b, a.o_acc.s_z,
                                                    a.o_acc.s_row}, 4)))
    return fail(RSA_ERR_UNSUPPORTED, "rsa_fwd_factored_ex: o_acc / l_acc missing or misaligned");
  if (!a.o_acc.ptr && a.acc_in) return fail(RSA_ERR_INVALID, "rsa_fwd_factored_ex: acc_in without o_acc");
  if (a.rowmax_in && a.rm_stride < 1) return fail(RSA_ERR_INVALID, "rsa_fwd_factored_ex: rowmax_in_stride < 1");
  a.no_panel = panel.ptr == nullptr;
  if (!a.no_panel && key_chunk(g) != g->chunk)
    return fail(RSA_ERR_INVALID, "rsa_fwd_factored_ex: a panel needs key_chunk == chunk");
  if (!head_map(&a.tq, q, g, g->n_rank) || (!a.no_panel && !panel_map(&a.tp, panel, g, g->n_rank, 32)) ||
      (final_hop && !head_map_w32(&a.to, o_out, g, g->n_rank)))
    return RSA_ERR_UNSUPPORTED;
  if (a.no_panel) a.tp = a.tq;  // never used; keeps the prefetch harmless
  if (!final_hop) a.to = a.tq;
  a.g = to_geo(g);
  a.ck = key_chunk(g);
  a.sl = g->scale * LOG2E;
  a.flag = flag;
  a.rowscale = rowscale;
  static long long* trace_buf = nullptr;
  const char* trace_path = getenv("RSA_FF_TRACE");
  if (trace_path) {
    if (!trace_buf) cudaMalloc(&trace_buf, (FF_THREADS / 32) * 4096 * sizeof(long long));
    cudaMemset(trace_buf, 0, (FF_THREADS / 32) * 4096 * sizeof(long long));
    a.trace = trace_buf;
  }
  const int nq = g->n_rank * ((g->chunk + TR - 1) / TR);
  const int units = g->batch * g->heads * ((nq + 1) / 2);
  if (units <= 0) return RSA_OK;
  const bool ext = a.no_panel || a.rowmax || a.rowmax_in || a.o_acc.ptr || a.ck != g->chunk;
  auto kernel = a.no_panel ? fwd_factored_kernel<true, true>
                           : ext ? fwd_factored_kernel<true, false> : fwd_factored_kernel<false, FF_PANEL_TS != 0>;
  cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, FF_SMEM);
  cudaFuncAttributes fa{};
  if (cudaFuncGetAttributes(&fa, kernel) == cudaSuccess && fa.maxThreadsPerBlock < FF_THREADS)
    return fail(RSA_ERR_CUDA, "rsa_fwd_factored: %d registers/thread allow only %d threads per CTA (need %d)",
                fa.numRegs, fa.maxThreadsPerBlock, FF_THREADS);
  const int grid = persistent_grid(units);
  launch_grid(kernel, grid, FF_THREADS, FF_SMEM, a, stream);
  if (trace_path) {
    static long long host[(FF_THREADS / 32) * 4096];
    cudaMemcpy(host, trace_buf, sizeof(host), cudaMemcpyDeviceToHost);
    if (FILE* f = fopen(trace_path, "wb")) fwrite(host, sizeof(host), 1, f), fclose(f);
  }
  return check_launch("fwd_factored_kernel");
}

}  // namespace
}  // namespace rsa

extern "C" {

int rsa_fwd_factored(const rsa_geom* g, rsa_view q, rsa_view k, rsa_view v, rsa_view panel, rsa_view o_out,
                     float* rowscale, int* flag, void* stream) {
  using namespace rsa;
  if (!geom_ok(g)) return fail(RSA_ERR_INVALID, "rsa_fwd_factored: unsupported geometry");
  if (g->org_lo != 0 || g->n_org != g->seq_len / g->chunk)
    return fail(RSA_ERR_INVALID, "rsa_fwd_factored: every origin must be resident (org_lo = 0, n_org = L / c)");
  FfArgs a{};
  if (!head_map(&a.tk, k, g, g->n_org) || !head_map(&a.tv, v, g, g->n_org)) return RSA_ERR_UNSUPPORTED;
  return ff_launch(a, g, q, panel, o_out, rowscale, flag, stream);
}

int rsa_fwd_factored_ex(const rsa_geom* g, rsa_view q, rsa_view k, rsa_view v, const rsa_fwd_ext* ext,
                        rsa_view o_out, float* rowscale, int* flag, void* stream) {
  using namespace rsa;
  if (!ext) return fail(RSA_ERR_INVALID, "rsa_fwd_factored_ex: options missing");
  if (!geom_ok_keys(g)) return fail(RSA_ERR_INVALID, "rsa_fwd_factored_ex: unsupported geometry");
  if (!ext->panel.ptr && !ext->rowmax_exact && flag) {
    // the TS form checks no score after the first key tile: a non-finite key sets bit 0 here
    const int heads = g->n_org * g->batch * g->heads;
    if (heads > 0 && heads < 65536 && k.ptr && aligned16(k.ptr) && k.s_row % 8 == 0 && k.s_z % 8 == 0 &&
        k.s_b % 8 == 0 && k.s_rank % 8 == 0) {
      const dim3 grid((key_chunk(g) * (HD / 8) + 1023) / 1024, heads);
      k_scan_kernel<<<grid, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
          reinterpret_cast<const uint4*>(k.ptr), k.s_rank, k.s_b, k.s_z, k.s_row, g->batch, g->heads, key_chunk(g),
          flag);
      if (int rc = check_launch("k_scan_kernel")) return rc;
    }
  }
  FfArgs a{};
  if (!head_map(&a.tk, k, g, g->n_org, key_chunk(g)) || !head_map(&a.tv, v, g, g->n_org, key_chunk(g)))
    return RSA_ERR_UNSUPPORTED;
  a.rowmax = ext->rowmax;
  a.rowmax_in = ext->rowmax_in;
  a.rm_stride = ext->rowmax_in_stride > 0 ? ext->rowmax_in_stride : 1;
  a.rm_exact = ext->rowmax_exact;
  a.o_acc = to_out(ext->o_acc);
  a.l_acc = ext->l_acc;
  a.acc_in = ext->acc_in;
  a.final_hop = ext->final_hop;
  return ff_launch(a, g, q, ext->panel, o_out, rowscale, flag, stream);
}

int rsa_fwd_factored_peer(const rsa_geom* g, rsa_view q, const rsa_view* k_origin, const rsa_view* v_origin,
                          rsa_view panel, rsa_view o_out, float* rowscale, int* flag, void* stream) {
  using namespace rsa;
  if (!geom_ok(g) || !k_origin || !v_origin) return fail(RSA_ERR_INVALID, "rsa_fwd_factored_peer: bad arguments");
  if (g->n_rank != 1 || g->org_lo != 0 || g->n_org != g->seq_len / g->chunk)
    return fail(RSA_ERR_INVALID, "rsa_fwd_factored_peer: need n_rank = 1, org_lo = 0, n_org = L / c");
  FfArgs a{};
  a.peer = 1;
  if (!peer_maps(&a.pm, k_origin, v_origin, g)) return RSA_ERR_UNSUPPORTED;
  return ff_launch(a, g, q, panel, o_out, rowscale, flag, stream);
}

}  // extern "C"

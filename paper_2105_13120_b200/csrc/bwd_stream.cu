// Stream-mode RSA backward for sm_100a (head size A = 64): dQ, dK and dV with no saved
// probability panel.  Replaces the V-ring / K-ring backward of
// ringseq/ring_attention.py:168-209 when the forward kept only O and two numbers per row
// (rsa_fwd_factored_ex without a panel): the reference point m (scaled base 2) and the
// row scale r = 1 / sum_k P~.  Each tile of the factored panel is recomputed on chip,
//   S  = Q K_j^T                          (tensor core, TMEM; the forward's exact products)
//   P~ = 2^(S * scale * log2(e) - m)      (exp2_pack32: the forward's exact rounding)
// so P~ equals, bit for bit, the panel rsa_fwd_factored would have written, and the
// backward products run on it exactly as on a factored panel (rsa_rowdot_scale supplies
// dO' = dO * r and D' = D * r):
//   dP' = dO' V_j^T,  dS = P~ (dP' - D')  (= P (dP - D)),
//   dV_j += P~^T dO',  dK_j += dS^T Q,  dQ += dS K_j        (the 1/sqrt(A) at the end).
// Memory per rank is O(c) instead of O(c * L): the "max trainable length grows linearly
// with N" mode (hard part 5).  Keys per origin (key_chunk) may differ
// from query rows per rank, which serves the Linformer's projected keys too.
//
// Two persistent, warp-specialised kernels (warp 0 TMA producer, warp 1 tcgen05.mma issuer,
// warps 2..17 epilogue: warp w owns TMEM lanes 32*(w%4).. and column quarter (w-2)/4), each
// accumulating in TMEM in a fixed order (deterministic, no atomics):
//   bwd_kv_stream_kernel  item = (origin, b, z, key tile); walks every query tile:
//                         S, dP' -> P~ to smem -> dV += P~^T dO' -> dS in place -> dK += dS^T Q
//   bwd_q_stream_kernel   item = (rank, b, z, query tile); walks every key tile:
//                         S, dP' -> dS to smem -> dQ += dS K
#include <cstdlib>

#include "fused_common.cuh"

namespace rsa {
namespace {

struct StreamArgs {
  CUtensorMap tq, tk, tv, tdo;  // q / dO': query rows (chunk); k / v: key rows (key_chunk)
  CUtensorMap tm, td;           // rowmax / dvec as 128-row boxes (bwd_kv_stream)
  CUtensorMap tdq;              // fp32 dQ accumulator, 16-column x 32-row boxes (bwd_*_fused)
  CUtensorMap tp;               // the factored panel, 64-key x 128-row boxes (rsa_bwd_panel_fused)
  Geo g;
  int ck;    // keys per origin chunk
  float sl;  // scale * log2(e)
  const float* rowmax;  // m per query row [rank][b][z][c]
  const float* dvec;    // D * r per query row
  OutView dk, dv, dq_acc, dq_out;
  int dkv_bf16, accumulate;
  int dbg;  // RSA_FS_DBG experiment bits (bwd_stream_fused): 1 no reduce, 2 no staging, 4 no dQ product
  int qsplit;  // one-pass kernels: items per key tile, each over a contiguous share of the query tiles
};

// item = ((origin * B*Z + head) * ntk + key tile) * qsplit + query share
struct OpItem {
  int jo, bz, kt, q0, q1;
  __device__ __forceinline__ OpItem(int item, int qsplit, int ntk, int BZ, int T) {
    const int qs = item % qsplit;
    const int rest = item / qsplit;
    kt = rest % ntk, bz = (rest / ntk) % BZ, jo = rest / (ntk * BZ);
    const int tq = (T + qsplit - 1) / qsplit;
    q0 = qs * tq, q1 = min(T, q0 + tq);
  }
  __device__ __forceinline__ int len() const { return q1 - q0; }
  // the first tile: with one share, each key tile of a head starts at its own tile (kt mod T)
  // and wraps, so concurrent items add into different dQ tiles; with several, the share's first
  __device__ __forceinline__ int start(int qsplit, int T) const { return qsplit == 1 ? kt % T : q0; }
};

// 16 epilogue warps: each thread owns one TMEM lane (a key of the tile in bwd_kv_stream, a
// query in bwd_q_stream) and a quarter of the 128 columns, so four warps per SM
// sub-partition share the MUFU-bound exp2 and hide each other's TMEM / barrier latencies.
constexpr int SE_WARPS = 16;
constexpr int SE_THREADS = 64 + 32 * SE_WARPS;  // 576: 18 warps, 5 on some SMSP (16K registers each): at most 96 registers per thread
constexpr int SE_COLS = 32;                     // columns per thread (128 / (SE_WARPS / 4))

__device__ __forceinline__ int64_t row_index(const Geo& g, int d, int b, int z, int row) {
  return (int64_t(d * g.B + b) * g.Z + z) * g.c + row;
}

// ============================================================ dK / dV
//
// The transposed formulation: a CTA owns a key tile, so every product is written with the
// keys on the TMEM lanes.  S^T = K Q^T and dP'^T = V dO'^T come from shared memory; the
// epilogue thread of key k turns its row of S^T into P~^T (the forward's exp2 of the same
// score, with each query's own reference point) and, with dP'^T, into
// dS^T = P~^T (dP'^T - D') -- and writes both straight back to TMEM (tcgen05.st), where
// they are the A operands of dV += P~^T dO' and dK += dS^T Q (the "TS" tcgen05.mma form:
// A from TMEM, so a 128 x 64 x 16 product reads only its 2 KB B operand from shared memory
// and runs at the 32-clk math rate instead of 48).  Nothing the epilogue produces goes
// through shared memory: no proxy fence, no write-after-read hazard on a P slot.
// The per-query statistics (m, D') arrive by TMA with their query tile.

constexpr int KS_ST = 3;                     // (Q, dO', m, D') stages
constexpr uint32_t KS_STAGE = 2 * TILE + 2 * TR * 4;
constexpr uint32_t KS_OFF_KV = 0;            // [buffer][K | V]
constexpr uint32_t KS_OFF_ST = 4 * TILE;     // [stage][Q | dO' | m | D']
constexpr uint32_t KS_OFF_BAR = KS_OFF_ST + KS_ST * KS_STAGE;
constexpr uint32_t KS_SMEM = KS_OFF_BAR + 512 + 1024;
static_assert(KS_SMEM <= 232448, "bwd_kv_stream smem over the sm_100 per-CTA limit");
// TMEM: S^T [0,128), dP'^T [128,256), P~^T bf16 [256,320), dS^T bf16 [320,384), dV [384,448), dK [448,512)
constexpr uint32_t KS_COL_S = 0, KS_COL_DP = 128, KS_COL_P = 256, KS_COL_DS = 320, KS_COL_DV = 384,
                   KS_COL_DK = 448;

__global__ void __maxnreg__(96) bwd_kv_stream_kernel(const __grid_constant__ StreamArgs p) {
  uint8_t* smem = smem_base();
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + KS_OFF_BAR);
  uint64_t *kv_full = bar, *kv_empty = bar + 2;
  uint64_t *ld_full = bar + 4, *ld_empty = ld_full + KS_ST;
  uint64_t *s_full = ld_empty + KS_ST, *s_empty = s_full + 1;
  uint64_t *dp_full = s_empty + 1, *dp_empty = dp_full + 1;
  uint64_t *p_full = dp_empty + 1, *p_empty = p_full + 1, *ds_full = p_empty + 1, *ds_empty = ds_full + 1;
  uint64_t *acc_full = ds_empty + 1, *acc_empty = acc_full + 1;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 1);

  const Geo& g = p.g;
  const int ntk = (p.ck + TK - 1) / TK, nrt = (g.c + TR - 1) / TR;
  const int T = g.n_rank * nrt;  // query tiles walked per key tile
  const int BZ = g.B * g.Z;
  const int items = g.n_org * BZ * ntk;
  const uint32_t warp = warp_id(), lane = lane_id();

  if (warp == 1) tmem_alloc(tmem_slot, 512);
  if (threadIdx.x == 0) {
    for (int s = 0; s < 2; ++s) mbar_init(&kv_full[s], 1), mbar_init(&kv_empty[s], 1);
    for (int s = 0; s < KS_ST; ++s) mbar_init(&ld_full[s], 1), mbar_init(&ld_empty[s], 1);
    mbar_init(s_full, 1), mbar_init(s_empty, SE_WARPS);
    mbar_init(dp_full, 1), mbar_init(dp_empty, SE_WARPS);
    mbar_init(p_full, SE_WARPS), mbar_init(p_empty, 1);
    mbar_init(ds_full, SE_WARPS), mbar_init(ds_empty, 1);
    mbar_init(acc_full, 1), mbar_init(acc_empty, SE_WARPS);
    fence_barrier_init();
    tma_prefetch(&p.tq), tma_prefetch(&p.tk), tma_prefetch(&p.tv), tma_prefetch(&p.tdo);
    tma_prefetch(&p.tm), tma_prefetch(&p.td);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base(tmem_slot);

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      Pos lq;
      uint32_t it = 0;
      for (int item = blockIdx.x; item < items; item += gridDim.x, ++it) {
        const int kt = item % ntk, bz = (item / ntk) % BZ, jo = item / (ntk * BZ);
        const int b = bz / g.Z, z = bz % g.Z;
        const uint32_t kb = it & 1;
        mbar_wait(&kv_empty[kb], ((it >> 1) & 1) ^ 1);
        mbar_arrive_expect_tx(&kv_full[kb], 2 * TILE);
        uint8_t* kv = smem + KS_OFF_KV + kb * 2 * TILE;
        tma_load_4d(kv, &p.tk, &kv_full[kb], 0, kt * TK, z, jo * g.B + b);
        tma_load_4d(kv + TILE, &p.tv, &kv_full[kb], 0, kt * TK, z, jo * g.B + b);
        for (int t = 0, d = 0, r0 = 0; t < T; ++t, r0 = r0 + TR >= nrt * TR ? (++d, 0) : r0 + TR) {
          const uint32_t s = lq.slot(KS_ST);
          mbar_wait(&ld_empty[s], lq.phase(KS_ST) ^ 1);
          mbar_arrive_expect_tx(&ld_full[s], KS_STAGE);
          uint8_t* st = smem + KS_OFF_ST + s * KS_STAGE;
          tma_load_4d(st, &p.tq, &ld_full[s], 0, r0, z, d * g.B + b);
          tma_load_4d(st + TILE, &p.tdo, &ld_full[s], 0, r0, z, d * g.B + b);
          tma_load_3d(st + 2 * TILE, &p.tm, &ld_full[s], r0, z, d * g.B + b);
          tma_load_3d(st + 2 * TILE + TR * 4, &p.td, &ld_full[s], r0, z, d * g.B + b);
          ++lq.i;
        }
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------- MMA issuer
    const uint32_t idesc_s = idesc_bf16_f32(TK, TR, 0, 0);   // K (K-major) x Q (K-major) -> keys x queries
    const uint32_t idesc_ts = idesc_bf16_f32(TK, HD, 0, 1);  // P~^T / dS^T (TMEM) x dO' / Q (MN-major)
    Pos lq_s, lq_d, lq_v, lq_k;
    uint32_t n_s = 0, n_d = 0, n_p = 0, n_ds = 0, it = 0;
    for (int item = blockIdx.x; item < items; item += gridDim.x, ++it) {
      const uint32_t kb = it & 1;
      const uint32_t ka = smem_u32(smem + KS_OFF_KV + kb * 2 * TILE), va = ka + TILE;
      mbar_wait(&kv_full[kb], (it >> 1) & 1);
      mbar_wait(acc_empty, (it & 1) ^ 1);
      auto issue_s = [&]() {  // S^T(t) = K Q^T
        const uint32_t s = lq_s.slot(KS_ST);
        mbar_wait(&ld_full[s], lq_s.phase(KS_ST));
        mbar_wait(s_empty, (n_s & 1) ^ 1);
        tc_fence_after();
        const uint32_t qa = smem_u32(smem + KS_OFF_ST + s * KS_STAGE);
#pragma unroll
        for (int k = 0; k < HD / 16; ++k)
          umma_bf16_ws(tmem + KS_COL_S, smem_desc_sw128(ka + k * 32, 0, 1024), smem_desc_sw128(qa + k * 32, 0, 1024),
                       idesc_s, k > 0);
        umma_commit_ws(s_full);
        ++lq_s.i, ++n_s;
      };
      auto issue_dp = [&]() {  // dP'^T(t) = V dO'^T
        const uint32_t s = lq_d.slot(KS_ST);
        mbar_wait(&ld_full[s], lq_d.phase(KS_ST));
        mbar_wait(dp_empty, (n_d & 1) ^ 1);
        tc_fence_after();
        const uint32_t doa = smem_u32(smem + KS_OFF_ST + s * KS_STAGE) + TILE;
#pragma unroll
        for (int k = 0; k < HD / 16; ++k)
          umma_bf16_ws(tmem + KS_COL_DP, smem_desc_sw128(va + k * 32, 0, 1024), smem_desc_sw128(doa + k * 32, 0, 1024),
                       idesc_s, k > 0);
        umma_commit_ws(dp_full);
        ++lq_d.i, ++n_d;
      };
      auto issue_dv = [&](int t) {  // dV += P~^T dO' (A from TMEM) once the epilogue has stored P~^T(t)
        const uint32_t s = lq_v.slot(KS_ST);
        mbar_wait(p_full, n_p & 1);
        tc_fence_after();
        const uint32_t doa = smem_u32(smem + KS_OFF_ST + s * KS_STAGE) + TILE;
#pragma unroll
        for (int k = 0; k < TR / 16; ++k)  // 16 queries per step: 8 TMEM columns of A, 2 KB of B
          umma_bf16_ts_ws(tmem + KS_COL_DV, tmem + KS_COL_P + 8 * k, smem_desc_sw128(doa + k * 2048, ATOM, 1024),
                          idesc_ts, (t | k) != 0);
        umma_commit_ws(p_empty);  // P~^T consumed: the next step's may be stored
        ++lq_v.i, ++n_p;
      };
      auto issue_dk = [&](int t) {  // dK += dS^T Q (A from TMEM) once the epilogue has stored dS^T(t)
        const uint32_t s = lq_k.slot(KS_ST);
        mbar_wait(ds_full, n_ds & 1);
        tc_fence_after();
        const uint32_t qa = smem_u32(smem + KS_OFF_ST + s * KS_STAGE);
#pragma unroll
        for (int k = 0; k < TR / 16; ++k)
          umma_bf16_ts_ws(tmem + KS_COL_DK, tmem + KS_COL_DS + 8 * k, smem_desc_sw128(qa + k * 2048, ATOM, 1024),
                          idesc_ts, (t | k) != 0);
        umma_commit_ws(ds_empty);
        umma_commit_ws(&ld_empty[s]);  // the stage's last readers: dK (Q) and the epilogue (m, D', before ds_full)
        ++lq_k.i, ++n_ds;
      };
      issue_s();
      issue_dp();
      for (int t = 0; t < T; ++t) {
        if (t + 1 < T) issue_s();
        issue_dv(t);
        if (t + 1 < T) issue_dp();
        issue_dk(t);
      }
      umma_commit_ws(&kv_empty[kb]);
      umma_commit_ws(acc_full);
    }
  } else {
    // ------------------------------------------------------------ epilogue
    // warp w: TMEM lanes 32*(w%4).. = keys of the tile; query columns part*32 .. +31
    const uint32_t quad = warp & 3;
    const int part = (warp - 2) >> 2;
    const int r = quad * 32 + lane;
    const uint32_t lane_base = (quad * 32u) << 16;
    const float sl = p.sl;
    Pos lq;
    uint32_t n_s = 0, n_d = 0, n_p = 0, n_ds = 0, it = 0;
    for (int item = blockIdx.x; item < items; item += gridDim.x, ++it) {
      const int kt = item % ntk, bz = (item / ntk) % BZ, jo = item / (ntk * BZ);
      const int b = bz / g.Z, z = bz % g.Z, k0 = kt * TK;
      for (int t = 0, r0 = 0; t < T; ++t, r0 = r0 + TR >= nrt * TR ? 0 : r0 + TR) {
        const int nvalid = min(TR, g.c - r0) - part * SE_COLS;  // valid query columns of this part
        const uint32_t s = lq.slot(KS_ST);
        const uint32_t stat = smem_u32(smem + KS_OFF_ST + s * KS_STAGE + 2 * TILE) + part * SE_COLS * 4;
        mbar_wait(&ld_full[s], lq.phase(KS_ST));  // m and D' of the step's queries
        // S^T -> P~^T (the forward's values), back to TMEM as bf16 pairs along the queries
        uint32_t w[16];
        {
          float v[32], m[32];
          mbar_wait(s_full, n_s & 1);
          tc_fence_after();
          __syncwarp();
          tmem_ld32(tmem + lane_base + KS_COL_S + part * SE_COLS, v);
#pragma unroll
          for (int j = 0; j < 32; j += 4) ld_shared_f4(stat + j * 4, m + j);
          tmem_ld_wait();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(s_empty);
          ++n_s;
          exp2_pack32_cols(v, nvalid, sl, m, w);
        }
        mbar_wait(p_empty, (n_p & 1) ^ 1);  // dV(t-1) has read the previous P~^T
        tc_fence_after();
        tmem_st16(tmem + lane_base + KS_COL_P + part * 16, w);
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(p_full);
        ++n_p;
        // dP'^T -> dS^T = P~^T (dP'^T - D') (the 1/sqrt(A) scale is applied to dK at the end)
        {
          float dp[32], dd[32];
          mbar_wait(dp_full, n_d & 1);
          tc_fence_after();
          __syncwarp();
          tmem_ld32(tmem + lane_base + KS_COL_DP + part * SE_COLS, dp);
#pragma unroll
          for (int j = 0; j < 32; j += 4) ld_shared_f4(stat + TR * 4 + j * 4, dd + j);
          tmem_ld_wait();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(dp_empty);
          ++n_d;
#pragma unroll
          for (int e = 0; e < 16; ++e) w[e] = ds_pair2(w[e], dp[2 * e], dp[2 * e + 1], dd[2 * e], dd[2 * e + 1]);
        }
        mbar_wait(ds_empty, (n_ds & 1) ^ 1);  // dK(t-1) has read the previous dS^T
        tc_fence_after();
        tmem_st16(tmem + lane_base + KS_COL_DS + part * 16, w);
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(ds_full);
        ++n_ds, ++lq.i;
      }
      // the key tile's dV (parts 0, 1) and dK (parts 2, 3): 32 columns per thread
      mbar_wait(acc_full, it & 1);
      tc_fence_after();
      float acc[32];
      const bool is_dk = part >= 2;
      const int col = (part & 1) * 32;
      __syncwarp();
      tmem_ld32(tmem + lane_base + (is_dk ? KS_COL_DK : KS_COL_DV) + col, acc);
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(acc_empty);
      if (is_dk) {
#pragma unroll
        for (int e = 0; e < 32; ++e) acc[e] *= g.scale;
      }
      const int key = k0 + r;
      if (key < p.ck) {
        const OutView none{nullptr, 0, 0, 0, 0};
        const OutView& dst = is_dk ? p.dk : p.dv;
        if (p.dkv_bf16) store_row32(none, dst, 0, jo, b, z, key, col, acc);
        else store_row32(dst, none, p.accumulate, jo, b, z, key, col, acc);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, 512);
}

// ================================================================== dQ
//
// Query rows on the TMEM lanes (the forward's orientation): the epilogue turns S into P~ and,
// with dP', into dS, and writes dS straight to TMEM, where it is the A operand of
// dQ += dS K (TS form: only the K tile is read from shared memory).

constexpr int QS_ST = 4;                    // (K, V) stages
constexpr uint32_t QS_OFF_QD = 0;           // [buffer][Q | dO']
constexpr uint32_t QS_OFF_ST = 4 * TILE;    // [stage][K | V]
constexpr uint32_t QS_OFF_BAR = QS_OFF_ST + QS_ST * 2 * TILE;
constexpr uint32_t QS_SMEM = QS_OFF_BAR + 512 + 1024;
static_assert(QS_SMEM <= 232448, "bwd_q_stream smem over the sm_100 per-CTA limit");
// TMEM: S [0,128), dP' [128,256), dS bf16 [256,320), dQ x 2 [320,448)
constexpr uint32_t QS_COL_S = 0, QS_COL_DP = 128, QS_COL_DS = 256, QS_COL_DQ = 320;

__global__ void __maxnreg__(96) bwd_q_stream_kernel(const __grid_constant__ StreamArgs p) {
  uint8_t* smem = smem_base();
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + QS_OFF_BAR);
  uint64_t *qd_full = bar, *qd_empty = bar + 2;
  uint64_t *ld_full = bar + 4, *ld_empty = ld_full + QS_ST;
  uint64_t *s_full = ld_empty + QS_ST, *s_empty = s_full + 1;
  uint64_t *dp_full = s_empty + 1, *dp_empty = dp_full + 1;
  uint64_t *ds_full = dp_empty + 1, *ds_empty = ds_full + 1;
  uint64_t *acc_full = ds_empty + 1, *acc_empty = acc_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);

  const Geo& g = p.g;
  const int ntk = (p.ck + TK - 1) / TK, nrt = (g.c + TR - 1) / TR;
  const int T = g.n_org * ntk;  // key tiles walked per query tile
  const int BZ = g.B * g.Z;
  const int items = g.n_rank * BZ * nrt;
  const uint32_t warp = warp_id(), lane = lane_id();

  if (warp == 1) tmem_alloc(tmem_slot, 512);
  if (threadIdx.x == 0) {
    for (int s = 0; s < 2; ++s) {
      mbar_init(&qd_full[s], 1), mbar_init(&qd_empty[s], 1);
      mbar_init(&acc_full[s], 1), mbar_init(&acc_empty[s], SE_WARPS);
    }
    for (int s = 0; s < QS_ST; ++s) mbar_init(&ld_full[s], 1), mbar_init(&ld_empty[s], 1);
    mbar_init(s_full, 1), mbar_init(s_empty, SE_WARPS);
    mbar_init(dp_full, 1), mbar_init(dp_empty, SE_WARPS);
    mbar_init(ds_full, SE_WARPS), mbar_init(ds_empty, 1);
    fence_barrier_init();
    tma_prefetch(&p.tq), tma_prefetch(&p.tk), tma_prefetch(&p.tv), tma_prefetch(&p.tdo);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base(tmem_slot);

  if (warp == 0) {
    if (lane == 0) {
      Pos lq;
      uint32_t it = 0;
      for (int item = blockIdx.x; item < items; item += gridDim.x, ++it) {
        const int rt = item % nrt, bz = (item / nrt) % BZ, d = item / (nrt * BZ);
        const int b = bz / g.Z, z = bz % g.Z;
        const uint32_t qb = it & 1;
        mbar_wait(&qd_empty[qb], ((it >> 1) & 1) ^ 1);
        mbar_arrive_expect_tx(&qd_full[qb], 2 * TILE);
        uint8_t* qd = smem + QS_OFF_QD + qb * 2 * TILE;
        tma_load_4d(qd, &p.tq, &qd_full[qb], 0, rt * TR, z, d * g.B + b);
        tma_load_4d(qd + TILE, &p.tdo, &qd_full[qb], 0, rt * TR, z, d * g.B + b);
        for (int t = 0, jo = 0, k0 = 0; t < T; ++t, k0 = k0 + TK >= ntk * TK ? (++jo, 0) : k0 + TK) {
          const uint32_t s = lq.slot(QS_ST);
          mbar_wait(&ld_empty[s], lq.phase(QS_ST) ^ 1);
          mbar_arrive_expect_tx(&ld_full[s], 2 * TILE);
          uint8_t* st = smem + QS_OFF_ST + s * 2 * TILE;
          tma_load_4d(st, &p.tk, &ld_full[s], 0, k0, z, jo * g.B + b);
          tma_load_4d(st + TILE, &p.tv, &ld_full[s], 0, k0, z, jo * g.B + b);
          ++lq.i;
        }
      }
    }
  } else if (warp == 1) {
    const uint32_t idesc_s = idesc_bf16_f32(TR, TK, 0, 0);   // Q x K^T, dO' x V^T (K-major both)
    const uint32_t idesc_ts = idesc_bf16_f32(TR, HD, 0, 1);  // dS (TMEM) x K (MN-major)
    Pos lq_s, lq_d, lq_q;
    uint32_t n_s = 0, n_d = 0, n_ds = 0, it = 0;
    for (int item = blockIdx.x; item < items; item += gridDim.x, ++it) {
      const uint32_t qb = it & 1;
      const uint32_t qa = smem_u32(smem + QS_OFF_QD + qb * 2 * TILE), doa = qa + TILE;
      mbar_wait(&qd_full[qb], (it >> 1) & 1);
      mbar_wait(&acc_empty[qb], ((it >> 1) & 1) ^ 1);
      auto issue_s = [&]() {
        const uint32_t s = lq_s.slot(QS_ST);
        mbar_wait(&ld_full[s], lq_s.phase(QS_ST));
        mbar_wait(s_empty, (n_s & 1) ^ 1);
        tc_fence_after();
        const uint32_t ka = smem_u32(smem + QS_OFF_ST + s * 2 * TILE);
#pragma unroll
        for (int k = 0; k < HD / 16; ++k)
          umma_bf16_ws(tmem + QS_COL_S, smem_desc_sw128(qa + k * 32, 0, 1024), smem_desc_sw128(ka + k * 32, 0, 1024),
                       idesc_s, k > 0);
        umma_commit_ws(s_full);
        ++lq_s.i, ++n_s;
      };
      auto issue_dp = [&]() {
        const uint32_t s = lq_d.slot(QS_ST);
        mbar_wait(&ld_full[s], lq_d.phase(QS_ST));
        mbar_wait(dp_empty, (n_d & 1) ^ 1);
        tc_fence_after();
        const uint32_t va = smem_u32(smem + QS_OFF_ST + s * 2 * TILE) + TILE;
#pragma unroll
        for (int k = 0; k < HD / 16; ++k)
          umma_bf16_ws(tmem + QS_COL_DP, smem_desc_sw128(doa + k * 32, 0, 1024), smem_desc_sw128(va + k * 32, 0, 1024),
                       idesc_s, k > 0);
        umma_commit_ws(dp_full);
        ++lq_d.i, ++n_d;
      };
      auto issue_dq = [&](int t) {
        const uint32_t s = lq_q.slot(QS_ST);
        mbar_wait(ds_full, n_ds & 1);
        tc_fence_after();
        const uint32_t ka = smem_u32(smem + QS_OFF_ST + s * 2 * TILE);
#pragma unroll
        for (int k = 0; k < TK / 16; ++k)  // 16 keys per step: 8 TMEM columns of dS, 2 KB of K
          umma_bf16_ts_ws(tmem + QS_COL_DQ + qb * HD, tmem + QS_COL_DS + 8 * k,
                          smem_desc_sw128(ka + k * 2048, ATOM, 1024), idesc_ts, (t | k) != 0);
        umma_commit_ws(ds_empty);
        umma_commit_ws(&ld_empty[s]);
        ++lq_q.i, ++n_ds;
      };
      issue_s();
      issue_dp();
      for (int t = 0; t < T; ++t) {
        if (t + 1 < T) issue_s(), issue_dp();
        issue_dq(t);
      }
      umma_commit_ws(&qd_empty[qb]);
      umma_commit_ws(&acc_full[qb]);
    }
  } else {
    const uint32_t quad = warp & 3;
    const int part = (warp - 2) >> 2;
    const int r = quad * 32 + lane;
    const uint32_t lane_base = (quad * 32u) << 16;
    const float sl = p.sl;
    uint32_t n_s = 0, n_d = 0, n_ds = 0, it = 0;
    for (int item = blockIdx.x; item < items; item += gridDim.x, ++it) {
      const int rt = item % nrt, bz = (item / nrt) % BZ, d = item / (nrt * BZ);
      const int b = bz / g.Z, z = bz % g.Z, row = rt * TR + r;
      const float msl = row < g.c ? __ldg(p.rowmax + row_index(g, d, b, z, row)) : 0.f;
      const float dval = row < g.c ? __ldg(p.dvec + row_index(g, d, b, z, row)) : 0.f;
      const uint64_t nd = neg_pair(dval);
      for (int t = 0, k0 = 0; t < T; ++t, k0 = k0 + TK >= ntk * TK ? 0 : k0 + TK) {
        const int nvalid = min(TK, p.ck - k0) - part * SE_COLS;
        uint32_t w[16];
        {
          float v[32];
          mbar_wait(s_full, n_s & 1);
          tc_fence_after();
          __syncwarp();
          tmem_ld32(tmem + lane_base + QS_COL_S + part * SE_COLS, v);
          tmem_ld_wait();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(s_empty);
          ++n_s;
          exp2_pack32(v, nvalid, sl, msl, w);
        }
        {
          float dp[32];
          mbar_wait(dp_full, n_d & 1);
          tc_fence_after();
          __syncwarp();
          tmem_ld32(tmem + lane_base + QS_COL_DP + part * SE_COLS, dp);
          tmem_ld_wait();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(dp_empty);
          ++n_d;
#pragma unroll
          for (int e = 0; e < 16; ++e) w[e] = ds_pair(w[e], dp[2 * e], dp[2 * e + 1], nd);
        }
        mbar_wait(ds_empty, (n_ds & 1) ^ 1);  // dQ(t-1) has read the previous dS
        tc_fence_after();
        tmem_st16(tmem + lane_base + QS_COL_DS + part * 16, w);
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(ds_full);
        ++n_ds;
      }
      // dQ: parts 0 and 1 read out 32 columns each
      const uint32_t ab = it & 1;
      mbar_wait(&acc_full[ab], (it >> 1) & 1);
      tc_fence_after();
      float o[32];
      __syncwarp();
      if (part < 2) {
        tmem_ld32(tmem + lane_base + QS_COL_DQ + ab * HD + part * 32, o);
        tmem_ld_wait();
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[ab]);
      if (part < 2) {
#pragma unroll
        for (int e = 0; e < 32; ++e) o[e] *= g.scale;
        if (row < g.c) store_row32(p.dq_acc, p.dq_out, p.accumulate, d, b, z, row, part * 32, o);
      }
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, 512);
}

// ====================================================== dQ, dK and dV in one pass
//
// The dK / dV kernel above plus dQ, so S, dP' and every exp2 are computed once instead of
// twice.  Per step (key tile x query tile), keys on the TMEM lanes:
//   S^T = K Q^T                            SS form, issued a step ahead (as bwd_kv_stream)
//   dV += P~^T dO'                         TS form, A = P~^T (bf16) in TMEM
//   dP'^T = V dO'^T                        SS form
//   dK += dS^T Q                           TS form, A = dS^T (bf16) in TMEM
//   dQ_part = dS K_j                       SS form, A = dS in shared memory (MN-major)
// The epilogue writes dS^T to TMEM and to shared memory with the queries contiguous.
// dQ_part(t) lands in the columns dS^T(t) occupied: tcgen05.mma executes in issue order, so
// it overwrites dS^T(t) only after dK(t) (issued before it) has read it, and the epilogue of
// step t+1 reads dQ_part(t) out of exactly the columns it then writes dS^T(t+1) into (each
// thread its own lanes and columns), so the shared buffer needs no barrier beyond
// dQ_part's own completion -- and dP'^T(t+1) can still be issued as soon as dP'^T(t) is
// read.  The epilogue scales dQ_part, stages it per warp (32 rows x 16 columns,
// SWIZZLE_64B) and the
// TMA unit adds it into an fp32 dQ accumulator in L2 (cp.reduce.async.bulk.tensor .add;
// tools/membench/red_bulk: ~5.9 TB/s chip-wide).  So dQ's sum over key tiles is taken in
// arrival order -- not bitwise reproducible, unlike dK / dV (TMEM, fixed order) and the
// two-kernel form.  Items walk the query tiles from their own starting tile (kt mod T) so
// concurrent items of a head add into different dQ tiles.
// (Measured on the way, L = 8192, B4 Z12, against 3016 us for the two kernels: P~^T and
// dS^T taking one TMEM buffer in turn, 3085 us; dS^T in shared memory only, read by dK as a
// K-major SS operand, 2424 us; P~^T / dS^T written over S^T / dP'^T, so S^T(t+1) waits for
// dV(t), 2474 us; P~^T(t) then dQ_part(t) in one buffer, read out before P~^T(t+1) is
// written, 2402 us, with the epilogue waiting on dQ_part at every step; dS^T over dP'^T,
// so dP'^T(t+1) waits for dK(t), 2407 us.)

// The same kernel serves the panel mode (PANEL = true, rsa_bwd_panel_fused): P~ comes from
// the saved factored panel instead of S^T and the exp2 -- the producer loads the step's
// 128 x 128 panel tile with Q and dO', the epilogue reads its key's column of it, and dV is an
// SS product with A = the panel tile read as MN-major (keys contiguous).  One read of the
// panel at any length, where rsa_bwd_dkdv + rsa_bwd_dq read it twice.
// Shared memory: stream stages carry Q | dO' | m | D' (3 deep); panel stages Q | dO' (2 deep)
// with D' in a small ring of its own, and the panel tiles a 2-deep ring whose slot is freed
// as soon as dV and the epilogue's column reads have consumed it (early in the step), so
// two panel tiles are in flight from HBM (with the tile in the Q / dO stage, freed only at
// the step's end, one was: 2644 us at L = 8192, 0.37 of HBM).
template <bool PANEL>
struct FsLayout {
  static constexpr int ST = PANEL ? 2 : 3;
  static constexpr uint32_t STAGE = PANEL ? 2 * TILE : KS_STAGE;
  static constexpr uint32_t OFF_KV = 0;                        // K | V (one buffer)
  static constexpr uint32_t OFF_ST = 2 * TILE;                 // [stage]
  static constexpr uint32_t OFF_P = OFF_ST + ST * STAGE;       // panel mode: [slot] P~ tile
  static constexpr uint32_t OFF_DS = OFF_P + (PANEL ? 2 * PTILE : 0);  // dS: [8-key group][64-query atom][8 keys][128 B]
  static constexpr uint32_t OFF_STG = OFF_DS + PTILE;          // dQ_part staging: [epilogue warp][32 rows][64 B]
  static constexpr uint32_t OFF_D = OFF_STG + SE_WARPS * 2048;  // panel mode: [stage][128] D'
  static constexpr uint32_t OFF_BAR = OFF_D + (PANEL ? ST * TR * 4 : 0);
  static constexpr uint32_t SMEM = OFF_BAR + 512 + 1024;
  static_assert(OFF_DS % 1024 == 0 && OFF_STG % 1024 == 0 && STAGE % 1024 == 0, "swizzled tiles: 1024-byte alignment");
  static_assert(SMEM <= 232448, "bwd_*_fused smem over the sm_100 per-CTA limit");
};
// TMEM: S^T [0,128), dP'^T [128,256), P~^T [256,320), dS^T then dQ_part [320,384), dV [384,448), dK [448,512)
constexpr uint32_t FS_COL_S = 0, FS_COL_DP = 128, FS_COL_P = 256, FS_COL_DSQ = 320, FS_COL_DV = 384,
                   FS_COL_DK = 448;

// Key k's 32 dS values for queries part*32.. (bf16 pairs) into the MN-major SWIZZLE_128B dS
// tile: row k of its 8-key group, 16-byte chunks XOR-swizzled by k % 8.
__device__ __forceinline__ void st_ds_mn(uint32_t tile, uint32_t key, int part, const uint32_t* w) {
  const uint32_t kr = key & 7;
  const uint32_t row = tile + (key >> 3) * 2048 + (part >> 1) * 1024 + kr * 128;
#pragma unroll
  for (int j = 0; j < 4; ++j)
    st_shared_v4(row + ((((part & 1) * 4 + j) ^ kr) << 4), w[4 * j], w[4 * j + 1], w[4 * j + 2], w[4 * j + 3]);
}

// Key k's column of a panel tile: P~ of queries part*32 .. +31 as bf16 pairs (the tile is
// [64-key atom][128 query rows][128 B], SWIZZLE_128B; a warp's 32 keys read 64 contiguous
// bytes of one row per load).
__device__ __forceinline__ void ld_col32(uint32_t tile, uint32_t key, int part, uint32_t* w) {
  const uint32_t base = tile + (key >> 6) * ATOM + (key & 7) * 2, chunk = (key & 63) >> 3;
#pragma unroll
  for (int e = 0; e < 16; ++e) {
    const uint32_t q0 = part * 32 + 2 * e, q1 = q0 + 1;
    uint16_t lo, hi;
    asm volatile("ld.shared.u16 %0, [%1];" : "=h"(lo) : "r"(base + q0 * 128 + ((chunk ^ (q0 & 7)) << 4)));
    asm volatile("ld.shared.u16 %0, [%1];" : "=h"(hi) : "r"(base + q1 * 128 + ((chunk ^ (q1 & 7)) << 4)));
    w[e] = uint32_t(lo) | (uint32_t(hi) << 16);
  }
}

template <bool PANEL>
__global__ void __maxnreg__(96) bwd_onepass_kernel(const __grid_constant__ StreamArgs p) {
  using Lay = FsLayout<PANEL>;
  constexpr int FS_ST = Lay::ST;
  constexpr uint32_t FS_OFF_KV = Lay::OFF_KV, FS_OFF_ST = Lay::OFF_ST, FS_OFF_DS = Lay::OFF_DS,
                     FS_OFF_STG = Lay::OFF_STG, STAGE = Lay::STAGE;
  uint8_t* smem = smem_base();
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + Lay::OFF_BAR);
  uint64_t *kv_full = bar, *kv_empty = bar + 1;
  uint64_t *ld_full = bar + 2, *ld_empty = ld_full + FS_ST;
  uint64_t *s_full = ld_empty + FS_ST, *s_empty = s_full + 1, *dp_full = s_empty + 1, *dp_empty = dp_full + 1;
  uint64_t *p_full = dp_empty + 1, *p_empty = p_full + 1, *ds_full = p_empty + 1, *dq_full = ds_full + 1;
  uint64_t *acc_full = dq_full + 1, *acc_empty = acc_full + 1;
  uint64_t *pp_full = acc_empty + 1, *pp_empty = pp_full + 2;  // panel mode: the P~ tile ring
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(pp_empty + 2);

  const Geo& g = p.g;
  const int ntk = (p.ck + TK - 1) / TK, nrt = (g.c + TR - 1) / TR;
  const int T = g.n_rank * nrt;  // query tiles walked per key tile
  const int BZ = g.B * g.Z;
  const int items = g.n_org * BZ * ntk * p.qsplit;
  const uint32_t warp = warp_id(), lane = lane_id();

  if (warp == 1) tmem_alloc(tmem_slot, 512);
  if (threadIdx.x == 0) {
    mbar_init(kv_full, 1), mbar_init(kv_empty, 1);
    for (int s = 0; s < 2; ++s) mbar_init(&pp_full[s], 1), mbar_init(&pp_empty[s], SE_WARPS + 1);
    for (int s = 0; s < FS_ST; ++s) mbar_init(&ld_full[s], 1), mbar_init(&ld_empty[s], 1);
    mbar_init(s_full, 1), mbar_init(s_empty, SE_WARPS), mbar_init(dp_full, 1), mbar_init(dp_empty, SE_WARPS);
    mbar_init(p_full, SE_WARPS), mbar_init(p_empty, 1), mbar_init(ds_full, SE_WARPS), mbar_init(dq_full, 1);
    mbar_init(acc_full, 1), mbar_init(acc_empty, SE_WARPS);
    fence_barrier_init();
    tma_prefetch(&p.tq), tma_prefetch(&p.tk), tma_prefetch(&p.tv), tma_prefetch(&p.tdo);
    tma_prefetch(&p.td), tma_prefetch(&p.tdq);
    if (PANEL) tma_prefetch(&p.tp);
    else tma_prefetch(&p.tm);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = tmem_base(tmem_slot);

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      const uint64_t pol = l2_evict_first();  // the panel streams through once
      Pos lq, lp;
      uint32_t it = 0;
      for (int item = blockIdx.x; item < items; item += gridDim.x, ++it) {
        const OpItem oi(item, p.qsplit, ntk, BZ, T);
        const int kt = oi.kt, jo = oi.jo, b = oi.bz / g.Z, z = oi.bz % g.Z;
        mbar_wait(kv_empty, (it & 1) ^ 1);
        mbar_arrive_expect_tx(kv_full, 2 * TILE);
        uint8_t* kv = smem + FS_OFF_KV;
        tma_load_4d(kv, &p.tk, kv_full, 0, kt * TK, z, jo * g.B + b);
        tma_load_4d(kv + TILE, &p.tv, kv_full, 0, kt * TK, z, jo * g.B + b);
        const int t0 = oi.start(p.qsplit, T);
        int d = t0 / nrt, r0 = (t0 % nrt) * TR;
        for (int t = 0; t < oi.len(); ++t) {
          if (PANEL) {  // the panel tile first: its slot frees before the stage's
            const uint32_t ps = lp.slot(2);
            mbar_wait(&pp_empty[ps], lp.phase(2) ^ 1);
            mbar_arrive_expect_tx(&pp_full[ps], PTILE);
            uint8_t* pt = smem + Lay::OFF_P + ps * PTILE;
            const int k0 = kt * TK;
            tma_load_5d_hint(pt, &p.tp, &pp_full[ps], k0, g.org_lo + jo, r0, z, d * g.B + b, pol);
            tma_load_5d_hint(pt + ATOM, &p.tp, &pp_full[ps], k0 + 64, g.org_lo + jo, r0, z, d * g.B + b, pol);
            ++lp.i;
          }
          const uint32_t s = lq.slot(FS_ST);
          mbar_wait(&ld_empty[s], lq.phase(FS_ST) ^ 1);
          mbar_arrive_expect_tx(&ld_full[s], PANEL ? STAGE + TR * 4 : STAGE);
          uint8_t* st = smem + FS_OFF_ST + s * STAGE;
          tma_load_4d(st, &p.tq, &ld_full[s], 0, r0, z, d * g.B + b);
          tma_load_4d(st + TILE, &p.tdo, &ld_full[s], 0, r0, z, d * g.B + b);
          if (PANEL) {
            tma_load_3d(smem + Lay::OFF_D + s * TR * 4, &p.td, &ld_full[s], r0, z, d * g.B + b);
          } else {
            tma_load_3d(st + 2 * TILE, &p.tm, &ld_full[s], r0, z, d * g.B + b);
            tma_load_3d(st + 2 * TILE + TR * 4, &p.td, &ld_full[s], r0, z, d * g.B + b);
          }
          ++lq.i;
          if ((r0 += TR) >= nrt * TR) r0 = 0, d = d + 1 == g.n_rank ? 0 : d + 1;
        }
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------- MMA issuer
    const uint32_t idesc_s = idesc_bf16_f32(TK, TR, 0, 0);   // K x Q^T, V x dO'^T -> keys x queries
    const uint32_t idesc_ts = idesc_bf16_f32(TK, HD, 0, 1);  // P~^T / dS^T (TMEM) x dO' / Q (MN-major)
    const uint32_t idesc_dq = idesc_bf16_f32(TR, HD, 1, 1);  // dS (smem, MN-major) x K (MN-major)
    const uint32_t idesc_pv = idesc_bf16_f32(TK, HD, 1, 1);  // panel P~^T (smem, MN-major) x dO' (MN-major)
    const uint32_t ka = smem_u32(smem + FS_OFF_KV), va = ka + TILE, dsa = smem_u32(smem + FS_OFF_DS);
    Pos lq_s, lq_d, lq_v, lq_k, lp;
    uint32_t n_s = 0, n_d = 0, n_p = 0, n_ds = 0, it = 0;
    for (int item = blockIdx.x; item < items; item += gridDim.x, ++it) {
      const int T = OpItem(item, p.qsplit, ntk, BZ, g.n_rank * nrt).len();  // this item's steps
      mbar_wait(kv_full, it & 1);
      auto issue_s = [&]() {  // S^T(t) = K Q^T once the epilogue has read S^T(t-1)
        const uint32_t s = lq_s.slot(FS_ST);
        mbar_wait(&ld_full[s], lq_s.phase(FS_ST));
        mbar_wait(s_empty, (n_s & 1) ^ 1);
        tc_fence_after();
        const uint32_t qa = smem_u32(smem + FS_OFF_ST + s * STAGE);
        umma_ss_x4<2, 2>(tmem + FS_COL_S, smem_desc_sw128(ka, 0, 1024), smem_desc_sw128(qa, 0, 1024), idesc_s, 0);
        umma_commit_ws(s_full);
        ++lq_s.i, ++n_s;
      };
      auto issue_dp = [&]() {  // dP'^T(t) = V dO'^T once the epilogue has read dP'^T(t-1)
        const uint32_t s = lq_d.slot(FS_ST);
        mbar_wait(&ld_full[s], lq_d.phase(FS_ST));
        mbar_wait(dp_empty, (n_d & 1) ^ 1);
        tc_fence_after();
        const uint32_t doa = smem_u32(smem + FS_OFF_ST + s * STAGE) + TILE;
        umma_ss_x4<2, 2>(tmem + FS_COL_DP, smem_desc_sw128(va, 0, 1024), smem_desc_sw128(doa, 0, 1024), idesc_s, 0);
        umma_commit_ws(dp_full);
        ++lq_d.i, ++n_d;
      };
      auto issue_dv = [&](int t) {  // dV += P~^T dO' (A from TMEM, or the panel tile in smem)
        const uint32_t s = lq_v.slot(FS_ST);
        if (PANEL) mbar_wait(&ld_full[s], lq_v.phase(FS_ST)), mbar_wait(&pp_full[lp.slot(2)], lp.phase(2));
        else mbar_wait(p_full, n_p & 1);
        if (t == 0) mbar_wait(acc_empty, (it & 1) ^ 1);  // the previous item's dK / dV are read out
        tc_fence_after();
        const uint32_t sa = smem_u32(smem + FS_OFF_ST + s * STAGE), doa = sa + TILE;
        if (PANEL) {
          const uint32_t ps = lp.slot(2);
          const uint64_t pd = smem_desc_sw128(smem_u32(smem + Lay::OFF_P + ps * PTILE), ATOM, 1024);
          const uint64_t dd = smem_desc_sw128(doa, ATOM, 1024);
          umma_ss_x4<128, 128>(tmem + FS_COL_DV, pd, dd, idesc_pv, t != 0);  // MN-major: +16 query rows (2048 B) per k step
          umma_ss_x4<128, 128>(tmem + FS_COL_DV, pd + 512, dd + 512, idesc_pv, 1);
          umma_commit_ws(&pp_empty[ps]);  // dV's read of the panel tile (the epilogue arrives too)
          ++lp.i;
        } else {
          umma_ts_x4<128>(tmem + FS_COL_DV, tmem + FS_COL_P, smem_desc_sw128(doa, ATOM, 1024), idesc_ts, t != 0);
          umma_ts_x4<128>(tmem + FS_COL_DV, tmem + FS_COL_P + 32, smem_desc_sw128(doa + 8192, ATOM, 1024), idesc_ts, 1);
          umma_commit_ws(p_empty);
        }
        ++lq_v.i, ++n_p;
      };
      auto issue_dk = [&](int t) {  // dK += dS^T Q (A from TMEM)
        const uint32_t s = lq_k.slot(FS_ST);
        mbar_wait(ds_full, n_ds & 1);
        tc_fence_after();
        const uint32_t qa = smem_u32(smem + FS_OFF_ST + s * STAGE);
        umma_ts_x4<128>(tmem + FS_COL_DK, tmem + FS_COL_DSQ, smem_desc_sw128(qa, ATOM, 1024), idesc_ts, t != 0);
        umma_ts_x4<128>(tmem + FS_COL_DK, tmem + FS_COL_DSQ + 32, smem_desc_sw128(qa + 8192, ATOM, 1024), idesc_ts, 1);
        umma_commit_ws(&ld_empty[s]);  // the stage's last readers: dK (Q), dV (dO'), the epilogue (m, D')
        ++lq_k.i, ++n_ds;
      };
      auto issue_dq = [&]() {  // dQ_part = dS K (A = the smem dS tile) over dS^T, which dK has read
        if (!(p.dbg & 4)) {
          // 16 keys per product: two 8-key groups of dS (4 KB), 2 KB of K
          umma_ss_x4<256, 128>(tmem + FS_COL_DSQ, smem_desc_sw128(dsa, 1024, 2048), smem_desc_sw128(ka, ATOM, 1024),
                               idesc_dq, 0);
          umma_ss_x4<256, 128>(tmem + FS_COL_DSQ, smem_desc_sw128(dsa + 16384, 1024, 2048),
                               smem_desc_sw128(ka + 8192, ATOM, 1024), idesc_dq, 1);
        }
        umma_commit_ws(dq_full);
      };
      if (!PANEL) issue_s();
      issue_dp();
      for (int t = 0; t < T; ++t) {
        if (!PANEL && t + 1 < T) issue_s();
        issue_dv(t);
        if (t + 1 < T) issue_dp();
        issue_dk(t);
        issue_dq();
      }
      umma_commit_ws(kv_empty);
      umma_commit_ws(acc_full);
    }
  } else {
    // ------------------------------------------------------------ epilogue
    // warp w: TMEM lanes 32*(w%4).. = keys of the tile (queries for dQ_part); query columns
    // part*32 .. +31 (dQ_part columns part*16 .. +15)
    const uint32_t quad = warp & 3;
    const int part = (warp - 2) >> 2;
    const int r = quad * 32 + lane;
    const uint32_t lane_base = (quad * 32u) << 16;
    const float sl = p.sl;
    const uint32_t dsa = smem_u32(smem + FS_OFF_DS);
    uint8_t* stg = smem + FS_OFF_STG + (warp - 2) * 2048;
    const uint32_t stg_row = smem_u32(stg) + lane * 64, sw = (lane >> 1) & 3;
    Pos lq, lp;
    uint32_t n_s = 0, n_d = 0, n_p = 0, n_dq = 0, it = 0;
    // dQ_part of the previous step (lanes = queries): read out, scaled and staged; the TMA
    // reduce is issued after the step's proxy fence
    auto dq_stage = [&]() {
      float o[16];
      mbar_wait(dq_full, n_dq & 1);
      tc_fence_after();
      __syncwarp();
      tmem_ld16(tmem + lane_base + FS_COL_DSQ + part * 16, o);
      tmem_ld_wait();
      ++n_dq;
      if (p.dbg & 2) return;
      if (lane == 0) tma_store_wait_read<0>();  // this warp's previous reduce has read its staging
      __syncwarp();
#pragma unroll
      for (int j = 0; j < 4; ++j)
        st_shared_v4(stg_row + ((j ^ sw) << 4), __float_as_uint(o[4 * j]), __float_as_uint(o[4 * j + 1]),
                     __float_as_uint(o[4 * j + 2]), __float_as_uint(o[4 * j + 3]));  // 1/sqrt(A) at the cast
    };
    auto dq_reduce = [&](int d, int b, int z, int r0) {
      if (lane == 0 && !(p.dbg & 3)) {
        tma_reduce_add_4d(&p.tdq, stg, part * 16, r0 + int(quad) * 32, z, d * g.B + b);
        tma_store_commit();
      }
    };
    for (int item = blockIdx.x; item < items; item += gridDim.x, ++it) {
      const OpItem oi(item, p.qsplit, ntk, BZ, T);
      const int jo = oi.jo, b = oi.bz / g.Z, z = oi.bz % g.Z, k0 = oi.kt * TK;
      const int t0 = oi.start(p.qsplit, T);
      int d = t0 / nrt, r0 = (t0 % nrt) * TR, pd = 0, pr0 = 0;
      for (int t = 0; t < oi.len(); ++t) {
        const int nvalid = min(TR, g.c - r0) - part * SE_COLS;  // valid query columns of this part
        const uint32_t s = lq.slot(FS_ST);
        const uint32_t stat = smem_u32(smem + FS_OFF_ST + s * STAGE + 2 * TILE) + part * SE_COLS * 4;  // m | D'
        const uint32_t dstat = PANEL ? smem_u32(smem + Lay::OFF_D + s * TR * 4) + part * SE_COLS * 4 : stat + TR * 4;
        mbar_wait(&ld_full[s], lq.phase(FS_ST));  // the step's operands and per-query statistics
        uint32_t w[16];
        if (PANEL) {  // this key's column of the panel tile
          const uint32_t ps = lp.slot(2);
          mbar_wait(&pp_full[ps], lp.phase(2));
          ld_col32(smem_u32(smem + Lay::OFF_P + ps * PTILE), r, part, w);
          __syncwarp();
          if (lane == 0) mbar_arrive(&pp_empty[ps]);
          ++lp.i;
        } else {  // S^T -> P~^T
          float v[32], m[32];
          mbar_wait(s_full, n_s & 1);
          tc_fence_after();
          __syncwarp();
          tmem_ld32(tmem + lane_base + FS_COL_S + part * SE_COLS, v);
#pragma unroll
          for (int j = 0; j < 32; j += 4) ld_shared_f4(stat + j * 4, m + j);
          tmem_ld_wait();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(s_empty);
          ++n_s;
          exp2_pack32_cols(v, nvalid, sl, m, w);
        }
        if (!PANEL) {
          mbar_wait(p_empty, (n_p & 1) ^ 1);  // dV(t-1) has read P~^T(t-1)
          ++n_p;
          tc_fence_after();
          tmem_st16(tmem + lane_base + FS_COL_P + part * 16, w);
          tmem_st_wait();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(p_full);
        }
        // stream mode: dQ_part(t-1) out of the DSQ columns and staged before dP' is awaited, so
        // the staging stores have drained by the step's proxy fence (L = 8K: 2,220 -> 2,200 us;
        // the panel instantiation measured +-0 and keeps the later spot)
        if (!PANEL && t > 0) dq_stage();
        {  // dP'^T -> dS^T = P~^T (dP'^T - D')
          float dp[32], dd[32];
          mbar_wait(dp_full, n_d & 1);
          tc_fence_after();
          __syncwarp();
          tmem_ld32(tmem + lane_base + FS_COL_DP + part * SE_COLS, dp);
#pragma unroll
          for (int j = 0; j < 32; j += 4) ld_shared_f4(dstat + j * 4, dd + j);
          tmem_ld_wait();
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(dp_empty);
          ++n_d;
#pragma unroll
          for (int e = 0; e < 16; ++e) w[e] = ds_pair2(w[e], dp[2 * e], dp[2 * e + 1], dd[2 * e], dd[2 * e + 1]);
        }
        if (PANEL && t > 0) dq_stage();  // frees this thread's DSQ columns (dQ_part(t-1) complete)
        tmem_st16(tmem + lane_base + FS_COL_DSQ + part * 16, w);
        st_ds_mn(dsa, r, part, w);  // dQ_part(t-1), complete above, was the previous dS's last reader
        fence_proxy_async_smem();
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(ds_full);
        if (t > 0) dq_reduce(pd, b, z, pr0);
        ++lq.i;
        pd = d, pr0 = r0;
        if ((r0 += TR) >= nrt * TR) r0 = 0, d = d + 1 == g.n_rank ? 0 : d + 1;
      }
      dq_stage();
      fence_proxy_async_smem();
      __syncwarp();
      dq_reduce(pd, b, z, pr0);
      // the key tile's dV (parts 0, 1) and dK (parts 2, 3): 32 columns per thread
      mbar_wait(acc_full, it & 1);
      tc_fence_after();
      float acc[32];
      const bool is_dk = part >= 2;
      const int col = (part & 1) * 32;
      __syncwarp();
      tmem_ld32(tmem + lane_base + (is_dk ? FS_COL_DK : FS_COL_DV) + col, acc);
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(acc_empty);
      if (is_dk) {
#pragma unroll
        for (int e = 0; e < 32; ++e) acc[e] *= g.scale;
      }
      const int key = k0 + r;
      if (key < p.ck) {
        const OutView none{nullptr, 0, 0, 0, 0};
        const OutView& dst = is_dk ? p.dk : p.dv;
        if (p.qsplit > 1) {  // several items share this key tile: fp32 adds in L2
          float* row = reinterpret_cast<float*>(dst.ptr) + out_off(dst, jo, b, z, key) + col;
#pragma unroll
          for (int e = 0; e < 32; e += 4)
            asm volatile("red.relaxed.gpu.global.add.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(row + e), "f"(acc[e]),
                         "f"(acc[e + 1]), "f"(acc[e + 2]), "f"(acc[e + 3])
                         : "memory");
        } else if (p.dkv_bf16) {
          store_row32(none, dst, 0, jo, b, z, key, col, acc);
        } else {
          store_row32(dst, none, p.accumulate, jo, b, z, key, col, acc);
        }
      }
    }
    if (lane == 0) tma_store_wait_all<0>();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, 512);
}

// dQ = bf16(scale * dq_acc): fp32 [rank][b][z][row][64] contiguous (the unscaled sum of the
// dS K_j partials) into a strided bf16 view, 8 columns per thread.
__global__ void dq_cast_kernel(const float* __restrict__ acc, OutView out, int c, int Z, int B, int64_t rows,
                               float scale) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < rows * 8; i += int64_t(gridDim.x) * blockDim.x) {
    const int64_t row = i >> 3;
    const int col = int(i & 7) * 8;
    const int rr = int(row % c);
    int64_t hb = row / c;
    const int z = int(hb % Z);
    hb /= Z;
    const int b = int(hb % B), d = int(hb / B);
    float4 x = *reinterpret_cast<const float4*>(acc + row * HD + col);
    float4 y = *reinterpret_cast<const float4*>(acc + row * HD + col + 4);
    x.x *= scale, x.y *= scale, x.z *= scale, x.w *= scale, y.x *= scale, y.y *= scale, y.z *= scale, y.w *= scale;
    *reinterpret_cast<uint4*>(reinterpret_cast<__nv_bfloat16*>(out.ptr) + out_off(out, d, b, z, rr) + col) =
        make_uint4(pack_bf16(x.x, x.y), pack_bf16(x.z, x.w), pack_bf16(y.x, y.y), pack_bf16(y.z, y.w));
  }
}

// fp32 dQ accumulator [rank][b][z][row][64] (contiguous) as a 4-D map (col, row, z, b*rank)
// with 16-column x 32-row boxes, SWIZZLE_64B (the staging layout of bwd_stream_fused).
inline bool dq_acc_map(CUtensorMap* m, float* base, const rsa_geom* g) {
  if (!base || !aligned16(base)) return fail(RSA_ERR_UNSUPPORTED, "dq_acc must be 16-byte aligned"), false;
  uint64_t dims[4] = {uint64_t(HD), uint64_t(g->chunk), uint64_t(g->heads), uint64_t(g->batch) * g->n_rank};
  uint64_t str[3] = {uint64_t(HD) * 4, uint64_t(g->chunk) * HD * 4, uint64_t(g->heads) * g->chunk * HD * 4};
  uint32_t box[4] = {16, 32, 1, 1};
  return encode_tmap(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, base, dims, str, box, CU_TENSOR_MAP_SWIZZLE_64B);
}

// How many items share each key tile of a one-pass backward: 1, unless the launch has fewer
// key-tile items than SMs (the Linformer's few projected keys: B*Z*2 items over ~10^3 query
// tiles each) and dK/dV are fp32 outputs laid out contiguously, which the items then add
// into (red.global.add) after a zero-fill.
inline int onepass_qsplit(const rsa_geom* g, int dkv_bf16, const rsa_view& dk, const rsa_view& dv) {
  const int ck = key_chunk(g), ntk = (ck + TK - 1) / TK;
  const int64_t base = int64_t(g->n_org) * g->batch * g->heads * ntk;
  const int T = g->n_rank * ((g->chunk + TR - 1) / TR);
  const int sms = num_sms();
  if (dkv_bf16 || base >= sms || T < 16) return 1;
  auto dense = [&](const rsa_view& x) {
    return x.s_row == HD && x.s_z == int64_t(ck) * HD && x.s_b == int64_t(g->heads) * ck * HD &&
           (g->n_org == 1 || x.s_rank == int64_t(g->batch) * g->heads * ck * HD);
  };
  if (!dense(dk) || !dense(dv)) return 1;
  static const int per_sm = [] {  // experiment switch: items per SM to aim for (RSA_OP_ITEMS_PER_SM)
    const char* e = getenv("RSA_OP_ITEMS_PER_SM");
    return e ? std::max(1, atoi(e)) : 4;
  }();
  int qs = int(std::min<int64_t>((per_sm * sms + base - 1) / base, T / 8));
  const int tq = (T + qs - 1) / qs;
  return (T + tq - 1) / tq;  // no empty share
}

inline int onepass_zero_dkv(const rsa_geom* g, int qsplit, int accumulate, const rsa_view& dk, const rsa_view& dv,
                            cudaStream_t st) {
  if (qsplit == 1 || accumulate) return RSA_OK;
  const size_t bytes = size_t(g->n_org) * g->batch * g->heads * key_chunk(g) * HD * 4;
  if (cudaMemsetAsync(dk.ptr, 0, bytes, st) != cudaSuccess || cudaMemsetAsync(dv.ptr, 0, bytes, st) != cudaSuccess)
    return check_launch("one-pass backward: dK / dV zero-fill");
  return RSA_OK;
}

int dq_cast(const float* dq_acc, const rsa_view& dq_out, const rsa_geom* g, int64_t rows, cudaStream_t st) {
  const int64_t work = rows * 8;
  const int blocks = int(std::min<int64_t>((work + 255) / 256, int64_t(num_sms()) * 8));
  dq_cast_kernel<<<blocks, 256, 0, st>>>(dq_acc, to_out(dq_out), g->chunk, g->heads, g->batch, rows, g->scale);
  return check_launch("dq_cast_kernel");
}

bool stream_args(StreamArgs* a, const rsa_geom* g, rsa_view q, rsa_view k, rsa_view v, rsa_view dout,
                 const float* rowmax, const float* dvec) {
  if (!head_map(&a->tq, q, g, g->n_rank) || !head_map(&a->tdo, dout, g, g->n_rank) ||
      !head_map(&a->tk, k, g, g->n_org, key_chunk(g)) || !head_map(&a->tv, v, g, g->n_org, key_chunk(g)))
    return false;
  if (!rows_map(&a->tm, rowmax, g, g->n_rank) || !rows_map(&a->td, dvec, g, g->n_rank)) return false;
  a->g = to_geo(g);
  a->ck = key_chunk(g);
  a->sl = g->scale * LOG2E;
  a->rowmax = rowmax;
  a->dvec = dvec;
  return true;
}

}  // namespace
}  // namespace rsa

extern "C" {

int rsa_bwd_kv_stream(const rsa_geom* g, rsa_view q, rsa_view k, rsa_view v, rsa_view dout_scaled,
                      const float* rowmax, const float* dvec, rsa_view dk, rsa_view dv, int dkv_dtype,
                      int accumulate, void* stream) {
  using namespace rsa;
  if (!geom_ok_keys(g) || !rowmax || !dvec) return fail(RSA_ERR_INVALID, "rsa_bwd_kv_stream: unsupported geometry");
  const int esz = dkv_dtype == RSA_BF16 ? 2 : 4;
  if (!dk.ptr || !dv.ptr || !out_ok(dk, esz) || !out_ok(dv, esz))
    return fail(RSA_ERR_UNSUPPORTED, "rsa_bwd_kv_stream: output views missing or misaligned");
  StreamArgs a{};
  if (!stream_args(&a, g, q, k, v, dout_scaled, rowmax, dvec)) return RSA_ERR_UNSUPPORTED;
  a.dk = to_out(dk);
  a.dv = to_out(dv);
  a.dkv_bf16 = dkv_dtype == RSA_BF16;
  a.accumulate = accumulate;
  const int items = g->n_org * g->batch * g->heads * ((key_chunk(g) + TK - 1) / TK);
  return launch(bwd_kv_stream_kernel, items, KS_SMEM, a, stream, "bwd_kv_stream_kernel", SE_THREADS);
}

int rsa_bwd_q_stream(const rsa_geom* g, rsa_view q, rsa_view k, rsa_view v, rsa_view dout_scaled,
                     const float* rowmax, const float* dvec, rsa_view dq_acc, int accumulate, rsa_view dq_out,
                     void* stream) {
  using namespace rsa;
  if (!geom_ok_keys(g) || !rowmax || !dvec) return fail(RSA_ERR_INVALID, "rsa_bwd_q_stream: unsupported geometry");
  if ((!dq_acc.ptr && !dq_out.ptr) || !out_ok(dq_acc, 4) || !out_ok(dq_out, 2))
    return fail(RSA_ERR_UNSUPPORTED, "rsa_bwd_q_stream: output views missing or misaligned");
  StreamArgs a{};
  if (!stream_args(&a, g, q, k, v, dout_scaled, rowmax, dvec)) return RSA_ERR_UNSUPPORTED;
  a.dq_acc = to_out(dq_acc);
  a.dq_out = to_out(dq_out);
  a.accumulate = accumulate;
  const int items = g->n_rank * g->batch * g->heads * ((g->chunk + TR - 1) / TR);
  return launch(bwd_q_stream_kernel, items, QS_SMEM, a, stream, "bwd_q_stream_kernel", SE_THREADS);
}

int rsa_bwd_stream_fused(const rsa_geom* g, rsa_view q, rsa_view k, rsa_view v, rsa_view dout_scaled,
                         const float* rowmax, const float* dvec, rsa_view dk, rsa_view dv, int dkv_dtype,
                         int accumulate_dkv, float* dq_acc, int accumulate_dq, rsa_view dq_out, void* stream) {
  using namespace rsa;
  if (!geom_ok_keys(g) || !rowmax || !dvec) return fail(RSA_ERR_INVALID, "rsa_bwd_stream_fused: unsupported geometry");
  const int esz = dkv_dtype == RSA_BF16 ? 2 : 4;
  if (!dk.ptr || !dv.ptr || !out_ok(dk, esz) || !out_ok(dv, esz) || !out_ok(dq_out, 2))
    return fail(RSA_ERR_UNSUPPORTED, "rsa_bwd_stream_fused: output views missing or misaligned");
  StreamArgs a{};
  if (!stream_args(&a, g, q, k, v, dout_scaled, rowmax, dvec) || !dq_acc_map(&a.tdq, dq_acc, g))
    return RSA_ERR_UNSUPPORTED;
  a.dk = to_out(dk);
  a.dv = to_out(dv);
  a.dkv_bf16 = dkv_dtype == RSA_BF16;
  a.accumulate = accumulate_dkv;
  static const int dbg = [] {  // experiment switch (tools/fs_exp.py), read once
    const char* e = getenv("RSA_FS_DBG");
    return e ? atoi(e) : 0;
  }();
  a.dbg = dbg;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const int64_t rows = int64_t(g->n_rank) * g->batch * g->heads * g->chunk;
  if (!accumulate_dq && cudaMemsetAsync(dq_acc, 0, size_t(rows) * HD * 4, st) != cudaSuccess)
    return check_launch("rsa_bwd_stream_fused: dq_acc memset");
  a.qsplit = onepass_qsplit(g, a.dkv_bf16, dk, dv);
  if (int rc = onepass_zero_dkv(g, a.qsplit, accumulate_dkv, dk, dv, st)) return rc;
  const int items = g->n_org * g->batch * g->heads * ((key_chunk(g) + TK - 1) / TK) * a.qsplit;
  const int rc = launch(bwd_onepass_kernel<false>, items, FsLayout<false>::SMEM, a, stream, "bwd_onepass_kernel<stream>",
                        SE_THREADS);
  if (rc != RSA_OK || !dq_out.ptr) return rc;
  return dq_cast(dq_acc, dq_out, g, rows, st);
}

int rsa_bwd_panel_fused(const rsa_geom* g, rsa_view q, rsa_view k, rsa_view v, rsa_view dout_scaled, rsa_view panel,
                        const float* dvec, rsa_view dk, rsa_view dv, int dkv_dtype, int accumulate_dkv, float* dq_acc,
                        int accumulate_dq, rsa_view dq_out, void* stream) {
  using namespace rsa;
  if (!geom_ok(g) || !dvec) return fail(RSA_ERR_INVALID, "rsa_bwd_panel_fused: unsupported geometry");
  const int esz = dkv_dtype == RSA_BF16 ? 2 : 4;
  if (!dk.ptr || !dv.ptr || !out_ok(dk, esz) || !out_ok(dv, esz) || !out_ok(dq_out, 2))
    return fail(RSA_ERR_UNSUPPORTED, "rsa_bwd_panel_fused: output views missing or misaligned");
  StreamArgs a{};
  if (!head_map(&a.tq, q, g, g->n_rank) || !head_map(&a.tdo, dout_scaled, g, g->n_rank) ||
      !head_map(&a.tk, k, g, g->n_org) || !head_map(&a.tv, v, g, g->n_org) || !panel_map(&a.tp, panel, g, g->n_rank) ||
      !rows_map(&a.td, dvec, g, g->n_rank) || !dq_acc_map(&a.tdq, dq_acc, g))
    return RSA_ERR_UNSUPPORTED;
  a.g = to_geo(g);
  a.ck = g->chunk;
  a.dvec = dvec;
  a.dk = to_out(dk);
  a.dv = to_out(dv);
  a.dkv_bf16 = dkv_dtype == RSA_BF16;
  a.accumulate = accumulate_dkv;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const int64_t rows = int64_t(g->n_rank) * g->batch * g->heads * g->chunk;
  if (!accumulate_dq && cudaMemsetAsync(dq_acc, 0, size_t(rows) * HD * 4, st) != cudaSuccess)
    return check_launch("rsa_bwd_panel_fused: dq_acc memset");
  a.qsplit = onepass_qsplit(g, a.dkv_bf16, dk, dv);
  if (int rc = onepass_zero_dkv(g, a.qsplit, accumulate_dkv, dk, dv, st)) return rc;
  const int items = g->n_org * g->batch * g->heads * ((g->chunk + TK - 1) / TK) * a.qsplit;
  const int rc = launch(bwd_onepass_kernel<true>, items, FsLayout<true>::SMEM, a, stream, "bwd_onepass_kernel<panel>",
                        SE_THREADS);
  if (rc != RSA_OK || !dq_out.ptr) return rc;
  return dq_cast(dq_acc, dq_out, g, rows, st);
}

}  // extern "C"

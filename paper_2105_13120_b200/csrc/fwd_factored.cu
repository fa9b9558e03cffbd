// Factored-panel RSA forward for sm_100a (head size A = 64, every origin
// resident): the probability panel is saved as P~ = 2^(s*sl - m) (bf16, the
// row max m taken over the whole row) plus one fp32 row scale r = 1 / sum(P~),
// so the reference's probs are P = r * P~ (ringseq/ring_attention.py:89-94,
// ringseq/tensor_ops.py:75-84) and its output O = P V = r * (P~ V)
// (ringseq/ring_attention.py:97-103).
//
// Why factored: the normalised panel needs the row sum before the first
// probability can be written, which costs a second exponential per panel
// element (fused.cu's pass A: max AND sum).  Here pass A is a max-only scan
// of S = Q K^T, pass B is one exp2 per element, and the row sum comes from
// the tensor core: the P~ V product runs with N = 80, whose last 16 B-operand
// columns read a constant block of bf16 ones, so TMEM column 64 of the O
// accumulator holds sum_k P~[row, k] -- the sum of exactly the rounded values
// written to the panel.  The panel bytes are the same as the normalised
// panel's (2 per element) plus 4 bytes per row.
//
// Roles and buffers follow fwd_kernel (fused.cu): warp 0 TMA producer, warp 1
// tcgen05.mma issuer (owns TMEM), warps 2..9 epilogue (TMEM lane quarter
// w % 4, column half (w - 2) / 4).  TMEM: S double buffer [0, 256), O double
// buffer at 256 + 128 * ob (80 columns each).
#include "fused_common.cuh"

namespace rsa {
namespace {

struct FfArgs {
  CUtensorMap tq, tk, tv, tp;
  Geo g;
  float sl;  // scale * log2(e)
  int* flag;
  OutView o_out;
  float* rowscale;  // [rank][b][z][c]
};

constexpr int FF_KST = 3, FF_VST = 2;
constexpr int PV_N = HD + 16;  // O columns + 16 row-sum columns
constexpr uint32_t FF_OFF_Q = 0;
constexpr uint32_t FF_OFF_K = FF_OFF_Q + 2 * TILE;
constexpr uint32_t FF_OFF_V = FF_OFF_K + FF_KST * TILE;
constexpr uint32_t FF_OFF_ONES = FF_OFF_V + FF_VST * TILE;  // 128 rows x 128 B of bf16 1.0
constexpr uint32_t FF_OFF_P = FF_OFF_ONES + TILE;
constexpr uint32_t FF_OFF_X = FF_OFF_P + 2 * PTILE;  // row-max exchange, 2 x 256 floats
constexpr uint32_t FF_OFF_BAR = FF_OFF_X + 2 * EPI_THREADS * 4;
constexpr uint32_t FF_SMEM = FF_OFF_BAR + 512 + 1024;
constexpr uint32_t COL_O = 2 * TK;
static_assert(FF_SMEM <= 232448, "fwd_factored smem over the sm_100 per-CTA limit");

// The two epilogue warps holding the two column halves of the same 32 rows.
__device__ __forceinline__ void bar_rows(uint32_t quad) {
  asm volatile("bar.sync %0, 64;" ::"r"(4 + quad) : "memory");
}

__device__ __forceinline__ float tmem_ld1(uint32_t taddr) {
  uint32_t r;
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];" : "=r"(r) : "r"(taddr));
  return __uint_as_float(r);
}

__global__ void __launch_bounds__(NTHREADS, 1) fwd_factored_kernel(const __grid_constant__ FfArgs p) {
  uint8_t* smem = smem_base();
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + FF_OFF_BAR);
  uint64_t *q_full = bar, *q_empty = bar + 2, *k_full = bar + 4, *k_empty = k_full + FF_KST;
  uint64_t *v_full = k_empty + FF_KST, *v_empty = v_full + FF_VST;
  uint64_t *s_full = v_empty + FF_VST, *s_empty = s_full + 2, *p_full = s_empty + 2, *p_empty = p_full + 2;
  uint64_t *o_full = p_empty + 2, *o_empty = o_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(o_empty + 2);

  const Geo& g = p.g;
  const int ntk = (g.c + TK - 1) / TK, nrt = (g.c + TR - 1) / TR;
  const int T = g.n_org * ntk;
  const int BZ = g.B * g.Z;
  const int items = g.n_rank * BZ * nrt;
  const uint32_t warp = warp_id(), lane = lane_id();

  {  // constant B-operand block of ones (read by the async proxy)
    uint4* ones = reinterpret_cast<uint4*>(smem + FF_OFF_ONES);
    for (uint32_t i = threadIdx.x; i < TILE / 16; i += NTHREADS) ones[i] = make_uint4(0x3F803F80u, 0x3F803F80u, 0x3F803F80u, 0x3F803F80u);
    fence_proxy_async_smem();
  }
  if (warp == 1) tmem_alloc(tmem_slot, 512);
  if (threadIdx.x == 0) {
    for (int s = 0; s < 2; ++s) {
      mbar_init(&q_full[s], 1), mbar_init(&q_empty[s], 1);
      mbar_init(&s_full[s], 1), mbar_init(&s_empty[s], EPI_WARPS);
      mbar_init(&p_full[s], EPI_WARPS), mbar_init(&p_empty[s], 1);
      mbar_init(&o_full[s], 1), mbar_init(&o_empty[s], EPI_WARPS);
    }
    for (int s = 0; s < FF_KST; ++s) mbar_init(&k_full[s], 1), mbar_init(&k_empty[s], 1);
    for (int s = 0; s < FF_VST; ++s) mbar_init(&v_full[s], 1), mbar_init(&v_empty[s], 1);
    fence_barrier_init();
    tma_prefetch(&p.tq), tma_prefetch(&p.tk), tma_prefetch(&p.tv), tma_prefetch(&p.tp);
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------ producer
    if (lane == 0) {
      Pos kq, vq;
      uint32_t it = 0;
      for (int item = blockIdx.x; item < items; item += gridDim.x, ++it) {
        const int rt = item % nrt, bz = (item / nrt) % BZ, d = item / (nrt * BZ);
        const int b = bz / g.Z, z = bz % g.Z;
        const int qb = it & 1;
        mbar_wait(&q_empty[qb], ((it >> 1) & 1) ^ 1);
        mbar_arrive_expect_tx(&q_full[qb], TILE);
        tma_load_4d(smem + FF_OFF_Q + qb * TILE, &p.tq, &q_full[qb], 0, rt * TR, z, d * g.B + b);
        for (int pass = 0; pass < 2; ++pass) {
          for (int t = 0; t < T; ++t) {
            const int jo = t / ntk, k0 = (t % ntk) * TK;
            const uint32_t ks = kq.slot(FF_KST);
            mbar_wait(&k_empty[ks], kq.phase(FF_KST) ^ 1);
            mbar_arrive_expect_tx(&k_full[ks], TILE);
            tma_load_4d(smem + FF_OFF_K + ks * TILE, &p.tk, &k_full[ks], 0, k0, z, (g.org_lo + jo) * g.B + b);
            ++kq.i;
            if (pass == 1) {
              const uint32_t vs = vq.slot(FF_VST);
              mbar_wait(&v_empty[vs], vq.phase(FF_VST) ^ 1);
              mbar_arrive_expect_tx(&v_full[vs], TILE);
              tma_load_4d(smem + FF_OFF_V + vs * TILE, &p.tv, &v_full[vs], 0, k0, z, (g.org_lo + jo) * g.B + b);
              ++vq.i;
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------------------------------------------------- MMA issuer
    const uint32_t idesc_s = idesc_bf16_f32(TR, TK, 0, 0);
    const uint32_t idesc_o = idesc_bf16_f32(TR, PV_N, 0, 1);
    Pos kq, vq, sq, pq;
    uint32_t it = 0;
    for (int item = blockIdx.x; item < items; item += gridDim.x, ++it) {
      const int qb = it & 1;
      mbar_wait(&q_full[qb], (it >> 1) & 1);
      const uint32_t qa = smem_u32(smem + FF_OFF_Q + qb * TILE);
      auto issue_s = [&]() {
        const uint32_t ks = kq.slot(FF_KST), sb = sq.slot(2);
        mbar_wait(&k_full[ks], kq.phase(FF_KST));
        mbar_wait(&s_empty[sb], sq.phase(2) ^ 1);
        tc_fence_after();
        const uint32_t ka = smem_u32(smem + FF_OFF_K + ks * TILE);
#pragma unroll
        for (int k = 0; k < HD / 16; ++k)
          umma_bf16_ws(tmem + sb * TK, smem_desc_sw128(qa + k * 32, 0, 1024), smem_desc_sw128(ka + k * 32, 0, 1024),
                       idesc_s, k > 0);
        umma_commit_ws(&k_empty[ks]);
        umma_commit_ws(&s_full[sb]);
        ++kq.i, ++sq.i;
      };
      for (int t = 0; t < T; ++t) issue_s();  // pass A: row max
      const uint32_t ob = it & 1;
      mbar_wait(&o_empty[ob], ((it >> 1) & 1) ^ 1);
      issue_s();
      for (int t = 0; t < T; ++t) {  // pass B: P~ and O~ = P~ [V | 1]
        if (t + 1 < T) issue_s();
        const uint32_t pb = pq.slot(2), vs = vq.slot(FF_VST);
        mbar_wait(&p_full[pb], pq.phase(2));
        mbar_wait(&v_full[vs], vq.phase(FF_VST));
        tc_fence_after();
        const uint32_t pa = smem_u32(smem + FF_OFF_P + pb * PTILE);
        const uint32_t va = smem_u32(smem + FF_OFF_V + vs * TILE);
        const uint32_t lbo = FF_OFF_ONES - (FF_OFF_V + vs * TILE);  // second 64-column atom: the ones block
#pragma unroll
        for (int k = 0; k < TK / 16; ++k)
          umma_bf16_ws(tmem + COL_O + ob * 128, smem_desc_sw128(pa + (k >> 2) * ATOM + (k & 3) * 32, 0, 1024),
                       smem_desc_sw128(va + k * 2048, lbo, 1024), idesc_o, (t | k) != 0);
        umma_commit_ws(&v_empty[vs]);
        umma_commit_ws(&p_empty[pb]);
        ++pq.i, ++vq.i;
      }
      umma_commit_ws(&o_full[ob]);
      umma_commit_ws(&q_empty[qb]);
    }
  } else {
    // ------------------------------------------------------------ epilogue
    const uint32_t quad = warp & 3;
    const int half = (warp - 2) >> 2;
    const int r = quad * 32 + lane;
    const int et = threadIdx.x - 64;  // 0..255
    const bool storer = (lane == 0) && (quad == 2);
    const uint32_t lane_base = (quad * 32u) << 16;
    const uint32_t xbase = smem_u32(smem + FF_OFF_X);
    const uint32_t pbase = smem_u32(smem + FF_OFF_P);
    const float sl = p.sl;
    const OutView none{nullptr, 0, 0, 0, 0};
    Pos sq, pq;
    uint32_t it = 0;
    bool bad = false;
    auto load_s = [&](float* v) {
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
      // ---- pass A: raw row max (and the non-finite check) over every key
      float m = -INFINITY;
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
        m = fmaxf(m, cmax);
      }
      {  // combine the two column halves of each row
        const uint32_t slot = xbase + ((it & 1) * EPI_THREADS) * 4;
        asm volatile("st.shared.f32 [%0], %1;" ::"r"(slot + et * 4), "f"(m) : "memory");
        bar_rows(quad);
        float o;
        asm volatile("ld.shared.f32 %0, [%1];" : "=f"(o) : "r"(slot + ((et + 128) & 255) * 4) : "memory");
        m = fmaxf(m, o);
      }
      const float msl = (m == -INFINITY || !(fabsf(m) <= 3.402823466e38f)) ? 0.f : m * sl;
      // ---- pass B: P~ = 2^(s*sl - m*sl) -> smem -> TMA store; UMMA accumulates P~ [V | 1]
      int jo = 0;
      k0 = 0;
      for (int t = 0; t < T; ++t) {
        const uint32_t pb = pq.slot(2);
        const int nvalid = min(TK, g.c - k0) - half * 64;
        float v[64];
        load_s(v);
        if (nvalid >= 64) {
#pragma unroll
          for (int e = 0; e < 64; ++e) v[e] = fast_exp2(fmaf(v[e], sl, -msl));
        } else {
#pragma unroll
          for (int e = 0; e < 64; ++e) v[e] = e < nvalid ? fast_exp2(fmaf(v[e], sl, -msl)) : 0.f;
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
            tma_store_5d(&p.tp, smem + FF_OFF_P + pb * PTILE + half * ATOM, k0 + half * 64, g.org_lo + jo, rt * TR,
                         z, d * g.B + b);
          tma_store_commit();
        }
        ++pq.i;
        if (k0 + TK >= g.c) k0 = 0, ++jo;
        else k0 += TK;
      }
      // ---- O = O~ / l, r = 1 / l (l >= 1: the max element contributes 2^0)
      const uint32_t ob = it & 1;
      mbar_wait(&o_full[ob], (it >> 1) & 1);
      tc_fence_after();
      float o[32];
      __syncwarp();
      tmem_ld32(tmem + lane_base + COL_O + ob * 128 + half * 32, o);
      const float l = tmem_ld1(tmem + lane_base + COL_O + ob * 128 + HD);
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&o_empty[ob]);
      const float rinv = 1.f / l;
#pragma unroll
      for (int e = 0; e < 32; ++e) o[e] *= rinv;
      if (row < g.c) {
        store_row32(none, p.o_out, 0, d, b, z, row, half * 32, o);
        if (half == 0) p.rowscale[(int64_t(d * g.B + b) * g.Z + z) * g.c + row] = rinv;
      }
    }
    if (bad && p.flag) atomicExch(p.flag, 1);
    if (storer) tma_store_wait_all<0>();
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) tmem_dealloc(tmem, 512);
}

}  // namespace
}  // namespace rsa

extern "C" {

int rsa_fwd_factored(const rsa_geom* g, rsa_view q, rsa_view k, rsa_view v, rsa_view panel, rsa_view o_out,
                     float* rowscale, int* nonfinite_flag, void* stream) {
  using namespace rsa;
  if (!geom_ok(g)) return fail(RSA_ERR_INVALID, "rsa_fwd_factored: unsupported geometry");
  if (g->org_lo != 0 || g->n_org != g->seq_len / g->chunk)
    return fail(RSA_ERR_INVALID, "rsa_fwd_factored: every origin must be resident (org_lo = 0, n_org = L / c)");
  if (!rowscale || !o_out.ptr || !out_ok(o_out, 2))
    return fail(RSA_ERR_UNSUPPORTED, "rsa_fwd_factored: output / row-scale buffers missing or misaligned");
  FfArgs a{};
  if (!head_map(&a.tq, q, g, g->n_rank) || !head_map(&a.tk, k, g, g->n_org) || !head_map(&a.tv, v, g, g->n_org) ||
      !panel_map(&a.tp, panel, g, g->n_rank))
    return RSA_ERR_UNSUPPORTED;
  a.g = to_geo(g);
  a.sl = g->scale * LOG2E;
  a.flag = nonfinite_flag;
  a.o_out = to_out(o_out);
  a.rowscale = rowscale;
  const int items = g->n_rank * g->batch * g->heads * ((g->chunk + TR - 1) / TR);
  return launch(fwd_factored_kernel, items, FF_SMEM, a, stream, "fwd_factored_kernel");
}

}  // extern "C"

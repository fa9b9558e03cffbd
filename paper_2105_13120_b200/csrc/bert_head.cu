// BERT harness kernels around the RSA encoder: the
// embedding lookup at the bottom of the stack and the masked-LM loss at the top, so a
// timed step is the paper's whole-model BERT training step rather than
// the encoder layers alone.  The reference has neither (it is an attention simulator);
// these are harness pieces, not the RSA hot path.
//
//   rsa_embed        x[row] = tok[ids[row]] + pos[position(row)] for rows laid out
//                    [rank][b][i] (rank d holds positions d*c .. d*c + c - 1: the
//                    contiguous chunk layout of ringseq/cluster.py:73-88)
//   rsa_embed_bwd    dtok[ids[row]] += dx[row] (fp32 atomics: the one non-deterministic
//                    sum in this repository, confined to the harness's token-embedding
//                    gradient); dpos likewise when given (the harness instead sums the
//                    batch with rsa_sum_ranks: 64-way contention per address otherwise)
//   rsa_softmax_xent per masked row: loss = logsumexp(logits) - logits[target] and
//                    dlogits = (softmax(logits) - onehot(target)) * grad_scale, one CTA
//                    per row, one read pass (online max / sum) and one write pass
#include "common.h"
#include "ptx.cuh"

namespace rsa {
namespace {

__device__ __forceinline__ int64_t embed_position(int64_t row, int64_t per_rank, int64_t c) {
  return (row / per_rank) * c + row % c;  // rank * c + position within the chunk
}

// one warp per row, 8 bf16 (16 bytes) per lane per step
__global__ void __launch_bounds__(256) embed_kernel(const int* __restrict__ ids, int64_t rows,
                                                    const __nv_bfloat16* __restrict__ tok,
                                                    const __nv_bfloat16* __restrict__ pos, int64_t h,
                                                    int64_t per_rank, int64_t c, __nv_bfloat16* __restrict__ x) {
  const int64_t row = int64_t(blockIdx.x) * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;
  const __nv_bfloat16* t = tok + int64_t(ids[row]) * h;
  const __nv_bfloat16* p = pos + embed_position(row, per_rank, c) * h;
  for (int64_t col = lane * 8; col < h; col += 256) {
    const uint4 a = *reinterpret_cast<const uint4*>(t + col);
    const uint4 b = *reinterpret_cast<const uint4*>(p + col);
    const uint32_t aw[4] = {a.x, a.y, a.z, a.w}, bw[4] = {b.x, b.y, b.z, b.w};
    uint32_t o[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float2 fa = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&aw[e]));
      const float2 fb = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&bw[e]));
      o[e] = pack_bf16(fa.x + fb.x, fa.y + fb.y);
    }
    *reinterpret_cast<uint4*>(x + row * h + col) = make_uint4(o[0], o[1], o[2], o[3]);
  }
}

__global__ void __launch_bounds__(256) embed_bwd_kernel(const int* __restrict__ ids, int64_t rows,
                                                        const __nv_bfloat16* __restrict__ dx, int64_t h,
                                                        int64_t per_rank, int64_t c, float* __restrict__ dtok,
                                                        float* __restrict__ dpos) {
  const int64_t row = int64_t(blockIdx.x) * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;
  float* t = dtok + int64_t(ids[row]) * h;
  float* p = dpos ? dpos + embed_position(row, per_rank, c) * h : nullptr;
  for (int64_t col = lane * 2; col < h; col += 64) {
    const float2 g = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(dx + row * h + col));
    atomicAdd(t + col, g.x), atomicAdd(t + col + 1, g.y);
    if (p) atomicAdd(p + col, g.x), atomicAdd(p + col + 1, g.y);
  }
}

__device__ __forceinline__ void online_merge(float& m, float& s, float m2, float s2) {
  const float mn = fmaxf(m, m2);
  if (mn == -INFINITY) return;
  s = s * __expf(m - mn) + s2 * __expf(m2 - mn);
  m = mn;
}

// one CTA (256 threads) per row; logits fp32, dlogits bf16
__global__ void __launch_bounds__(256) softmax_xent_kernel(const float* __restrict__ logits, int64_t ld,
                                                           const int* __restrict__ targets, int64_t v,
                                                           float* __restrict__ loss, __nv_bfloat16* __restrict__ dl,
                                                           int64_t ld_d, float grad_scale) {
  __shared__ float sm[8], ss[8];
  const int64_t row = blockIdx.x;
  const float* x = logits + row * ld;
  float m = -INFINITY, s = 0.f;
  for (int64_t j = threadIdx.x; j < v; j += 256) {
    const float xv = x[j];
    if (xv > m) s = s * __expf(m - xv) + 1.f, m = xv;
    else s += __expf(xv - m);
  }
#pragma unroll
  for (int off = 16; off; off >>= 1) {
    const float m2 = __shfl_xor_sync(0xffffffffu, m, off), s2 = __shfl_xor_sync(0xffffffffu, s, off);
    online_merge(m, s, m2, s2);
  }
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) sm[warp] = m, ss[warp] = s;
  __syncthreads();
  m = sm[0], s = ss[0];
  for (int w = 1; w < 8; ++w) online_merge(m, s, sm[w], ss[w]);
  const float lse = m + __logf(s);
  const int tgt = targets[row];
  if (threadIdx.x == 0) loss[row] = lse - x[tgt];
  __nv_bfloat16* d = dl + row * ld_d;
  for (int64_t j = threadIdx.x; j < v; j += 256)
    d[j] = __float2bfloat16_rn((__expf(x[j] - lse) - (j == tgt ? 1.f : 0.f)) * grad_scale);
}

}  // namespace
}  // namespace rsa

extern "C" {

int rsa_embed(const int* ids, int64_t n_rank, int64_t batch, int64_t chunk, const void* tok, const void* pos,
              int64_t hidden, void* x, void* stream) {
  using namespace rsa;
  const int64_t rows = n_rank * batch * chunk;
  if (!ids || !tok || !pos || !x || hidden % 8 || rows < 0)
    return fail(RSA_ERR_INVALID, "rsa_embed: bad arguments (hidden must be a multiple of 8)");
  if (!aligned16(tok) || !aligned16(pos) || !aligned16(x)) return fail(RSA_ERR_UNSUPPORTED, "rsa_embed: alignment");
  if (rows == 0) return RSA_OK;
  embed_kernel<<<(rows + 7) / 8, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      ids, rows, static_cast<const __nv_bfloat16*>(tok), static_cast<const __nv_bfloat16*>(pos), hidden,
      batch * chunk, chunk, static_cast<__nv_bfloat16*>(x));
  return check_launch("embed_kernel");
}

int rsa_embed_bwd(const int* ids, int64_t n_rank, int64_t batch, int64_t chunk, const void* dx, int64_t hidden,
                  float* dtok, float* dpos, void* stream) {
  using namespace rsa;
  const int64_t rows = n_rank * batch * chunk;
  if (!ids || !dx || !dtok || hidden % 2 || rows < 0) return fail(RSA_ERR_INVALID, "rsa_embed_bwd: bad arguments");
  if (rows == 0) return RSA_OK;
  embed_bwd_kernel<<<(rows + 7) / 8, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      ids, rows, static_cast<const __nv_bfloat16*>(dx), hidden, batch * chunk, chunk, dtok, dpos);
  return check_launch("embed_bwd_kernel");
}

int rsa_softmax_xent(const float* logits, int64_t ld, const int* targets, int64_t rows, int64_t vocab, float* loss,
                     void* dlogits, int64_t ld_d, float grad_scale, void* stream) {
  using namespace rsa;
  if (!logits || !targets || !loss || !dlogits || rows < 0 || vocab < 1 || ld < vocab || ld_d < vocab)
    return fail(RSA_ERR_INVALID, "rsa_softmax_xent: bad arguments");
  if (rows == 0) return RSA_OK;
  softmax_xent_kernel<<<rows, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      logits, ld, targets, vocab, loss, static_cast<__nv_bfloat16*>(dlogits), ld_d, grad_scale);
  return check_launch("softmax_xent_kernel");
}

}  // extern "C"

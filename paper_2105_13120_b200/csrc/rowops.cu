// Row-wise kernels of the staged RSA path: softmax, softmax Jacobian, row dot.
//
// One warp per row.  The softmax makes one online pass (running max and
// rescaled sum, ringseq/tensor_ops.py:82-84 restated as a single sweep) and
// one write pass; with 16-byte vector loads a row of L fp32 scores is read
// from HBM once and re-read from L1/L2.  The Jacobian
// (ringseq/ring_attention.py:187-190) is the same skeleton: one reduction
// pass for rowsum(dP * P), one write pass.
#include "common.h"
#include "ptx.cuh"

namespace rsa {
namespace {

template <typename T>
__device__ __forceinline__ float ld1(const T* p, int64_t i);
template <>
__device__ __forceinline__ float ld1<float>(const float* p, int64_t i) {
  return p[i];
}
template <>
__device__ __forceinline__ float ld1<__nv_bfloat16>(const __nv_bfloat16* p, int64_t i) {
  return __bfloat162float(p[i]);
}

// Load 4 consecutive elements as floats (caller guarantees alignment).
template <typename T>
__device__ __forceinline__ void ld4(const T* p, float* v);
template <>
__device__ __forceinline__ void ld4<float>(const float* p, float* v) {
  float4 x = *reinterpret_cast<const float4*>(p);
  v[0] = x.x, v[1] = x.y, v[2] = x.z, v[3] = x.w;
}
template <>
__device__ __forceinline__ void ld4<__nv_bfloat16>(const __nv_bfloat16* p, float* v) {
  uint2 x = *reinterpret_cast<const uint2*>(p);
  __nv_bfloat162 a = *reinterpret_cast<__nv_bfloat162*>(&x.x);
  __nv_bfloat162 b = *reinterpret_cast<__nv_bfloat162*>(&x.y);
  float2 fa = __bfloat1622float2(a), fb = __bfloat1622float2(b);
  v[0] = fa.x, v[1] = fa.y, v[2] = fb.x, v[3] = fb.y;
}

template <typename T>
__device__ __forceinline__ void st1(T* p, int64_t i, float v);
template <>
__device__ __forceinline__ void st1<float>(float* p, int64_t i, float v) {
  p[i] = v;
}
template <>
__device__ __forceinline__ void st1<__nv_bfloat16>(__nv_bfloat16* p, int64_t i, float v) {
  p[i] = __float2bfloat16_rn(v);
}

template <typename T>
__device__ __forceinline__ void st4(T* p, const float* v);
template <>
__device__ __forceinline__ void st4<float>(float* p, const float* v) {
  *reinterpret_cast<float4*>(p) = make_float4(v[0], v[1], v[2], v[3]);
}
template <>
__device__ __forceinline__ void st4<__nv_bfloat16>(__nv_bfloat16* p, const float* v) {
  *reinterpret_cast<uint2*>(p) = make_uint2(pack_bf16(v[0], v[1]), pack_bf16(v[2], v[3]));
}

constexpr float LOG2E = 1.4426950408889634f;

template <typename TI, typename TO, bool VEC>
__global__ void __launch_bounds__(256) softmax_rows_kernel(const TI* __restrict__ x, int64_t rows, int64_t cols,
                                                           int64_t ldx, float scale, TO* __restrict__ y, int64_t ldy,
                                                           int* flag) {
  const int64_t row = int64_t(blockIdx.x) * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;
  const TI* xr = x + row * ldx;
  TO* yr = y + row * ldy;
  const float sl = scale * LOG2E;  // work in base 2: exp(s*x - m) = 2^(sl*x - m2)
  float m = -INFINITY, s = 0.f;
  bool bad = false;
  if (VEC) {
    for (int64_t c = int64_t(lane) * 4; c < cols; c += 128) {
      float v[4];
      ld4<TI>(xr + c, v);
      float lm = -INFINITY;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        bad |= !isfinite(v[i]);
        lm = fmaxf(lm, __fmul_rn(v[i], sl));
      }
      if (lm > m) {
        s *= exp2f(m - lm);
        m = lm;
      }
#pragma unroll
      for (int i = 0; i < 4; ++i) s += exp2f(__fmul_rn(v[i], sl) - m);
    }
  } else {
    for (int64_t c = lane; c < cols; c += 32) {
      const float v = ld1<TI>(xr, c);
      bad |= !isfinite(v);
      const float t = __fmul_rn(v, sl);
      if (t > m) {
        s *= exp2f(m - t);
        m = t;
      }
      s += exp2f(t - m);
    }
  }
  // warp-combine (m, s) in base 2
#pragma unroll
  for (int off = 16; off; off >>= 1) {
    const float m2 = __shfl_xor_sync(0xffffffffu, m, off);
    const float s2 = __shfl_xor_sync(0xffffffffu, s, off);
    const float mn = fmaxf(m, m2);
    if (mn != -INFINITY) {
      s = s * exp2f(m - mn) + s2 * exp2f(m2 - mn);
      m = mn;
    }
  }
  if (__any_sync(0xffffffffu, bad)) {
    if (lane == 0) atomicExch(flag, 1);
  }
  const float inv = 1.f / s;
  if (VEC) {
    for (int64_t c = int64_t(lane) * 4; c < cols; c += 128) {
      float v[4];
      ld4<TI>(xr + c, v);
#pragma unroll
      for (int i = 0; i < 4; ++i) v[i] = exp2f(__fmul_rn(v[i], sl) - m) * inv;
      st4<TO>(yr + c, v);
    }
  } else {
    for (int64_t c = lane; c < cols; c += 32) st1<TO>(yr, c, exp2f(__fmul_rn(ld1<TI>(xr, c), sl) - m) * inv);
  }
}

template <typename TP, typename TD, bool VEC>
__global__ void __launch_bounds__(256) softmax_bwd_kernel(const TP* __restrict__ p, int64_t ldp,
                                                          const float* __restrict__ dp, int64_t lddp, int64_t rows,
                                                          int64_t cols, float scale, TD* __restrict__ ds, int64_t ldds) {
  const int64_t row = int64_t(blockIdx.x) * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;
  const TP* pr = p + row * ldp;
  const float* dr = dp + row * lddp;
  TD* sr = ds + row * ldds;
  float acc = 0.f;
  if (VEC) {
    for (int64_t c = int64_t(lane) * 4; c < cols; c += 128) {
      float a[4], b[4];
      ld4<TP>(pr + c, a);
      ld4<float>(dr + c, b);
#pragma unroll
      for (int i = 0; i < 4; ++i) acc += a[i] * b[i];
    }
  } else {
    for (int64_t c = lane; c < cols; c += 32) acc += ld1<TP>(pr, c) * dr[c];
  }
#pragma unroll
  for (int off = 16; off; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  if (VEC) {
    for (int64_t c = int64_t(lane) * 4; c < cols; c += 128) {
      float a[4], b[4], o[4];
      ld4<TP>(pr + c, a);
      ld4<float>(dr + c, b);
#pragma unroll
      for (int i = 0; i < 4; ++i) o[i] = a[i] * (b[i] - acc) * scale;
      st4<TD>(sr + c, o);
    }
  } else {
    for (int64_t c = lane; c < cols; c += 32) st1<TD>(sr, c, ld1<TP>(pr, c) * (dr[c] - acc) * scale);
  }
}

__global__ void __launch_bounds__(256) rowdot_kernel(const __nv_bfloat16* __restrict__ a, int64_t lda,
                                                     const __nv_bfloat16* __restrict__ b, int64_t ldb, int64_t rows,
                                                     int64_t cols, float* __restrict__ out) {
  const int64_t row = int64_t(blockIdx.x) * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;
  float acc = 0.f;
  for (int64_t c = lane; c < cols; c += 32) acc += __bfloat162float(a[row * lda + c]) * __bfloat162float(b[row * ldb + c]);
#pragma unroll
  for (int off = 16; off; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  if (lane == 0) out[row] = acc;
}

// cols == 64, 16-byte aligned rows: 8 lanes per row, one 16-byte load of a
// and of b per lane, 3 shuffles; 4 rows per warp, 32 per 256-thread block.
__global__ void __launch_bounds__(256) rowdot64_kernel(const __nv_bfloat16* __restrict__ a, int64_t lda,
                                                       const __nv_bfloat16* __restrict__ b, int64_t ldb, int64_t rows,
                                                       float* __restrict__ out) {
  const int64_t row = int64_t(blockIdx.x) * 32 + (threadIdx.x >> 3);
  const int sub = threadIdx.x & 7;
  float acc = 0.f;
  if (row < rows) {
    const uint4 x = __ldg(reinterpret_cast<const uint4*>(a + row * lda) + sub);
    const uint4 y = __ldg(reinterpret_cast<const uint4*>(b + row * ldb) + sub);
    const uint32_t* xs = reinterpret_cast<const uint32_t*>(&x);
    const uint32_t* ys = reinterpret_cast<const uint32_t*>(&y);
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float2 fx = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&xs[i]));
      const float2 fy = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&ys[i]));
      acc = fmaf(fx.x, fy.x, acc);
      acc = fmaf(fx.y, fy.y, acc);
    }
  }
  acc += __shfl_xor_sync(0xffffffffu, acc, 1);
  acc += __shfl_xor_sync(0xffffffffu, acc, 2);
  acc += __shfl_xor_sync(0xffffffffu, acc, 4);
  if (row < rows && sub == 0) out[row] = acc;
}


// rowdot with a per-row scale, and the scaled copy of `a` (bf16): cols == 64,
// 16-byte aligned rows, 8 lanes per row (one 16-byte load of a and of b, one
// 16-byte store of a * scale per lane).
__global__ void __launch_bounds__(256) rowdot64_scale_kernel(const __nv_bfloat16* __restrict__ a, int64_t lda,
                                                             const __nv_bfloat16* __restrict__ b, int64_t ldb,
                                                             const float* __restrict__ scale, int64_t rows,
                                                             float* __restrict__ out, __nv_bfloat16* __restrict__ as,
                                                             int64_t ldas) {
  const int64_t row = int64_t(blockIdx.x) * 32 + (threadIdx.x >> 3);
  const int sub = threadIdx.x & 7;
  float acc = 0.f, sc = 0.f;
  if (row < rows) {
    sc = __ldg(scale + row);
    const uint4 x = __ldg(reinterpret_cast<const uint4*>(a + row * lda) + sub);
    const uint4 y = __ldg(reinterpret_cast<const uint4*>(b + row * ldb) + sub);
    const uint32_t* xs = reinterpret_cast<const uint32_t*>(&x);
    const uint32_t* ys = reinterpret_cast<const uint32_t*>(&y);
    uint32_t w[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float2 fx = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&xs[i]));
      const float2 fy = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&ys[i]));
      acc = fmaf(fx.x, fy.x, acc);
      acc = fmaf(fx.y, fy.y, acc);
      w[i] = pack_bf16(fx.x * sc, fx.y * sc);
    }
    *(reinterpret_cast<uint4*>(as + row * ldas) + sub) = make_uint4(w[0], w[1], w[2], w[3]);
  }
  acc += __shfl_xor_sync(0xffffffffu, acc, 1);
  acc += __shfl_xor_sync(0xffffffffu, acc, 2);
  acc += __shfl_xor_sync(0xffffffffu, acc, 4);
  if (row < rows && sub == 0) out[row] = acc * sc;
}

// Generic shape: one warp per row.
__global__ void __launch_bounds__(256) rowdot_scale_kernel(const __nv_bfloat16* __restrict__ a, int64_t lda,
                                                           const __nv_bfloat16* __restrict__ b, int64_t ldb,
                                                           const float* __restrict__ scale, int64_t rows, int64_t cols,
                                                           float* __restrict__ out, __nv_bfloat16* __restrict__ as,
                                                           int64_t ldas) {
  const int64_t row = int64_t(blockIdx.x) * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;
  const float sc = scale[row];
  float acc = 0.f;
  for (int64_t c = lane; c < cols; c += 32) {
    const float x = __bfloat162float(a[row * lda + c]);
    acc += x * __bfloat162float(b[row * ldb + c]);
    as[row * ldas + c] = __float2bfloat16_rn(x * sc);
  }
#pragma unroll
  for (int off = 16; off; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  if (lane == 0) out[row] = acc * sc;
}

// y[r, c] = scale[r] * p[r, c]; one warp per row.
template <typename TO>
__global__ void __launch_bounds__(256) panel_normalize_kernel(const __nv_bfloat16* __restrict__ p, int64_t ldp,
                                                              const float* __restrict__ scale, int64_t rows,
                                                              int64_t cols, TO* __restrict__ y, int64_t ldy) {
  const int64_t row = int64_t(blockIdx.x) * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= rows) return;
  const float sc = scale[row];
  for (int64_t c = lane; c < cols; c += 32) y[row * ldy + c] = TO(__bfloat162float(p[row * ldp + c]) * sc);
}


// y[i] = sum_d x[d * rank_stride + i] over d = 0..n_rank-1 in ascending order (fp32, then
// fp32 or bf16 out): the per-rank partial projections summed across ranks -- the Linformer's
// ring-accumulate (ringseq/sparse_attention.py:59-71) when every rank is resident.
template <typename TI>
__device__ __forceinline__ float4 ld4(const TI* p);
template <>
__device__ __forceinline__ float4 ld4<float>(const float* p) {
  return *reinterpret_cast<const float4*>(p);
}
template <>
__device__ __forceinline__ float4 ld4<__nv_bfloat16>(const __nv_bfloat16* p) {
  const uint2 w = *reinterpret_cast<const uint2*>(p);
  const float2 a = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w.x));
  const float2 b = __bfloat1622float2(*reinterpret_cast<const __nv_bfloat162*>(&w.y));
  return make_float4(a.x, a.y, b.x, b.y);
}

template <typename TI, typename TO>
__global__ void __launch_bounds__(256) sum_ranks_kernel(const TI* __restrict__ x, int64_t n_rank, int64_t count,
                                                        int64_t rank_stride, TO* __restrict__ y) {
  for (int64_t i = (int64_t(blockIdx.x) * 256 + threadIdx.x) * 4; i < count; i += int64_t(gridDim.x) * 256 * 4) {
    float4 acc = ld4<TI>(x + i);
    for (int64_t d = 1; d < n_rank; ++d) {
      const float4 t = ld4<TI>(x + d * rank_stride + i);
      acc.x += t.x, acc.y += t.y, acc.z += t.z, acc.w += t.w;
    }
    st4(y + i, reinterpret_cast<const float*>(&acc));
  }
}

template <typename TI, typename TO>
__global__ void __launch_bounds__(256) sum_ranks_scalar_kernel(const TI* __restrict__ x, int64_t n_rank,
                                                               int64_t count, int64_t rank_stride, TO* __restrict__ y) {
  for (int64_t i = int64_t(blockIdx.x) * 256 + threadIdx.x; i < count; i += int64_t(gridDim.x) * 256) {
    float acc = ld1<TI>(x, i);
    for (int64_t d = 1; d < n_rank; ++d) acc += ld1<TI>(x, d * rank_stride + i);
    st1(y, i, acc);
  }
}

// Exact GELU (ringseq/tensor_ops.py:87-90): y = x * Phi(x), Phi(x) = (1 + erf(x / sqrt 2)) / 2,
// and its backward dx = dy * (Phi(x) + x * phi(x)).  Grid-stride, 4 elements per thread
// per iteration when the pointers allow it.
constexpr float INV_SQRT2 = 0.7071067811865476f;
constexpr float INV_SQRT_2PI = 0.3989422804014327f;

__device__ __forceinline__ float gelu_f(float x) { return 0.5f * x * (1.f + erff(x * INV_SQRT2)); }
__device__ __forceinline__ float gelu_grad_f(float x) {
  return 0.5f * (1.f + erff(x * INV_SQRT2)) + x * INV_SQRT_2PI * __expf(-0.5f * x * x);
}

template <typename TI, typename TO, bool VEC>
__global__ void __launch_bounds__(256) gelu_kernel(const TI* __restrict__ x, int64_t n, TO* __restrict__ y) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  if (VEC) {
    for (int64_t i = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) * 4; i < n; i += stride * 4) {
      float v[4];
      ld4<TI>(x + i, v);
#pragma unroll
      for (int e = 0; e < 4; ++e) v[e] = gelu_f(v[e]);
      st4<TO>(y + i, v);
    }
  } else {
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride) st1<TO>(y, i, gelu_f(ld1<TI>(x, i)));
  }
}

template <typename TI, typename TG, typename TO, bool VEC>
__global__ void __launch_bounds__(256) gelu_bwd_kernel(const TI* __restrict__ x, const TG* __restrict__ dy, int64_t n,
                                                       TO* __restrict__ dx) {
  const int64_t stride = int64_t(gridDim.x) * blockDim.x;
  if (VEC) {
    for (int64_t i = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) * 4; i < n; i += stride * 4) {
      float v[4], g[4];
      ld4<TI>(x + i, v);
      ld4<TG>(dy + i, g);
#pragma unroll
      for (int e = 0; e < 4; ++e) v[e] = g[e] * gelu_grad_f(v[e]);
      st4<TO>(dx + i, v);
    }
  } else {
    for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n; i += stride)
      st1<TO>(dx, i, ld1<TG>(dy, i) * gelu_grad_f(ld1<TI>(x, i)));
  }
}

template <typename T>
bool aligned_vec(const void* p) {
  return (reinterpret_cast<uintptr_t>(p) % (4 * sizeof(T))) == 0;
}

int elementwise_grid(int64_t n) {
  const int64_t blocks = (n / 4 + 255) / 256;
  const int64_t cap = int64_t(num_sms()) * 8;
  return int(blocks < 1 ? 1 : (blocks > cap ? cap : blocks));
}

template <typename TI, typename TO>
int gelu_launch(const void* x, int64_t n, void* y, cudaStream_t st) {
  const auto* xi = static_cast<const TI*>(x);
  auto* yo = static_cast<TO*>(y);
  if (n % 4 == 0 && aligned_vec<TI>(x) && aligned_vec<TO>(y))
    gelu_kernel<TI, TO, true><<<elementwise_grid(n), 256, 0, st>>>(xi, n, yo);
  else
    gelu_kernel<TI, TO, false><<<elementwise_grid(n), 256, 0, st>>>(xi, n, yo);
  return check_launch("gelu_kernel");
}

template <typename TI, typename TG, typename TO>
int gelu_bwd_launch(const void* x, const void* dy, int64_t n, void* dx, cudaStream_t st) {
  const auto* xi = static_cast<const TI*>(x);
  const auto* gi = static_cast<const TG*>(dy);
  auto* o = static_cast<TO*>(dx);
  if (n % 4 == 0 && aligned_vec<TI>(x) && aligned_vec<TG>(dy) && aligned_vec<TO>(dx))
    gelu_bwd_kernel<TI, TG, TO, true><<<elementwise_grid(n), 256, 0, st>>>(xi, gi, n, o);
  else
    gelu_bwd_kernel<TI, TG, TO, false><<<elementwise_grid(n), 256, 0, st>>>(xi, gi, n, o);
  return check_launch("gelu_bwd_kernel");
}

template <typename T>
bool vec_ok(const void* ptr, int64_t ld, int64_t cols) {
  const int64_t esz = sizeof(T);
  const int64_t need = 4 * esz;  // 4 elements per vector access
  return (reinterpret_cast<uintptr_t>(ptr) % need) == 0 && (ld * esz) % need == 0 && cols % 4 == 0;
}

template <typename TI, typename TO>
int softmax_launch(const void* x, int64_t rows, int64_t cols, int64_t ldx, float scale, void* y, int64_t ldy, int* flag,
                   cudaStream_t st) {
  const dim3 grid((rows + 7) / 8);
  const bool v = vec_ok<TI>(x, ldx, cols) && vec_ok<TO>(y, ldy, cols);
  if (v)
    softmax_rows_kernel<TI, TO, true><<<grid, 256, 0, st>>>(static_cast<const TI*>(x), rows, cols, ldx, scale,
                                                            static_cast<TO*>(y), ldy, flag);
  else
    softmax_rows_kernel<TI, TO, false><<<grid, 256, 0, st>>>(static_cast<const TI*>(x), rows, cols, ldx, scale,
                                                             static_cast<TO*>(y), ldy, flag);
  return check_launch("softmax_rows_kernel");
}

template <typename TP, typename TD>
int softmax_bwd_launch(const void* p, int64_t ldp, const float* dp, int64_t lddp, int64_t rows, int64_t cols,
                       float scale, void* ds, int64_t ldds, cudaStream_t st) {
  const dim3 grid((rows + 7) / 8);
  const bool v = vec_ok<TP>(p, ldp, cols) && vec_ok<float>(dp, lddp, cols) && vec_ok<TD>(ds, ldds, cols);
  if (v)
    softmax_bwd_kernel<TP, TD, true><<<grid, 256, 0, st>>>(static_cast<const TP*>(p), ldp, dp, lddp, rows, cols, scale,
                                                           static_cast<TD*>(ds), ldds);
  else
    softmax_bwd_kernel<TP, TD, false><<<grid, 256, 0, st>>>(static_cast<const TP*>(p), ldp, dp, lddp, rows, cols,
                                                            scale, static_cast<TD*>(ds), ldds);
  return check_launch("softmax_bwd_kernel");
}

template <typename TI, typename TO>
int sum_ranks_launch(const void* x, int64_t n_rank, int64_t count, int64_t rank_stride, void* y, int vec,
                     cudaStream_t st) {
  const int grid = elementwise_grid(count);
  const auto* xi = static_cast<const TI*>(x);
  auto* yo = static_cast<TO*>(y);
  if (vec) sum_ranks_kernel<TI, TO><<<grid, 256, 0, st>>>(xi, n_rank, count, rank_stride, yo);
  else sum_ranks_scalar_kernel<TI, TO><<<grid * 4, 256, 0, st>>>(xi, n_rank, count, rank_stride, yo);
  return check_launch("sum_ranks_kernel");
}

}  // namespace
}  // namespace rsa

extern "C" {

int rsa_softmax_rows(const void* x, int x_dtype, int64_t rows, int64_t cols, int64_t ld_x, float scale, void* y,
                     int y_dtype, int64_t ld_y, int* nonfinite_flag, void* stream) {
  using namespace rsa;
  if (rows < 0 || cols < 1 || ld_x < cols || ld_y < cols || !nonfinite_flag)
    return fail(RSA_ERR_INVALID, "softmax_rows: bad sizes");
  if (rows == 0) return RSA_OK;
  if ((rows + 7) / 8 > 0x7fffffff) return fail(RSA_ERR_INVALID, "softmax_rows: too many rows");
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const bool xb = x_dtype == RSA_BF16, yb = y_dtype == RSA_BF16;
  if (!xb && !yb) return softmax_launch<float, float>(x, rows, cols, ld_x, scale, y, ld_y, nonfinite_flag, st);
  if (!xb && yb) return softmax_launch<float, __nv_bfloat16>(x, rows, cols, ld_x, scale, y, ld_y, nonfinite_flag, st);
  if (xb && !yb) return softmax_launch<__nv_bfloat16, float>(x, rows, cols, ld_x, scale, y, ld_y, nonfinite_flag, st);
  return softmax_launch<__nv_bfloat16, __nv_bfloat16>(x, rows, cols, ld_x, scale, y, ld_y, nonfinite_flag, st);
}

int rsa_softmax_bwd(const void* p, int p_dtype, int64_t ld_p, const float* dp, int64_t ld_dp, int64_t rows,
                    int64_t cols, float scale, void* ds, int ds_dtype, int64_t ld_ds, void* stream) {
  using namespace rsa;
  if (rows < 0 || cols < 1) return fail(RSA_ERR_INVALID, "softmax_bwd: bad sizes");
  if (rows == 0) return RSA_OK;
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  const bool pb = p_dtype == RSA_BF16, db = ds_dtype == RSA_BF16;
  if (!pb && !db) return softmax_bwd_launch<float, float>(p, ld_p, dp, ld_dp, rows, cols, scale, ds, ld_ds, st);
  if (!pb && db) return softmax_bwd_launch<float, __nv_bfloat16>(p, ld_p, dp, ld_dp, rows, cols, scale, ds, ld_ds, st);
  if (pb && !db) return softmax_bwd_launch<__nv_bfloat16, float>(p, ld_p, dp, ld_dp, rows, cols, scale, ds, ld_ds, st);
  return softmax_bwd_launch<__nv_bfloat16, __nv_bfloat16>(p, ld_p, dp, ld_dp, rows, cols, scale, ds, ld_ds, st);
}

int rsa_rowdot(const void* a, int64_t lda, const void* b, int64_t ldb, int64_t rows, int64_t cols, float* out,
               void* stream) {
  using namespace rsa;
  if (rows < 0 || cols < 0) return fail(RSA_ERR_INVALID, "rowdot: bad sizes");
  if (rows == 0) return RSA_OK;
  if (cols == 64 && aligned16(a) && aligned16(b) && lda % 8 == 0 && ldb % 8 == 0) {
    rowdot64_kernel<<<(rows + 31) / 32, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
        static_cast<const __nv_bfloat16*>(a), lda, static_cast<const __nv_bfloat16*>(b), ldb, rows, out);
    return check_launch("rowdot64_kernel");
  }
  rowdot_kernel<<<(rows + 7) / 8, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(
      static_cast<const __nv_bfloat16*>(a), lda, static_cast<const __nv_bfloat16*>(b), ldb, rows, cols, out);
  return check_launch("rowdot_kernel");
}

int rsa_rowdot_scale(const void* a, int64_t lda, const void* b, int64_t ldb, const float* scale, int64_t rows,
                     int64_t cols, float* out, void* a_scaled, int64_t ld_as, void* stream) {
  using namespace rsa;
  if (rows < 0 || cols < 0 || !scale || !out || !a_scaled) return fail(RSA_ERR_INVALID, "rowdot_scale: bad arguments");
  if (rows == 0) return RSA_OK;
  auto st = reinterpret_cast<cudaStream_t>(stream);
  const auto* pa = static_cast<const __nv_bfloat16*>(a);
  const auto* pb = static_cast<const __nv_bfloat16*>(b);
  auto* ps = static_cast<__nv_bfloat16*>(a_scaled);
  if (cols == 64 && aligned16(a) && aligned16(b) && aligned16(a_scaled) && lda % 8 == 0 && ldb % 8 == 0 &&
      ld_as % 8 == 0) {
    rowdot64_scale_kernel<<<(rows + 31) / 32, 256, 0, st>>>(pa, lda, pb, ldb, scale, rows, out, ps, ld_as);
    return check_launch("rowdot64_scale_kernel");
  }
  rowdot_scale_kernel<<<(rows + 7) / 8, 256, 0, st>>>(pa, lda, pb, ldb, scale, rows, cols, out, ps, ld_as);
  return check_launch("rowdot_scale_kernel");
}

int rsa_panel_normalize(const void* p, int64_t ld_p, const float* scale, int64_t rows, int64_t cols, void* y,
                        int y_dtype, int64_t ld_y, void* stream) {
  using namespace rsa;
  if (rows < 0 || cols < 0 || !scale) return fail(RSA_ERR_INVALID, "panel_normalize: bad arguments");
  if (rows == 0) return RSA_OK;
  auto st = reinterpret_cast<cudaStream_t>(stream);
  const auto* pp = static_cast<const __nv_bfloat16*>(p);
  const dim3 grid((rows + 7) / 8);
  if (y_dtype == RSA_F32)
    panel_normalize_kernel<float><<<grid, 256, 0, st>>>(pp, ld_p, scale, rows, cols, static_cast<float*>(y), ld_y);
  else if (y_dtype == RSA_BF16)
    panel_normalize_kernel<__nv_bfloat16>
        <<<grid, 256, 0, st>>>(pp, ld_p, scale, rows, cols, static_cast<__nv_bfloat16*>(y), ld_y);
  else
    return fail(RSA_ERR_INVALID, "panel_normalize: bad output dtype");
  return check_launch("panel_normalize_kernel");
}

int rsa_sum_ranks(const void* x, int x_dtype, int64_t n_rank, int64_t count, int64_t rank_stride, void* y,
                  int y_dtype, void* stream) {
  using namespace rsa;
  if (!x || !y || n_rank < 1 || count < 0 || rank_stride < count || (x_dtype != RSA_F32 && x_dtype != RSA_BF16) ||
      (y_dtype != RSA_F32 && y_dtype != RSA_BF16))
    return fail(RSA_ERR_INVALID, "sum_ranks: bad arguments");
  if (count == 0) return RSA_OK;
  auto st = reinterpret_cast<cudaStream_t>(stream);
  const int vec = count % 4 == 0 && rank_stride % 4 == 0 && aligned16(x) && aligned16(y);
  if (x_dtype == RSA_F32)
    return y_dtype == RSA_F32 ? sum_ranks_launch<float, float>(x, n_rank, count, rank_stride, y, vec, st)
                              : sum_ranks_launch<float, __nv_bfloat16>(x, n_rank, count, rank_stride, y, vec, st);
  return y_dtype == RSA_F32 ? sum_ranks_launch<__nv_bfloat16, float>(x, n_rank, count, rank_stride, y, vec, st)
                            : sum_ranks_launch<__nv_bfloat16, __nv_bfloat16>(x, n_rank, count, rank_stride, y, vec, st);
}

int rsa_gelu(const void* x, int x_dtype, int64_t n, void* y, int y_dtype, void* stream) {
  using namespace rsa;
  if (n < 0 || !x || !y) return fail(RSA_ERR_INVALID, "gelu: bad arguments");
  if (n == 0) return RSA_OK;
  auto st = reinterpret_cast<cudaStream_t>(stream);
  if (x_dtype == RSA_F32 && y_dtype == RSA_F32) return gelu_launch<float, float>(x, n, y, st);
  if (x_dtype == RSA_F32 && y_dtype == RSA_BF16) return gelu_launch<float, __nv_bfloat16>(x, n, y, st);
  if (x_dtype == RSA_BF16 && y_dtype == RSA_F32) return gelu_launch<__nv_bfloat16, float>(x, n, y, st);
  if (x_dtype == RSA_BF16 && y_dtype == RSA_BF16) return gelu_launch<__nv_bfloat16, __nv_bfloat16>(x, n, y, st);
  return fail(RSA_ERR_INVALID, "gelu: bad dtype");
}

int rsa_gelu_bwd(const void* x, int x_dtype, const void* dy, int dy_dtype, int64_t n, void* dx, int dx_dtype,
                 void* stream) {
  using namespace rsa;
  if (n < 0 || !x || !dy || !dx) return fail(RSA_ERR_INVALID, "gelu_bwd: bad arguments");
  if (n == 0) return RSA_OK;
  auto st = reinterpret_cast<cudaStream_t>(stream);
  if (x_dtype == RSA_F32 && dy_dtype == RSA_F32 && dx_dtype == RSA_F32)
    return gelu_bwd_launch<float, float, float>(x, dy, n, dx, st);
  if (x_dtype == RSA_F32 && dy_dtype == RSA_F32 && dx_dtype == RSA_BF16)
    return gelu_bwd_launch<float, float, __nv_bfloat16>(x, dy, n, dx, st);
  if (x_dtype == RSA_BF16 && dy_dtype == RSA_BF16 && dx_dtype == RSA_BF16)
    return gelu_bwd_launch<__nv_bfloat16, __nv_bfloat16, __nv_bfloat16>(x, dy, n, dx, st);
  if (x_dtype == RSA_BF16 && dy_dtype == RSA_F32 && dx_dtype == RSA_BF16)
    return gelu_bwd_launch<__nv_bfloat16, float, __nv_bfloat16>(x, dy, n, dx, st);
  if (x_dtype == RSA_F32 && dy_dtype == RSA_BF16 && dx_dtype == RSA_BF16)
    return gelu_bwd_launch<float, __nv_bfloat16, __nv_bfloat16>(x, dy, n, dx, st);
  return fail(RSA_ERR_INVALID, "gelu_bwd: unsupported dtype combination");
}

}  // extern "C"

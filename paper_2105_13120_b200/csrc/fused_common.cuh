// Shared pieces of the fused RSA kernels (fused.cu, bwd_fused.cu): tile
// constants, pipeline positions, swizzled smem row moves, strided outputs,
// and the host-side TMA map builders.  Everything is internal linkage.
#pragma once

#include "common.h"
#include "ptx.cuh"

namespace rsa {
namespace {

constexpr int HD = 64;                      // head size the fused kernels tile
constexpr int TR = 128;                     // rows per tile (UMMA M)
constexpr int TK = 128;                     // keys per tile
constexpr uint32_t TILE = TR * HD * 2;      // 16 KB: 128 x 64 bf16
constexpr uint32_t PTILE = TR * TK * 2;     // 32 KB: 128 x 128 bf16 (two 64-key atoms)
constexpr uint32_t ATOM = TR * 128;         // 16 KB: one 128-row x 128-byte swizzle column
constexpr float LOG2E = 1.4426950408889634f;
constexpr int EPI_WARPS = 8;
constexpr int NTHREADS = 64 + 32 * EPI_WARPS;  // 320
constexpr int EPI_THREADS = 32 * EPI_WARPS;    // 256

enum { MODE_PASS_A = 1, MODE_PASS_B = 2, MODE_EXT_STATS = 4, MODE_WRITE_STATS = 8 };

__device__ __forceinline__ void bar_epi() { asm volatile("bar.sync 1, 256;" ::: "memory"); }
__device__ __forceinline__ void bar_half(int h) { asm volatile("bar.sync %0, 128;" ::"r"(2 + h) : "memory"); }

// Pipeline position: slot and phase of the i-th use of an n-deep ring.
struct Pos {
  uint32_t i = 0;
  __device__ __forceinline__ uint32_t slot(uint32_t n) const { return i % n; }
  __device__ __forceinline__ uint32_t phase(uint32_t n) const { return (i / n) & 1u; }
};

// 32 fp32 values of row r, columns col0..col0+31, as bf16 into a
// [64-col atom][128 rows][128 B] SWIZZLE_128B tile.
__device__ __forceinline__ void st_row32_sw128(uint32_t tile, uint32_t r, int col0, const float* v) {
  const uint32_t atom = col0 >> 6, chunk0 = (col0 & 63) >> 3;
#pragma unroll
  for (int q = 0; q < 4; ++q)
    st_shared_v4(tile + atom * ATOM + sw128_offset(r, chunk0 + q), pack_bf16(v[8 * q], v[8 * q + 1]),
                 pack_bf16(v[8 * q + 2], v[8 * q + 3]), pack_bf16(v[8 * q + 4], v[8 * q + 5]),
                 pack_bf16(v[8 * q + 6], v[8 * q + 7]));
}

__device__ __forceinline__ void ld_row32_sw128(uint32_t tile, uint32_t r, int col0, float* v) {
  const uint32_t atom = col0 >> 6, chunk0 = (col0 & 63) >> 3;
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    uint32_t w[4];
    ld_shared_v4(tile + atom * ATOM + sw128_offset(r, chunk0 + q), w[0], w[1], w[2], w[3]);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const float2 f = __bfloat1622float2(*reinterpret_cast<__nv_bfloat162*>(&w[e]));
      v[8 * q + 2 * e] = f.x;
      v[8 * q + 2 * e + 1] = f.y;
    }
  }
}

// dS of two adjacent keys: P * (dP - D) with packed fp32x2 arithmetic (FADD2 / FMUL2;
// the same roundings as the scalar form), packed to bf16x2.  pw: the bf16 pair of P;
// nd: (-D, -D).
__device__ __forceinline__ uint32_t ds_pair(uint32_t pw, float dp0, float dp1, uint64_t nd) {
  uint64_t x, pp;
  asm("mov.b64 %0, {%1, %2};" : "=l"(x) : "f"(dp0), "f"(dp1));
  asm("add.rn.f32x2 %0, %0, %1;" : "+l"(x) : "l"(nd));
  asm("mov.b64 %0, {%1, %2};" : "=l"(pp) : "f"(__uint_as_float(pw << 16)), "f"(__uint_as_float(pw & 0xFFFF0000u)));
  asm("mul.rn.f32x2 %0, %0, %1;" : "+l"(x) : "l"(pp));
  float a, b;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(x));
  return pack_bf16(a, b);
}

// ds_pair with a different D for each of the two elements (the transposed backward walks a
// key across queries, each query with its own D): the same roundings element for element.
__device__ __forceinline__ uint32_t ds_pair2(uint32_t pw, float dp0, float dp1, float d0, float d1) {
  uint64_t x, pp, nd;
  asm("mov.b64 %0, {%1, %2};" : "=l"(x) : "f"(dp0), "f"(dp1));
  asm("mov.b64 %0, {%1, %2};" : "=l"(nd) : "f"(-d0), "f"(-d1));
  asm("add.rn.f32x2 %0, %0, %1;" : "+l"(x) : "l"(nd));
  asm("mov.b64 %0, {%1, %2};" : "=l"(pp) : "f"(__uint_as_float(pw << 16)), "f"(__uint_as_float(pw & 0xFFFF0000u)));
  asm("mul.rn.f32x2 %0, %0, %1;" : "+l"(x) : "l"(pp));
  float a, b;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(x));
  return pack_bf16(a, b);
}

__device__ __forceinline__ void ld_shared_f4(uint32_t addr, float* v) {
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v[0]), "=f"(v[1]), "=f"(v[2]), "=f"(v[3]) : "r"(addr));
}

// dS = P * (dP - D) for 32 keys of row r in place over the bf16 P tile (columns
// col0..col0+31 of a SWIZZLE_128B [64-col atom][128 rows] tile); dp: the fp32 dP row
// chunk, nd: (-D, -D).
__device__ __forceinline__ void ds_row32_inplace(uint32_t tile, uint32_t r, int col0, const float* dp, uint64_t nd) {
  const uint32_t atom = col0 >> 6, chunk0 = (col0 & 63) >> 3;
  uint32_t w[16];  // every load before the first store (the compiler cannot reorder them)
#pragma unroll
  for (int q = 0; q < 4; ++q)
    ld_shared_v4(tile + atom * ATOM + sw128_offset(r, chunk0 + q), w[4 * q], w[4 * q + 1], w[4 * q + 2], w[4 * q + 3]);
#pragma unroll
  for (int e = 0; e < 16; ++e) w[e] = ds_pair(w[e], dp[2 * e], dp[2 * e + 1], nd);
#pragma unroll
  for (int q = 0; q < 4; ++q)
    st_shared_v4(tile + atom * ATOM + sw128_offset(r, chunk0 + q), w[4 * q], w[4 * q + 1], w[4 * q + 2], w[4 * q + 3]);
}

__device__ __forceinline__ uint64_t neg_pair(float d) {
  uint64_t nd;
  asm("mov.b64 %0, {%1, %1};" : "=l"(nd) : "f"(-d));
  return nd;
}

// max |v| over the first `nvalid` of 32 values (NaN-propagating): one 3-input
// FMNMX per two scores.  Finite iff every score is finite.
__device__ __forceinline__ void absmax32(const float* v, int nvalid, float& mx_out) {
  if (nvalid >= 32) {
    float mx[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) mx[e] = fabsf(v[e]);
#pragma unroll
    for (int e = 4; e < 32; ++e) mx[e & 3] = max_nan(mx[e & 3], fabsf(v[e]));
    mx_out = max_nan(mx_out, max_nan(max_nan(mx[0], mx[1]), max_nan(mx[2], mx[3])));
  } else {
#pragma unroll
    for (int e = 0; e < 32; ++e)
      if (e < nvalid) mx_out = max_nan(mx_out, fabsf(v[e]));
  }
}

// Max and min of the first `nvalid` of 32 values (NaN-propagating).
__device__ __forceinline__ void minmax32(const float* v, int nvalid, float& mx_out, float& mi_out) {
  if (nvalid >= 32) {
    float mx[4], mi[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) mx[e] = mi[e] = v[e];
#pragma unroll
    for (int e = 4; e < 32; ++e) mx[e & 3] = max_nan(mx[e & 3], v[e]), mi[e & 3] = min_nan(mi[e & 3], v[e]);
    mx_out = max_nan(mx_out, max_nan(max_nan(mx[0], mx[1]), max_nan(mx[2], mx[3])));
    mi_out = min_nan(mi_out, min_nan(min_nan(mi[0], mi[1]), min_nan(mi[2], mi[3])));
  } else {
#pragma unroll
    for (int e = 0; e < 32; ++e)
      if (e < nvalid) mx_out = max_nan(mx_out, v[e]), mi_out = min_nan(mi_out, v[e]);
  }
}

// The factored panel's values: 32 scores of one row (32 consecutive keys starting at a
// multiple of 32) -> 16 packed bf16 pairs of P~ = 2^(v*sl - msl), zero past nvalid, every
// exp2 on MUFU.  The forward that writes the panel (rsa_fwd_factored) and the stream-mode
// backward that recomputes it (bwd_stream.cu, which walks a KEY's scores across queries)
// apply this same per-element rounding to bitwise-identical tensor-core scores, so the
// recomputed P~ equals the stored panel bit for bit.  (An FMA-pipe polynomial for one exp2
// in four was measured neutral in the forward, and its key-position pattern cannot be
// followed by the transposed backward without computing both forms.)
__device__ __forceinline__ void exp2_pack32(const float* v, int nvalid, float sl, float msl, uint32_t* w) {
  if (nvalid >= 32) {
#pragma unroll
    for (int e = 0; e < 16; ++e)
      w[e] = pack_bf16(fast_exp2(fmaf(v[2 * e], sl, -msl)), fast_exp2(fmaf(v[2 * e + 1], sl, -msl)));
  } else {
#pragma unroll
    for (int e = 0; e < 16; ++e)
      w[e] = pack_bf16(2 * e < nvalid ? fast_exp2(fmaf(v[2 * e], sl, -msl)) : 0.f,
                       2 * e + 1 < nvalid ? fast_exp2(fmaf(v[2 * e + 1], sl, -msl)) : 0.f);
  }
}

// The transposed form: 32 scores of one KEY against 32 consecutive queries, each with its
// own reference point msl[j] (one per query row), zero past nvalid queries.  Element for
// element the same arithmetic as exp2_pack32.
__device__ __forceinline__ void exp2_pack32_cols(const float* v, int nvalid, float sl, const float* msl, uint32_t* w) {
  if (nvalid >= 32) {
#pragma unroll
    for (int e = 0; e < 16; ++e)
      w[e] = pack_bf16(fast_exp2(fmaf(v[2 * e], sl, -msl[2 * e])), fast_exp2(fmaf(v[2 * e + 1], sl, -msl[2 * e + 1])));
  } else {
#pragma unroll
    for (int e = 0; e < 16; ++e)
      w[e] = pack_bf16(2 * e < nvalid ? fast_exp2(fmaf(v[2 * e], sl, -msl[2 * e])) : 0.f,
                       2 * e + 1 < nvalid ? fast_exp2(fmaf(v[2 * e + 1], sl, -msl[2 * e + 1])) : 0.f);
  }
}

// fp32 row statistics [rank][b][z][row] as a 3-D TMA map (row, z, b*rank) with 128-row boxes:
// a query tile's 512 bytes land in shared memory next to its Q / dO tiles, rows past the
// chunk zero-filled.
inline bool rows_map(CUtensorMap* m, const float* base, const rsa_geom* g, int nrank) {
  if (!base || (reinterpret_cast<uintptr_t>(base) & 15) || (g->chunk * 4) % 16)
    return fail(RSA_ERR_UNSUPPORTED, "row statistics must be 16-byte aligned with chunk %% 4 == 0"), false;
  uint64_t dims[3] = {uint64_t(g->chunk), uint64_t(g->heads), uint64_t(g->batch) * nrank};
  uint64_t str[2] = {uint64_t(g->chunk) * 4, uint64_t(g->heads) * g->chunk * 4};
  uint32_t box[3] = {uint32_t(TR), 1, 1};
  return encode_tmap(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, base, dims, str, box, CU_TENSOR_MAP_SWIZZLE_NONE);
}

struct OutView {  // strided output [rank][b][z][row][a]
  void* ptr;
  int64_t s_rank, s_b, s_z, s_row;
};

__device__ __forceinline__ int64_t out_off(const OutView& o, int rank, int b, int z, int row) {
  return int64_t(rank) * o.s_rank + int64_t(b) * o.s_b + int64_t(z) * o.s_z + int64_t(row) * o.s_row;
}

// Store 32 fp32 values (columns col0..col0+31 of one row): fp32 (optionally
// accumulating) and/or bf16.
__device__ __forceinline__ void store_row32(const OutView& acc, const OutView& fin, int accumulate, int rank, int b,
                                            int z, int row, int col0, float* v) {
  if (acc.ptr) {
    float* p = reinterpret_cast<float*>(acc.ptr) + out_off(acc, rank, b, z, row) + col0;
#pragma unroll
    for (int i = 0; i < 32; i += 4) {
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
    __nv_bfloat16* p = reinterpret_cast<__nv_bfloat16*>(fin.ptr) + out_off(fin, rank, b, z, row) + col0;
    if ((reinterpret_cast<uintptr_t>(p) & 31) == 0) {
      // whole 32-byte sectors per instruction (256-bit stores): a warp's stores touch 32
      // rows, and half-sector writes cost the L2 a merge each
#pragma unroll
      for (int i = 0; i < 32; i += 16)
        asm volatile("st.global.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(p + i),
                     "r"(pack_bf16(v[i], v[i + 1])), "r"(pack_bf16(v[i + 2], v[i + 3])),
                     "r"(pack_bf16(v[i + 4], v[i + 5])), "r"(pack_bf16(v[i + 6], v[i + 7])),
                     "r"(pack_bf16(v[i + 8], v[i + 9])), "r"(pack_bf16(v[i + 10], v[i + 11])),
                     "r"(pack_bf16(v[i + 12], v[i + 13])), "r"(pack_bf16(v[i + 14], v[i + 15]))
                     : "memory");
    } else {
#pragma unroll
      for (int i = 0; i < 32; i += 8)
        *reinterpret_cast<uint4*>(p + i) = make_uint4(pack_bf16(v[i], v[i + 1]), pack_bf16(v[i + 2], v[i + 3]),
                                                      pack_bf16(v[i + 4], v[i + 5]), pack_bf16(v[i + 6], v[i + 7]));
    }
  }
}

struct Geo {
  int n_rank, B, Z, c, L, org_lo, n_org;
  float scale;
};

__device__ __forceinline__ uint8_t* smem_base() {
  extern __shared__ uint8_t smem_raw[];
  return reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
}

// ------------------------------------------------------------ host side

inline int key_chunk(const rsa_geom* g) { return g->key_chunk > 0 ? g->key_chunk : g->chunk; }

// Geometry of a stream-capable kernel: any key chunk (a multiple of 8) per origin.
inline bool geom_ok_keys(const rsa_geom* g) {
  if (!g || g->key_chunk < 0) return false;
  const int ck = key_chunk(g);
  return g->n_rank >= 1 && g->batch >= 1 && g->heads >= 1 && g->chunk >= 1 && g->head_dim == HD &&
         g->n_org >= 1 && g->org_lo >= 0 && ck % 8 == 0 && g->seq_len % ck == 0 && g->chunk % 8 == 0 &&
         g->org_lo + g->n_org <= g->seq_len / ck;
}

// Geometry of the panel kernels: keys per origin == query rows per rank (RSA chunks).
inline bool geom_ok(const rsa_geom* g) { return geom_ok_keys(g) && key_chunk(g) == g->chunk; }

inline Geo to_geo(const rsa_geom* g) {
  return Geo{g->n_rank, g->batch, g->heads, g->chunk, g->seq_len, g->org_lo, g->n_org, g->scale};
}

// [rank][b][z][row][a] with a = 64 contiguous; `nrank` ranks merged into b; `rows` rows per
// (rank, b, z) (default: the query chunk; key_chunk(g) for key / value maps).
inline bool head_map(CUtensorMap* m, const rsa_view& v, const rsa_geom* g, int nrank, int rows = 0) {
  if (!v.ptr || !aligned16(v.ptr)) return fail(RSA_ERR_UNSUPPORTED, "fused: tensor not 16-byte aligned"), false;
  if (nrank > 1 && g->batch > 1 && v.s_rank != int64_t(g->batch) * v.s_b)
    return fail(RSA_ERR_UNSUPPORTED, "fused: rank stride must equal B * batch stride"), false;
  const int64_t sb = (g->batch == 1 && nrank > 1) ? v.s_rank : v.s_b;
  if (!stride_ok(v.s_row * 2) || !stride_ok(v.s_z * 2) || !stride_ok(sb * 2))
    return fail(RSA_ERR_UNSUPPORTED, "fused: strides must be multiples of 8 elements"), false;
  uint64_t dims[4] = {uint64_t(HD), uint64_t(rows > 0 ? rows : g->chunk), uint64_t(g->heads),
                      uint64_t(g->batch) * nrank};
  uint64_t str[3] = {uint64_t(v.s_row) * 2, uint64_t(v.s_z) * 2, uint64_t(sb) * 2};
  uint32_t box[4] = {64, TR, 1, 1};
  return encode_tmap(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, v.ptr, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B);
}

// head_map with 32-row x 32-column boxes, SWIZZLE_64B: one warp's rows x one column half
// (64-byte rows), for per-warp TMA stores of a 128 x 64 tile.
inline bool head_map_w32(CUtensorMap* m, const rsa_view& v, const rsa_geom* g, int nrank) {
  if (!v.ptr || !aligned16(v.ptr)) return fail(RSA_ERR_UNSUPPORTED, "fused: tensor not 16-byte aligned"), false;
  if (nrank > 1 && g->batch > 1 && v.s_rank != int64_t(g->batch) * v.s_b)
    return fail(RSA_ERR_UNSUPPORTED, "fused: rank stride must equal B * batch stride"), false;
  const int64_t sb = (g->batch == 1 && nrank > 1) ? v.s_rank : v.s_b;
  if (!stride_ok(v.s_row * 2) || !stride_ok(v.s_z * 2) || !stride_ok(sb * 2))
    return fail(RSA_ERR_UNSUPPORTED, "fused: strides must be multiples of 8 elements"), false;
  uint64_t dims[4] = {uint64_t(HD), uint64_t(g->chunk), uint64_t(g->heads), uint64_t(g->batch) * nrank};
  uint64_t str[3] = {uint64_t(v.s_row) * 2, uint64_t(v.s_z) * 2, uint64_t(sb) * 2};
  uint32_t box[4] = {32, 32, 1, 1};
  return encode_tmap(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, v.ptr, dims, str, box, CU_TENSOR_MAP_SWIZZLE_64B);
}

// [rank][b][z][row][col], col = blk * c + key: 5-D (key, blk, row, z, b*rank).
inline bool panel_map(CUtensorMap* m, const rsa_view& v, const rsa_geom* g, int nrank, uint32_t box_rows = TR) {
  if (!v.ptr || !aligned16(v.ptr)) return fail(RSA_ERR_UNSUPPORTED, "fused: panel not 16-byte aligned"), false;
  if (nrank > 1 && g->batch > 1 && v.s_rank != int64_t(g->batch) * v.s_b)
    return fail(RSA_ERR_UNSUPPORTED, "fused: panel rank stride must equal B * batch stride"), false;
  const int64_t sb = (g->batch == 1 && nrank > 1) ? v.s_rank : v.s_b;
  if (!stride_ok(v.s_row * 2) || !stride_ok(v.s_z * 2) || !stride_ok(sb * 2))
    return fail(RSA_ERR_UNSUPPORTED, "fused: panel strides must be multiples of 8 elements"), false;
  const int nblk = g->seq_len / g->chunk;
  uint64_t dims[5] = {uint64_t(g->chunk), uint64_t(nblk), uint64_t(g->chunk), uint64_t(g->heads),
                      uint64_t(g->batch) * nrank};
  uint64_t str[4] = {uint64_t(g->chunk) * 2, uint64_t(v.s_row) * 2, uint64_t(v.s_z) * 2, uint64_t(sb) * 2};
  uint32_t box[5] = {64, 1, box_rows, 1, 1};
  return encode_tmap(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 5, v.ptr, dims, str, box, CU_TENSOR_MAP_SWIZZLE_128B);
}

// Per-origin K / V maps for peer-resident origins (one rank's chunk each, possibly in
// another GPU's memory through CUDA IPC / UVA): origin j's tile (k0, z, b) is
// map[j] at coordinates (0, k0, z, b).
struct PeerMaps {
  CUtensorMap k[RSA_MAX_PEERS], v[RSA_MAX_PEERS];
};

inline bool peer_maps(PeerMaps* pm, const rsa_view* k, const rsa_view* v, const rsa_geom* g) {
  if (g->n_org > RSA_MAX_PEERS) return fail(RSA_ERR_UNSUPPORTED, "peer kernels: at most %d origins", RSA_MAX_PEERS), false;
  for (int j = 0; j < g->n_org; ++j)
    if (!head_map(&pm->k[j], k[j], g, 1) || !head_map(&pm->v[j], v[j], g, 1)) return false;
  return true;
}

inline OutView to_out(const rsa_view& v) { return OutView{v.ptr, v.s_rank, v.s_b, v.s_z, v.s_row}; }

inline bool out_ok(const rsa_view& v, int esz) {
  if (!v.ptr) return true;
  return aligned16(v.ptr) && (v.s_row * esz) % 16 == 0 && (v.s_z * esz) % 16 == 0 && (v.s_b * esz) % 16 == 0 &&
         (v.s_rank * esz) % 16 == 0;
}

// One launch of a persistent kernel.
template <typename K, typename A>
void launch_grid(K kernel, int grid, int threads, uint32_t smem, const A& args, void* stream) {
  kernel<<<grid, threads, smem, reinterpret_cast<cudaStream_t>(stream)>>>(args);
}

template <typename K, typename A>
int launch(K kernel, int items, uint32_t smem, const A& args, void* stream, const char* name,
           int threads = NTHREADS) {
  if (items <= 0) return RSA_OK;
  cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  launch_grid(kernel, persistent_grid(items), threads, smem, args, stream);
  return check_launch(name);
}

}  // namespace
}  // namespace rsa

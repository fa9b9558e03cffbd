/*
 * rsa_b200.h -- C ABI of librsa_b200.so, the sm_100a kernels behind the
 * Ring Self-Attention (RSA) drop-in boundary.
 *
 * The reference (arXiv 2105.13120's `ringseq` package, a float64 NumPy
 * simulator) has no FFI layer: its boundary is the Python API of
 * ringseq.ring_attention / ringseq.sparse_attention / ringseq.tensor_ops.
 * Each entry point below replaces the arithmetic of one reference function
 * (cited per function); the host package paper_2105_13120_b200 binds them
 * with ctypes and keeps the reference's Python names and signatures.
 *
 * Conventions
 *   - Plain C types only.  Device buffers are raw pointers owned by the
 *     caller (the torch caching allocator); nothing is allocated here.
 *   - `stream` is a cudaStream_t passed as void*; every call is asynchronous
 *     on it and returns an int status (RSA_OK or an RSA_ERR_* code); no C++
 *     exception crosses the ABI.  rsa_last_error() describes the last
 *     failure on the calling thread.
 *   - Element strides are in elements (not bytes); the innermost dimension
 *     is always contiguous.
 *   - Per-head tensors are addressed as [rank][b][z][row][col] through an
 *     rsa_view, so the same kernels serve (a) N logical ranks resident in one
 *     GPU's HBM and (b) one rank per GPU with ring-delivered chunks.
 */
#ifndef RSA_B200_H
#define RSA_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RSA_ABI_VERSION 4

enum rsa_status {
  RSA_OK = 0,
  RSA_ERR_INVALID = 1,     /* bad argument (maps to ShapeError / ConfigError) */
  RSA_ERR_UNSUPPORTED = 2, /* layout the requested kernel cannot tile         */
  RSA_ERR_CUDA = 3,        /* CUDA runtime / launch failure                    */
  RSA_ERR_NUMERIC = 4      /* non-finite input (maps to NumericError)          */
};

enum rsa_dtype { RSA_F32 = 0, RSA_BF16 = 1 };

/* A strided 5-D view [rank][b][z][row][col] with unit column stride. */
typedef struct rsa_view {
  void* ptr;
  int64_t s_rank; /* elements between consecutive ranks (or origin blocks) */
  int64_t s_b;
  int64_t s_z;
  int64_t s_row;
} rsa_view;

/* Geometry shared by the fused RSA kernels. */
typedef struct rsa_geom {
  int32_t n_rank;    /* query ranks covered by this launch (1 per GPU, N when resident) */
  int32_t batch;     /* B */
  int32_t heads;     /* Z */
  int32_t chunk;     /* c = L / N */
  int32_t head_dim;  /* A */
  int32_t seq_len;   /* L: width of the probability panel */
  int32_t org_lo;    /* first origin chunk resident in this launch */
  int32_t n_org;     /* number of consecutive origin chunks resident */
  float scale;       /* 1/sqrt(A) */
  int32_t key_chunk; /* keys per origin chunk; 0 = chunk (RSA).  Only the stream-mode entry
                        points (rsa_fwd_factored_ex without a panel, rsa_bwd_*_stream) accept
                        key_chunk != chunk -- the Linformer's projected keys; seq_len is then
                        the total key count, a multiple of key_chunk. */
} rsa_geom;

int rsa_abi_version(void);
const char* rsa_last_error(void);
int rsa_num_sms(void);

/* Test hook: cap the grid of every persistent kernel at max_ctas CTAs (0 = one per SM,
 * the default), so small shapes exercise the multi-unit-per-CTA paths (resident K tiles,
 * next-head prefetch, phase flips) that large launches take.  Returns the previous cap. */
int rsa_set_max_ctas(int max_ctas);

/* ------------------------------------------------------------ primitives */

/*
 * Batched GEMM, C = alpha * op(A) * op(B) (+ C if accumulate).
 * Replaces ringseq/tensor_ops.py:44-72 (`matmul`).  trans_a=0: A stored
 * M x K; trans_a=1: A stored K x M.  trans_b=0: B stored K x N; trans_b=1:
 * B stored N x K.  Batch index i = i1 * nb2 + i2 with strides (s1, s2) per
 * operand; a zero stride broadcasts.  bf16 operands with 16-byte-aligned
 * rows run on tcgen05 tensor cores (fp32 accumulation in TMEM); any other
 * layout runs on the SIMT CUDA path.  c_dtype selects fp32 or bf16 output.
 */
int rsa_gemm(int M, int N, int K, const void* A, int a_dtype, int64_t lda, int trans_a, int64_t a_s1, int64_t a_s2,
             const void* B, int b_dtype, int64_t ldb, int trans_b, int64_t b_s1, int64_t b_s2, void* C, int c_dtype,
             int64_t ldc, int64_t c_s1, int64_t c_s2, int nb1, int nb2, float alpha, int accumulate, void* stream);

/* Force one backend: 0 = auto, 1 = tcgen05 only (RSA_ERR_UNSUPPORTED if it
 * cannot tile), 2 = SIMT only.  Used by the tests to cover both paths. */
int rsa_gemm_set_backend(int backend);

/*
 * Row softmax y = exp(s*x - max(s*x)) / sum, over `cols` per row.
 * Replaces ringseq/tensor_ops.py:75-84 (`softmax_rows`).  Any non-finite
 * input sets *nonfinite_flag (device int) to 1; the host raises NumericError.
 */
int rsa_softmax_rows(const void* x, int x_dtype, int64_t rows, int64_t cols, int64_t ld_x, float scale, void* y,
                     int y_dtype, int64_t ld_y, int* nonfinite_flag, void* stream);

/*
 * Softmax Jacobian, ds = p * (dp - rowsum(dp * p)) * scale.
 * Replaces ringseq/ring_attention.py:187-190 (and reference.py:99-100).
 */
int rsa_softmax_bwd(const void* p, int p_dtype, int64_t ld_p, const float* dp, int64_t ld_dp, int64_t rows,
                    int64_t cols, float scale, void* ds, int ds_dtype, int64_t ld_ds, void* stream);

/* out[r] = sum_c a[r,c] * b[r,c] (fp32 accumulate); a, b bf16. */
int rsa_rowdot(const void* a, int64_t lda, const void* b, int64_t ldb, int64_t rows, int64_t cols, float* out,
               void* stream);

/*
 * Backward prologue for a factored panel (see rsa_fwd_factored):
 * out[r] = scale[r] * sum_c a[r,c] * b[r,c] and a_scaled[r,:] = bf16(scale[r] * a[r,:]).
 * With a = dO, b = O and scale = the panel's row scale this gives D*r and
 * dO*r, which let rsa_bwd_fused / rsa_bwd_dkdv / rsa_bwd_dq consume the
 * factored panel P~ unchanged: P (dP - D) = P~ (dO*r V^T - D*r) and
 * P^T dO = P~^T (dO*r)  (ringseq/ring_attention.py:180-205).
 */
int rsa_rowdot_scale(const void* a, int64_t lda, const void* b, int64_t ldb, const float* scale, int64_t rows,
                     int64_t cols, float* out, void* a_scaled, int64_t ld_as, void* stream);

/*
 * Materialise probabilities from a factored panel: y[r,c] = scale[r] * p[r,c]
 * (p bf16; y fp32 or bf16 per y_dtype).  The reference's probs
 * (ringseq/ring_attention.py:89-94) on demand; not on the fwd/bwd path.
 */
int rsa_panel_normalize(const void* p, int64_t ld_p, const float* scale, int64_t rows, int64_t cols, void* y,
                        int y_dtype, int64_t ld_y, void* stream);

/*
 * Exact GELU y = x * Phi(x) (ringseq/tensor_ops.py:87-90, the reference's mlp_forward
 * activation, ringseq/reference.py:177-185) and its backward dx = dy * (Phi(x) + x phi(x)),
 * elementwise over n values; fp32 / bf16 per dtype argument.
 */
int rsa_gelu(const void* x, int x_dtype, int64_t n, void* y, int y_dtype, void* stream);
int rsa_gelu_bwd(const void* x, int x_dtype, const void* dy, int dy_dtype, int64_t n, void* dx, int dx_dtype,
                 void* stream);

/*
 * y[i] = sum over d = 0..n_rank-1 (ascending) of x[d * rank_stride + i], i < count; x and y
 * fp32 or bf16 per x_dtype / y_dtype, fp32 accumulation.  The cross-rank sum of per-rank
 * partial projections: the Linformer's ring-accumulate (ringseq/sparse_attention.py:59-71)
 * when every rank is resident on one GPU (also the BERT harness's position-embedding
 * gradient, a sum over the batch).  Vectorised when count and rank_stride are multiples
 * of 4 and the buffers 16-byte aligned; any layout otherwise.
 */
int rsa_sum_ranks(const void* x, int x_dtype, int64_t n_rank, int64_t count, int64_t rank_stride, void* y,
                  int y_dtype, void* stream);

/* --------------------------------------------------- fused RSA kernels */

/*
 * Stage 1 of the RSA forward (ringseq/ring_attention.py:89-94): for every
 * query row, the running max m and sum l of exp(scale * q.k) over the keys
 * of origins [org_lo, org_lo + n_org).  stats is float2 [slot][rank][b][z][c]
 * (slot stride = n_rank*B*Z*c); this launch writes slot `slot`.  Stats are
 * kept in base 2: m = max(scale*log2(e)*s), l = sum 2^(scale*log2(e)*s - m).
 * A non-finite score sets *nonfinite_flag (device int, may be NULL).
 */
int rsa_fwd_stats(const rsa_geom* g, rsa_view q, rsa_view k, float* stats, int slot, int* nonfinite_flag,
                  void* stream);

/*
 * Stage 2 of the RSA forward (ringseq/ring_attention.py:97-103 plus the
 * softmax normalisation): combines `n_slots` stat slots, recomputes the
 * score tiles, writes the bf16 probability panel blocks of the resident
 * origins, and accumulates O = sum_j P_j V_j in TMEM.  o_acc (fp32, may be
 * NULL) is read-modify-written when accumulate != 0; o_out (bf16, may be
 * NULL) receives the final output.
 */
int rsa_fwd_probs_pv(const rsa_geom* g, rsa_view q, rsa_view k, rsa_view v, const float* stats, int n_slots,
                     rsa_view panel, rsa_view o_acc, int accumulate, rsa_view o_out, void* stream);

/*
 * Both forward stages in one launch when every origin is resident (N logical
 * ranks in one GPU's HBM, or N = 1): per query tile a statistics pass over
 * all keys, then the probability/PV pass; replaces _score_panel +
 * _apply_values (ringseq/ring_attention.py:89-103) for all ranks at once.
 */
int rsa_fwd_resident(const rsa_geom* g, rsa_view q, rsa_view k, rsa_view v, rsa_view panel, rsa_view o_out,
                     int* nonfinite_flag, void* stream);

/*
 * Single-launch forward with a FACTORED probability panel, every origin
 * resident (org_lo = 0, n_org = L / c): panel = bf16(P~), P~ = 2^(s*sl - m)
 * with m the row max, and rowscale[row] = 1 / sum_k P~[row, k] (fp32,
 * [rank][b][z][c]), so the reference's probs are P = rowscale * P~
 * (ringseq/ring_attention.py:89-94) and o_out = P V (:97-103).  One exp2 per
 * panel element (rsa_fwd_resident spends two); the row sum is accumulated by
 * the tensor core from a block of ones next to V.  Backward consumers take
 * the factored panel through rsa_rowdot_scale.
 */
int rsa_fwd_factored(const rsa_geom* g, rsa_view q, rsa_view k, rsa_view v, rsa_view panel, rsa_view o_out,
                     float* rowscale, int* nonfinite_flag, void* stream);

/*
 * V-ring half of the RSA backward (ringseq/ring_attention.py:180-205) for
 * the resident origins: per key tile, dP = dO V_j^T and the softmax Jacobian
 * dS = P (dP - D) scale (kept in shared memory, never written to HBM), then
 * the key/value gradient contributions dK_j = dS_j^T Q, dV_j = P_j^T dO
 * summed over the launch's query ranks (the all-reduce of
 * ringseq/ring_attention.py:206-209 when the ranks are resident).
 * D[row] = rowsum(dO * O) = rowsum(dP * P) (see rsa_rowdot).  dk/dv are fp32
 * (accumulate != 0 adds) or bf16 outputs per dkv_dtype.
 */
int rsa_bwd_dkdv(const rsa_geom* g, rsa_view q, rsa_view v, rsa_view dout, rsa_view panel, const float* dvec,
                 rsa_view dk, rsa_view dv, int dkv_dtype, int accumulate, void* stream);

/*
 * K-ring half of the RSA backward (ringseq/ring_attention.py:192-196):
 * dQ = sum_j dS_j K_j over the resident origins, with dS recomputed from
 * P, dO V_j^T and D exactly as in rsa_bwd_dkdv (so no dS panel exists).
 * dq_acc fp32 (optional, accumulate != 0 adds) and/or dq_out bf16.
 */
int rsa_bwd_dq(const rsa_geom* g, rsa_view dout, rsa_view k, rsa_view v, rsa_view panel, const float* dvec,
               rsa_view dq_acc, int accumulate, rsa_view dq_out, void* stream);

/* Can the fused kernels tile this geometry (head_dim, chunk, alignment)? */
int rsa_fused_supported(const rsa_geom* g);

/*
 * Whole RSA backward of ringseq/ring_attention.py:168-209 in ONE pass over
 * the probability panel: per head, dP = dO V_j^T, dS = P (dP - D) scale
 * (shared memory only), dV_j = P_j^T dO and dK_j = dS_j^T Q summed over the
 * launch's query ranks (the all-reduce of :206-209 when resident), and
 * dQ = sum_j dS_j K_j (the K ring of :192-196), all accumulated in TMEM.
 * Replaces the rsa_bwd_dkdv + rsa_bwd_dq pair (which read the panel twice)
 * when a head's query rows fit four 128-row tiles:
 * n_rank * ceil(chunk / 128) <= 4 (rsa_bwd_fused_supported).
 * dq: fp32 dq_acc (accumulate_dq != 0 adds) and/or bf16 dq_out; dk/dv:
 * bf16 or fp32 per dkv_dtype (fp32 with accumulate_dkv != 0 adds).
 */
int rsa_bwd_fused(const rsa_geom* g, rsa_view q, rsa_view k, rsa_view v, rsa_view dout, rsa_view panel,
                  const float* dvec, rsa_view dq_acc, int accumulate_dq, rsa_view dq_out, rsa_view dk, rsa_view dv,
                  int dkv_dtype, int accumulate_dkv, void* stream);
int rsa_bwd_fused_supported(const rsa_geom* g);

/* ------------------------------------------------ stream mode and ring hops */

/*
 * Options of rsa_fwd_factored_ex, the generalised factored forward.  All-zero options give
 * rsa_fwd_factored's behaviour except that the panel is NOT written (stream mode):
 *
 *   panel          bf16 P~ panel to write (ptr NULL: stream mode -- only O and the row
 *                  statistics survive, so memory per rank is O(c) instead of O(c * L)).
 *   rowmax         out (may be NULL): m = the reference point per row, in the scaled base-2
 *                  units of the panel (P~ = 2^(s * scale * log2(e) - m)); with rowscale this
 *                  is everything the stream-mode backward needs to recompute P~ bit for bit.
 *   rowmax_in      in (may be NULL): use these reference points instead of the first key
 *                  tile's max (stride rowmax_in_stride floats per row: 1, or 2 to read the m
 *                  of rsa_fwd_stats' float2 (m, l) slots).  rowmax_exact != 0 declares them
 *                  the true row maxima (no headroom check: the two-pass fallback).
 *   o_acc, l_acc   ring hops: fp32 running O~ = sum_k P~ V and l = sum_k P~ over the origins
 *                  of earlier launches ([rank][b][z][row][a] and [rank][b][z][row]); acc_in
 *                  adds them in, final_hop = 0 writes them back instead of finishing.
 *   final_hop      != 0 (or o_acc NULL): O = O~ / l to o_out (bf16), rowscale = 1 / l.
 *
 * One K/V-ring hop of ringseq/ring_attention.py:89-103 in ONE pass: hop 0 computes the
 * reference point, later hops reuse it (rowmax_in), so neither the two-pass statistics nor
 * the recomputation of S of rsa_fwd_stats + rsa_fwd_probs_pv is needed.
 */
typedef struct rsa_fwd_ext {
  rsa_view panel;
  float* rowmax;
  const float* rowmax_in;
  int32_t rowmax_in_stride;
  int32_t rowmax_exact;
  rsa_view o_acc;
  float* l_acc;
  int32_t acc_in;
  int32_t final_hop;
} rsa_fwd_ext;

int rsa_fwd_factored_ex(const rsa_geom* g, rsa_view q, rsa_view k, rsa_view v, const rsa_fwd_ext* ext,
                        rsa_view o_out, float* rowscale, int* flag, void* stream);

/*
 * Stream-mode backward (ringseq/ring_attention.py:168-209 without a saved panel): the
 * probabilities are recomputed tile by tile as P~ = 2^(q.k * scale * log2(e) - rowmax) --
 * the same tensor-core products and the same exp2 as the forward, so P~ equals the panel
 * rsa_fwd_factored would have stored, bit for bit -- and used at once, never written.
 * dout_scaled = dO * r and dvec = D * r come from rsa_rowdot_scale with the forward's
 * rowscale r, exactly as for a factored panel.
 *   rsa_bwd_kv_stream: per key tile, walking every query tile of the launch's ranks:
 *     dV_j += P~^T (dO r), dK_j += dS^T Q with dS = P~ (dO r V^T - D r) (scale applied);
 *     dk / dv bf16, or fp32 (accumulate != 0 adds) per dkv_dtype.
 *   rsa_bwd_q_stream: per query tile, walking every key tile of the resident origins:
 *     dQ = sum_j dS_j K_j; fp32 dq_acc (accumulate != 0 adds) and/or bf16 dq_out.
 * key_chunk may differ from chunk (Linformer keys).
 */
int rsa_bwd_kv_stream(const rsa_geom* g, rsa_view q, rsa_view k, rsa_view v, rsa_view dout_scaled,
                      const float* rowmax, const float* dvec, rsa_view dk, rsa_view dv, int dkv_dtype,
                      int accumulate, void* stream);
int rsa_bwd_q_stream(const rsa_geom* g, rsa_view q, rsa_view k, rsa_view v, rsa_view dout_scaled,
                     const float* rowmax, const float* dvec, rsa_view dq_acc, int accumulate, rsa_view dq_out,
                     void* stream);

/*
 * The two stream-mode backward kernels above in ONE pass (ringseq/ring_attention.py:168-209,
 * the V-ring and K-ring backward, without a saved panel): per key tile, walking every query
 * tile, dV_j and dK_j as rsa_bwd_kv_stream and dQ_part = dS K_j added into the fp32
 * accumulator dq_acc ([n_rank][B][Z][chunk][64], contiguous, zeroed first unless
 * accumulate_dq; it holds the sum WITHOUT the 1/sqrt(A) factor) by TMA reduce-add in L2;
 * S, dP and every exp2 are computed once.  dq_out (optional, bf16 view) receives
 * bf16(dq_acc / sqrt(A)) at the end.  dK / dV are summed in a
 * fixed order; dQ's sum over key tiles is in arrival order (not bitwise reproducible).
 */
int rsa_bwd_stream_fused(const rsa_geom* g, rsa_view q, rsa_view k, rsa_view v, rsa_view dout_scaled,
                         const float* rowmax, const float* dvec, rsa_view dk, rsa_view dv, int dkv_dtype,
                         int accumulate_dkv, float* dq_acc, int accumulate_dq, rsa_view dq_out, void* stream);

/*
 * The panel-mode backward (ringseq/ring_attention.py:168-209 on the saved probs) in one pass
 * at ANY length: rsa_bwd_stream_fused's structure with P~ read from the factored panel instead
 * of recomputed, so the panel is read once where rsa_bwd_dkdv + rsa_bwd_dq read it twice (and
 * rsa_bwd_fused needs a head's query rows in 4 tiles).  Inputs as rsa_bwd_dkdv (dout_scaled
 * = dO * r, dvec = D * r from rsa_rowdot_scale); dQ through the fp32 accumulator dq_acc as in
 * rsa_bwd_stream_fused (arrival-order sum over key tiles).
 */
int rsa_bwd_panel_fused(const rsa_geom* g, rsa_view q, rsa_view k, rsa_view v, rsa_view dout_scaled, rsa_view panel,
                        const float* dvec, rsa_view dk, rsa_view dv, int dkv_dtype, int accumulate_dkv, float* dq_acc,
                        int accumulate_dq, rsa_view dq_out, void* stream);

/*
 * Linformer K/V projection (ringseq/sparse_attention.py:111-123, the sequence-sharded
 * K'_d = E_d K_d, V'_d = F_d V_d and their ring-accumulate) for every head at once:
 * K' = sum over the resident origins [org_lo, org_lo + n_org) of E_d K_d (likewise V'), one
 * contraction over their n_org * chunk positions.  e / f: bf16 (proj_dim x L) row-major with
 * leading dimension ld_proj (origin d's columns at d * chunk); k / v: [n_org][B][Z][chunk][64]
 * bf16 views.  k_acc / v_acc: fp32 [B][Z][proj_dim][64] contiguous outputs (zero-filled
 * here, then added into by TMA reduce-add); k_low / v_low (optional): bf16 copies of them.
 * Needs head_dim 64, chunk % 64 == 0, proj_dim % 128 == 0 and B*Z % 4 == 0.
 */
int rsa_linformer_project(const rsa_geom* g, int proj_dim, const void* e, const void* f, int64_t ld_proj, rsa_view k,
                          rsa_view v, float* k_acc, float* v_acc, void* k_low, void* v_low, void* stream);

/*
 * The projections' gradients (the Linformer backward): for every
 * resident origin d, grad_e[:, d-block] = sum over the B*Z heads of dK'_h K_{d,h}^T, and
 * grad_f likewise from dV' and V.  dk_low / dv_low: bf16 [B][Z][proj_dim][64] contiguous;
 * k / v as rsa_linformer_project; grad_e / grad_f: fp32 (proj_dim x L) row-major, leading
 * dimension ld_grad, written (not accumulated) at origin d's columns d * chunk.  Needs
 * head_dim 64, chunk % 256 == 0 and proj_dim % 128 == 0.
 */
int rsa_linformer_proj_grad(const rsa_geom* g, int proj_dim, const void* dk_low, const void* dv_low, rsa_view k,
                            rsa_view v, float* grad_e, float* grad_f, int64_t ld_grad, void* stream);

/*
 * The projections' transposes (the Linformer backward): for every
 * resident origin d and head h, dk[d][h] = E_d^T dK'_h and dv[d][h] = F_d^T dV'_h.  e / f as
 * rsa_linformer_project (origin d's columns at (org_lo + d) * chunk); dk_low / dv_low: bf16
 * [B][Z][proj_dim][64] contiguous; dk / dv: bf16 [n_org][B][Z][chunk][64] views.  Needs
 * head_dim 64, chunk % 128 == 0, proj_dim % 64 == 0 and B*Z % 4 == 0.
 */
int rsa_linformer_proj_back(const rsa_geom* g, int proj_dim, const void* e, const void* f, int64_t ld_proj,
                            const void* dk_low, const void* dv_low, rsa_view dk, rsa_view dv, void* stream);

/* ------------------------------------------ BERT harness */

/*
 * Not on the RSA path: the embedding lookup and masked-LM loss that turn the encoder stack
 * into the paper's whole-model BERT training step; the reference has
 * neither.  Rows are laid out [rank][b][i], rank d holding positions d*chunk + i (the
 * contiguous chunk layout of ringseq/cluster.py:73-88).
 *   rsa_embed:        x[row] = tok[ids[row]] + pos[position(row)]        (bf16, hidden % 8 == 0)
 *   rsa_embed_bwd:    dtok[ids[row]] += dx[row] (fp32 atomics); dpos[position(row)] += dx[row] when
 *                     dpos is not NULL (fp32 atomics; the harness sums positions with rsa_sum_ranks)
 *   rsa_softmax_xent: loss[r] = logsumexp(logits[r]) - logits[r][targets[r]] and
 *                     dlogits[r] = (softmax(logits[r]) - onehot(targets[r])) * grad_scale (bf16)
 */
int rsa_embed(const int* ids, int64_t n_rank, int64_t batch, int64_t chunk, const void* tok, const void* pos,
              int64_t hidden, void* x, void* stream);
int rsa_embed_bwd(const int* ids, int64_t n_rank, int64_t batch, int64_t chunk, const void* dx, int64_t hidden,
                  float* dtok, float* dpos, void* stream);
int rsa_softmax_xent(const float* logits, int64_t ld, const int* targets, int64_t rows, int64_t vocab, float* loss,
                     void* dlogits, int64_t ld_d, float grad_scale, void* stream);

/* --------------------------------------------- peer-resident origins (NVLink) */

#define RSA_MAX_PEERS 8

/*
 * One rank's whole RSA forward / backward with every origin's K and V chunk read
 * in place from the rank that owns it -- device pointers opened through CUDA IPC
 * (CUDA IPC), so on an NVSwitch box the tiles stream over NVLink inside the
 * kernel's TMA pipeline instead of travelling a ring of NCCL hops (the K/V rings of
 * ringseq/ring_attention.py:124-217).  g: n_rank = 1 (this rank's query chunk),
 * org_lo = 0, n_org = N <= RSA_MAX_PEERS; k_origin[j] / v_origin[j] view origin j's
 * [1][B][Z][c][A] chunk (peers' buffers come from rsa_ipc_alloc / rsa_ipc_open below,
 * driven by paper_2105_13120_b200/distributed.py:PeerRing).  The forward is rsa_fwd_factored's single pass (factored
 * panel, row scale); the backward is rsa_bwd_fused's single pass with fp32 dK / dV
 * partials for every origin ([N][B][Z][c][A], dk_part / dv_part) left for the
 * caller's reduce-scatter (the reference's all-reduce + slice, :206-209).
 */
int rsa_fwd_factored_peer(const rsa_geom* g, rsa_view q, const rsa_view* k_origin, const rsa_view* v_origin,
                          rsa_view panel, rsa_view o_out, float* rowscale, int* flag, void* stream);
int rsa_bwd_fused_peer(const rsa_geom* g, rsa_view q, const rsa_view* k_origin, const rsa_view* v_origin,
                       rsa_view dout, rsa_view panel, const float* dvec, rsa_view dq_out, rsa_view dk_part,
                       rsa_view dv_part, void* stream);

/*
 * The registered K/V buffers those kernels read: rsa_ipc_alloc cudaMallocs `bytes`
 * and writes its 64-byte CUDA IPC handle to `handle`; every other rank maps it with
 * rsa_ipc_open (cudaIpcOpenMemHandle, lazy peer access).  Tear down in the order
 * rsa_ipc_close on every mapping, then rsa_ipc_free by the owner.  Stands in for the
 * ring's per-hop send/recv buffers (ringseq/ring_attention.py:124-217).
 */
#define RSA_IPC_HANDLE_BYTES 64
int rsa_ipc_alloc(size_t bytes, void** ptr, void* handle);
int rsa_ipc_open(const void* handle, void** ptr);
int rsa_ipc_close(void* ptr);
int rsa_ipc_free(void* ptr);


#ifdef __cplusplus
}
#endif

#endif /* RSA_B200_H */

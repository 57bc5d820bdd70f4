/*
 * s24.h -- C ABI of libs24.so, the sm_100a (B200) backend for the Squared-ReLU
 * FFN with 2:4 activation sparsity (arXiv 2503.16672).
 *
 * The reference (pkg/src/srelu24, pure Python/numpy) has no FFI: its operator
 * boundary is the Python function API re-exported by
 * pkg/src/srelu24/__init__.py:7-91. Each entry point below is the device
 * kernel that replaces one stage of that API; the Python package
 * paper_2503_16672_b200 binds them with ctypes and keeps
 * the reference's function names, arguments and exceptions above them.
 *
 * Conventions
 *  - Every pointer argument is a DEVICE pointer unless stated; the caller owns
 *    all memory (including outputs and workspace). The library never frees
 *    caller memory and holds no device memory of its own: the GEMMs distribute
 *    their tiles with Blackwell cluster launch control (the hardware cancels
 *    not-yet-started clusters of the same launch and a running cluster takes
 *    their tiles), so no scheduler counters live between or across calls and
 *    any launch may run concurrently with any other, captured in a CUDA graph
 *    or not.
 *  - `stream` is a cudaStream_t passed as void*; every call is asynchronous on
 *    it. Shape/argument validation happens on the host before any launch.
 *  - Return value: 0 (S24_OK) or an s24_status code; s24_last_error() returns
 *    a thread-local message for the last failure on the calling thread. The
 *    codes map 1:1 onto pkg/src/srelu24/errors.py classes.
 *  - Matrices are row-major with explicit leading dimensions in ELEMENTS.
 *    bf16 = IEEE bfloat16 stored as uint16.
 *  - "hw metadata": the tcgen05.mma.sp operand-E layout documented in
 *    paper_2503_16672_b200/csrc/meta.cuh: 4 bits (i0 | i1<<2) per group of 4,
 *    in 2048-byte atoms of 128 rows x 128 logical columns. Row count padded to
 *    a multiple of 128, column count a multiple of 128.
 *    Size = s24_meta_hw_bytes(rows, cols).
 *  - "ref metadata": uint8 [rows, cols/4, 2] positions (i0, i1), i0 < i1, the
 *    reference's Sparse24Matrix.meta (pkg/src/srelu24/sparse24.py:30-47).
 *  - Thread safety: re-entrant. Host-side state is limited to read-only,
 *    once-initialised caches (kernel attributes, the SM count, the driver's
 *    tensor-map encoder entry point); there is no device-side state.
 */
#ifndef S24_H_
#define S24_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  S24_OK = 0,
  S24_ERR_DIMENSION = 1,   /* errors.py:4   DimensionError   */
  S24_ERR_ORIENTATION = 2, /* errors.py:12  OrientationError */
  S24_ERR_MASK = 3,        /* errors.py:16  MaskError        */
  S24_ERR_PRECISION = 4,   /* errors.py:8   PrecisionError   */
  S24_ERR_CONFIG = 5,      /* errors.py:34  ConfigError      */
  S24_ERR_STATE = 6,       /* errors.py:42  StateError       */
  S24_ERR_CUDA = 7         /* launch / runtime failure       */
} s24_status;

typedef enum { S24_F32 = 0, S24_BF16 = 1 } s24_dtype;

/* ---------------------------------------------------------------- misc */
const char* s24_last_error(void);
const char* s24_version(void);
/* bytes of a hw-metadata buffer for a rows x cols (logical) 2:4 matrix */
int64_t s24_meta_hw_bytes(int64_t rows, int64_t cols);

/* ---------------------------------------------------------------- sparsify
 * Replaces sparsify_token_wise (pkg/src/srelu24/sparse24.py:80-93).
 * a: [rows, cols] (dtype, lda). Outputs (each nullable except vals):
 *   vals    bf16 [rows, cols/2]   kept values, group g at [2g, 2g+1]
 *   meta_ref uint8 [rows, cols/4, 2]
 *   meta_hw  hw layout (needs cols % 128 == 0; rows padded to 128 by caller)
 *   mask    uint8 [rows, cols] 0/1 keep mask
 *   stats   uint64[2] += (nonzeros before, nonzeros after)   */
int s24_sparsify_token(const void* a, int dtype, int64_t rows, int64_t cols, int64_t lda, void* vals,
                       uint8_t* meta_ref, uint8_t* meta_hw, uint8_t* mask, unsigned long long* stats,
                       void* stream);

/* Replaces sparsify_feature_wise (sparse24.py:96-115): groups of 4 rows down
 * each column. vals_t: bf16 [cols, rows/2] (transposed: K-major along rows);
 * meta_ref uint8 [rows/4, cols, 2]; meta_hw: rows=cols (features), K=rows. */
int s24_sparsify_feature(const void* a, int dtype, int64_t rows, int64_t cols, int64_t lda, void* vals_t,
                         uint8_t* meta_ref, uint8_t* meta_hw, uint8_t* mask, unsigned long long* stats,
                         void* stream);

/* Replaces sparsify_feature_wise_masked (sparse24.py:118-129): as
 * s24_sparsify_feature, with every entry where fwd_mask (uint8 [rows, cols],
 * 0/1, row-major) is 0 read as zero before the selection and before the
 * counts, so masked-out values never count as dropped. */
int s24_sparsify_feature_masked(const void* a, int dtype, int64_t rows, int64_t cols, int64_t lda,
                                const uint8_t* fwd_mask, void* vals_t, uint8_t* meta_ref, uint8_t* meta_hw,
                                uint8_t* mask, unsigned long long* stats, void* stream);

/* Replaces compress_token_wise_with_mask (sparse24.py:138-154). bad_groups
 * (device int, caller-zeroed) counts groups whose mask does not have exactly 2
 * bits; the binding raises MaskError when it is non-zero. */
int s24_compress_token_with_mask(const void* a, int dtype, int64_t rows, int64_t cols, int64_t lda,
                                 const uint8_t* mask, void* vals, uint8_t* meta_ref, uint8_t* meta_hw,
                                 int* bad_groups, void* stream);

/* Replaces decompress (sparse24.py:157-167), token orientation. Exactly one
 * of meta_ref / meta_hw is non-null. out: [rows, cols] (out_dtype, ldo). */
int s24_decompress_token(const void* vals, const uint8_t* meta_ref, const uint8_t* meta_hw, int64_t rows,
                         int64_t cols, void* out, int out_dtype, int64_t ldo, void* stream);

/* feature orientation: vals_t [cols, rows/2]; meta_ref [rows/4, cols, 2] or
 * meta_hw (rows=cols, K=rows). out [rows, cols]. */
int s24_decompress_feature(const void* vals_t, const uint8_t* meta_ref, const uint8_t* meta_hw, int64_t rows,
                           int64_t cols, void* out, int out_dtype, int64_t ldo, void* stream);

/* metadata converters, token orientation (rows x cols logical) */
int s24_meta_hw_to_ref(const uint8_t* meta_hw, int64_t rows, int64_t cols, uint8_t* meta_ref, void* stream);
int s24_meta_ref_to_hw(const uint8_t* meta_ref, int64_t rows, int64_t cols, uint8_t* meta_hw, void* stream);

/* ---------------------------------------------------------------- permutation
 * Row gather out[i, :] = in[src[i], :] over `row_bytes` bytes per row.
 * permute_rows (matcore.py:291-296) uses src = inverse(p);
 * inverse_permute_rows (matcore.py:299-302) uses src = p. */
int s24_gather_rows(const void* in, int64_t rows, int64_t row_bytes, int64_t ld_in_bytes, const int* src,
                    void* out, int64_t ld_out_bytes, void* stream);

/* diagnostics: one thread writes the GPU's global nanosecond timer to *out
 * when the stream reaches it (per-kernel timelines inside CUDA graphs,
 * scripts/timeline.py --graph) */
int s24_timestamp(unsigned long long* out, void* stream);
/* diagnostics: `ctas` one-warp CTAs busy-wait `ns` nanoseconds and write
 * (SM clock cycles, nanoseconds) pairs to out[2*ctas]: the SM clock while
 * other work runs (scripts/clock_probe.py) */
int s24_clock_probe(unsigned long long* out, int ctas, int64_t ns, void* stream);

/* ---------------------------------------------------------------- split plan
 * Replaces partition_features (splitgemm.py:41-52) on device counts: stable
 * ascending (count, index) order, the first n_sparse features form the sparse
 * set. Outputs ascending index lists sparse_idx[n_sparse], dense_idx[h -
 * n_sparse], and feat_pos[h] = rank in sparse list, or -(rank in dense)-1.
 * h <= 65536. */
int s24_plan(const int* counts, int64_t h, int64_t n_sparse, int* sparse_idx, int* dense_idx, int* feat_pos,
             void* stream);

/* ---------------------------------------------------------------- K4
 * Feature-wise (transposed) split of a token-wise compressed [n, h] matrix
 * (vals [n, h/2] + meta_hw; e.g. the forward activation or g_pre), replacing
 * the apply_mask -> column gather -> sparsify_feature_wise part of
 * split_gemm_t (splitgemm.py:72-80):
 *   vs   bf16 [n_sparse_pad128, n/2] + es (hw meta, rows = sparse rank, K = n)
 *        feature-wise 2:4 of the sparse features, K-major along tokens
 *   vd   bf16 [n_dense_pad128, n] dense features, transposed
 *   stats uint64[2] += (nonzeros before, after) over the sparse features.
 * Requires n % 128 == 0 and h % 128 == 0. Padding rows of vs/es/vd are
 * written (zeros / valid metadata). With vs == es == NULL only the dense
 * features are produced (the sparse ones come from the fused epilogues).
 * operand_nonneg = 1 declares the values >= 0 and NaN-free (the relu^2
 * activation): the feature-wise top-2 then ranks raw values (same result,
 * fewer instructions); 0 ranks magnitudes with NaN last (any operand).
 * pair_rows = 2 * n_dense selects the paired layout: no vd; vs rows
 * [0, pair_rows) hold dense feature r as the two fixed-selector 2:4 rows
 * 2r (tokens 4j, 4j+1) and 2r+1 (tokens 4j+2, 4j+3), and the sparse feature
 * of rank s is row pair_rows + s (vs holds pad128(pair_rows + n_sparse) rows).
 * A 2:4 GEMM with the same pair_rows then yields the whole split product.
 * pair_rows = -1: dense features go to vd. */
int s24_feature_split(const void* vals, const uint8_t* meta_hw, int64_t n, int64_t h, const int* feat_pos,
                      int64_t n_sparse, int64_t n_dense, void* vs, uint8_t* es, void* vd,
                      unsigned long long* stats, int operand_nonneg, int64_t pair_rows, void* stream);

/* K4 on the hot path: s24_feature_split in the paired layout (pair_rows =
 * 2 * n_dense), without drop statistics, one warp per 16 features x 128
 * tokens with the per-feature output offsets tabled in shared memory.
 * operand_nonneg = 1 (the relu^2 activation) ranks raw values unless
 * *nan_flag (nullable; K1's stats[2]) is non-zero, in which case values are
 * ranked by magnitude with NaN last, as with operand_nonneg = 0. */
int s24_feature_split_x(const void* vals, const uint8_t* meta_hw, int64_t n, int64_t h, const int* feat_pos,
                        int64_t n_sparse, int64_t n_dense, void* vs, uint8_t* es, int operand_nonneg,
                        const unsigned long long* nan_flag, void* stream);

/* ---------------------------------------------------------------- GEMMs
 * Operand conventions: A is logically [M, K], B is logically [K, N].
 *   a_mn_major = 0: A stored [M][K] (lda >= K);  1: stored [K][M] (lda >= M)
 *   b_mn_major = 0: B stored [N][K] (ldb >= K);  1: stored [K][N] (ldb >= N)
 * D: [M, N] out_dtype with ldd; row m is written to row d_row_map[m] (if non
 * null); d_transposed writes D[n * ldd + row]. Rows >= d_rows_valid are
 * skipped, and so are rows with d_row_valid[m] < 0 (if non null).
 * N % 32 == 0, leading dimensions 16-byte aligned.
 * Replaces gemm / gemm_at (matcore.py:71-106) on tensor cores (fp32 accum). */
int s24_gemm(const void* A, int a_mn_major, int64_t lda, const void* B, int b_mn_major, int64_t ldb, int64_t M,
             int64_t N, int64_t K, void* D, int out_dtype, int64_t ldd, const int* d_row_map, int d_transposed,
             int64_t d_rows_valid, const int* d_row_valid, void* stream);

/* Split-K variant of s24_gemm for thin, long-K products (the dense remainder
 * of the split weight gradient): k_splits partial GEMMs over K ranges write
 * workspace fp32 [k_splits, M, N], then a fixed-order reduction writes D with
 * the same row-map / transpose conventions (deterministic). */
int s24_gemm_splitk(const void* A, int a_mn_major, int64_t lda, const void* B, int b_mn_major, int64_t ldb,
                    int64_t M, int64_t N, int64_t K, int k_splits, float* workspace, void* D, int out_dtype,
                    int64_t ldd, const int* d_row_map, int d_transposed, void* stream);

/* 2:4 sparse A (token-wise along K): a_vals bf16 [M_pad128, K/2] + a_meta hw
 * (rows M_pad128, K). K % 128 == 0. Replaces sp_gemm (sparse24.py:170-192)
 * and, with the feature-wise operand from s24_feature_split, sp_gemm_t
 * (sparse24.py:195-216). pair_rows (even, usually 0): rows below it come in
 * (even, odd) pairs whose sum is written as the even row (row map of the
 * even row) -- the paired dense features of s24_feature_split. */
int s24_spmm(const void* a_vals, const uint8_t* a_meta, const void* B, int b_mn_major, int64_t ldb, int64_t M,
             int64_t N, int64_t K, void* D, int out_dtype, int64_t ldd, const int* d_row_map, int d_transposed,
             int64_t d_rows_valid, const int* d_row_valid, int64_t pair_rows, void* stream);

/* Two s24_spmm problems of identical (M, N, K) and output dtype in ONE
 * persistent launch (group-major work units): the two split weight gradients
 * (dW2 and dW1^T, ffn.py:430-450 via splitgemm.py:55-81) share one tile
 * schedule, so the second fills the first one's partial last wave. Rows are
 * valid up to M; d_row_valid* as in s24_gemm. */
int s24_spmm_pair(int b_mn_major, int64_t M, int64_t N, int64_t K, int out_dtype, const void* a_vals0,
                  const uint8_t* a_meta0, const void* B0, int64_t ldb0, void* D0, int64_t ldd0, const int* d_row_map0,
                  int d_transposed0, const int* d_row_valid0, const void* a_vals1, const uint8_t* a_meta1,
                  const void* B1, int64_t ldb1, void* D1, int64_t ldd1, const int* d_row_map1, int d_transposed1,
                  const int* d_row_valid1, int64_t pair_rows, void* stream);

/* K1: Y1 = X_in . W1 with the fused relu^2 + token-wise 2:4 epilogue
 * (ffn.py:305-329). x: [M, K] row-major; w1: [K, N] row-major (N = h,
 * N % 128 == 0). Outputs act_vals bf16 [M_pad128, N/2], act_meta hw (padding
 * rows up to M_pad128 written as zero groups), counts int32[N] (+=,
 * nullable), stats uint64[3]: [0] += nonzeros before, [1] += nonzeros after
 * the token-wise selection, [2] |= 1 when a kept value is NaN (the caller
 * zeroes it); y_dbg fp32 [M, N] nullable (the pre-activation, for parity
 * checks). Non-finite values follow the reference's numpy semantics: relu
 * keeps NaN (ffn.py:167-169), NaN counts as nonzero (splitgemm.py:28-30) and
 * ranks below zero in the top-2 (sparse24.py:72-77). */
int s24_fwd_gemm1_fused(const void* x, int64_t ldx, const void* w1, int64_t ldw1, int64_t M, int64_t N,
                        int64_t K, void* act_vals, uint8_t* act_meta, int* counts, unsigned long long* stats,
                        float* y_dbg, void* stream);

/* K3: G = dY_c . W2^T with the fused relu^2-derivative + forward-mask
 * epilogue (ffn.py:395-417, 440-443). g: [M, K=d] row-major; w2: [N=h, K=d]
 * row-major. act_vals/act_meta: from K1. Output g_vals bf16 [M_pad128, N/2]
 * on the same metadata (compress_token_wise_with_mask, exact by
 * construction). */
int s24_bwd_dact_fused(const void* g, int64_t ldg, const void* w2, int64_t ldw2, int64_t M, int64_t N,
                       int64_t K, const void* act_vals, const uint8_t* act_meta, void* g_vals, void* stream);

/* dense-mode twins: act = bf16(relu(X W1)^2) [M, N] (w1 stored [K][N]) */
int s24_gemm_relu2(const void* x, int64_t ldx, const void* w1, int64_t ldw1, int64_t M, int64_t N, int64_t K,
                   void* act, int64_t ld_act, void* stream);
/* g_pre = bf16((g . W2^T) * 2 sqrt(act)) [M, N]; w2 stored [N][K] */
int s24_gemm_dact(const void* g, int64_t ldg, const void* w2, int64_t ldw2, int64_t M, int64_t N, int64_t K,
                  const void* act, int64_t ld_act, void* gpre, int64_t ld_g, void* stream);

/* ---------------------------------------------------------------- e4m3 (fp8) path
 * FfnConfig.fp8_emulation / fp8_backward (ref pkg/src/srelu24/ffn.py:206-268,
 * :305, :330-341, :395-447) on the kind::f8f6f4 tensor cores. Quantization
 * follows ref matcore.py:113-261: scale = amax/448 per row or column (1 when
 * amax == 0), codes = e4m3(x / scale), round-to-nearest-even, saturating.
 * "f8 metadata": the e4m3 2:4 operand-E layout, 2048-byte atoms of 128 rows x
 * 128 logical columns with row r's 16 bytes at 16*r (same size as hw). */

/* per-row (rows < pair_rows: per (even, odd) row pair) e4m3 codes + scales of
 * an fp32/bf16 [rows, cols] matrix; amax_in (nullable, float bits) supplies
 * precomputed row maxima; deq_bf16 / raw_bf16 (nullable) receive the bf16
 * dequantized (code * scale) / unquantized images. ref matcore.py:203-225,
 * ffn.py:221-237. */
int s24_fp8_quant_rows(const void* in, int in_dtype, int64_t rows, int64_t cols, int64_t ld_in,
                       const unsigned* amax_in, int64_t pair_rows, uint8_t* codes, int64_t ld_codes, float* scales,
                       void* deq_bf16, int64_t ld_deq, void* raw_bf16, int64_t ld_raw, void* stream);
/* per-column codes of an fp32/bf16 [rows, cols] matrix, written transposed
 * codes_t[cols, rows] (the K-major operand), scales[cols]; amax_ws: cols
 * uint32 of workspace. ref matcore.py:203-225 with axis="cols". */
int s24_fp8_quant_cols_t(const void* in, int in_dtype, int64_t rows, int64_t cols, int64_t ld_in, uint8_t* codes_t,
                         int64_t ld_out, float* scales, unsigned* amax_ws, void* stream);
/* hw metadata -> f8 metadata (same logical content) */
int s24_meta_hw_to_f8(const uint8_t* meta_hw, int64_t rows, int64_t kdim, uint8_t* meta_f8, void* stream);
/* elementwise e4m3 encode of fp32 values (ref matcore.py:155-197) */
int s24_e4m3_encode(const float* x, int64_t n, uint8_t* codes, void* stream);
/* D = (row_scale[i] * col_scale[j]) * sum_k A[i,k] B[j,k] over e4m3 codes
 * (A [M,K], B [N,K], both K-major): ref matcore.py:238-258 */
int s24_gemm_f8(const uint8_t* A, int64_t lda, const uint8_t* B, int64_t ldb, int64_t M, int64_t N, int64_t K,
                const float* row_scale, const float* col_scale, void* D, int out_dtype, int64_t ldd,
                const int* d_row_map, int d_transposed, int64_t d_rows_valid, void* stream);
/* the same with a 2:4 A: codes [Mpad, K/2] + f8 metadata; K % 128 == 0.
 * ref ffn.py:240-255 (_sp_mm / _sp_mm_t) and the split weight gradient. */
int s24_spmm_f8(const uint8_t* a_codes, const uint8_t* a_meta_f8, const uint8_t* B, int64_t ldb, int64_t M,
                int64_t N, int64_t K, const float* row_scale, const float* col_scale, void* D, int out_dtype,
                int64_t ldd, const int* d_row_map, int d_transposed, int64_t d_rows_valid, const int* d_row_valid,
                int64_t pair_rows, void* stream);
/* two s24_spmm_f8 problems of one (M, N, K) in one grouped launch (dW2 and
 * dW1^T of the fp8_backward split weight gradient) */
int s24_spmm_pair_f8(int64_t M, int64_t N, int64_t K, int out_dtype, const uint8_t* a0, const uint8_t* meta0,
                     const uint8_t* B0, int64_t ldb0, const float* rs0, const float* cs0, void* D0, int64_t ldd0,
                     const int* d_row_map0, int d_transposed0, const int* d_row_valid0, const uint8_t* a1,
                     const uint8_t* meta1, const uint8_t* B1, int64_t ldb1, const float* rs1, const float* cs1,
                     void* D1, int64_t ldd1, const int* d_row_map1, int d_transposed1, const int* d_row_valid1,
                     int64_t pair_rows, void* stream);
/* K1 on e4m3 operands (W1 codes as [N, K]): y = (sx * s1) * acc, then as
 * s24_fwd_gemm1_fused but the kept values go out fp32 [Mpad, N/2] with the
 * per-row max kept value in row_amax (float bits, zeroed by the caller) */
int s24_fwd_gemm1_f8(const uint8_t* xq, int64_t ldx, const uint8_t* w1q, int64_t ldw1, int64_t M, int64_t N,
                     int64_t K, const float* x_scale, const float* w1_scale, float* act_vals32, unsigned* row_amax,
                     uint8_t* act_meta, int* counts, unsigned long long* stats, float* y_dbg, void* stream);
/* K3 on e4m3 operands (W2 codes as [N=h, K=d]): G = (sg * s2) * acc, then as
 * s24_bwd_dact_fused */
int s24_bwd_dact_f8(const uint8_t* gq, int64_t ldg, const uint8_t* w2q, int64_t ldw2, int64_t M, int64_t N,
                    int64_t K, const float* g_scale, const float* w2_scale, const void* act_vals,
                    const uint8_t* act_meta, void* g_vals, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* S24_H_ */

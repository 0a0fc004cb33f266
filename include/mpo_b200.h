/*
 * mpo_b200.h -- C ABI of the B200-native TNrSVD / sparse->MPO hot path.
 *
 * The reference (arXiv 1707.07803's Python package `mposvd`) has no FFI;
 * its boundary is the Python API re-exported by
 * /root/reference/pkg/src/mposvd/__init__.py:3-50.  Each entry point below
 * is what a ctypes/cffi binding of that API binds to,
 * and cites the reference function it replaces.
 *
 * Conventions
 *  - Plain pointers and sizes only.  `from_host` / `to_host` select whether
 *    a buffer is host memory (copied with cudaMemcpyAsync) or a device
 *    pointer (e.g. a torch CUDA tensor's data_ptr).
 *  - Cores are FP64, F-ordered (first index fastest), shape (R, I, J, S),
 *    exactly the serialized layout of mpo.py:17-23.
 *  - Optional rounding tolerances are passed as (round_tol, has_tol);
 *    has_tol == 0 is the reference's `round_tol=None`.
 *  - Every call returns MPO_OK or an error code; mpo_b200_last_error()
 *    returns the message (thread-local).  MPO_EVALUE maps to the
 *    reference's ValueError, MPO_ENOMEM to MemoryError, MPO_ECUDA to
 *    RuntimeError.
 *  - Handles (mpo_ctx, mpo_dev, mpo_conv) own device memory allocated
 *    stream-ordered on the context's stream.  No global state beyond the
 *    launch counter; calls on different contexts are independent.
 */
#ifndef MPO_B200_H
#define MPO_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { MPO_OK = 0, MPO_EVALUE = 1, MPO_ECUDA = 2, MPO_ENOMEM = 3, MPO_EINTERNAL = 4 };

typedef struct mpo_ctx mpo_ctx;   /* device + stream */
typedef struct mpo_dev mpo_dev;   /* device-resident MPO (mpo.py:119 `Mpo`) */
typedef struct mpo_conv mpo_conv; /* conversion structure (sparse.py:207 result) */

/* ---- library / context ------------------------------------------------ */
const char* mpo_b200_last_error(void);
int mpo_b200_abi_version(void);
unsigned long long mpo_b200_launch_count(void); /* kernels launched so far */
/* how the truncating R2L steps were rounded so far (out[5]): certificate
 * wide / tall, tail cut wide / tall, full SVD */
int mpo_b200_round_paths(unsigned long long* out);
/* CUDA-event timing per kernel family (bench roofline): which = 0
 * jacobi_gram, 1 jacobi_eig, 2 jacobi_apply, 3 dgemm (incl. split-K
 * reduction), 4 QR panel, 5 QR panel-reflector application (in-block and
 * look-ahead updates); enable(1) resets.  Timed launches synchronise
 * (profiling runs only). */
int mpo_b200_profile_enable(int on);
int mpo_b200_profile_read(int which, double* ms, double* flops, unsigned long long* launches);

int mpo_ctx_create(int device, void* cuda_stream, mpo_ctx** out);
int mpo_ctx_set_stream(mpo_ctx* ctx, void* cuda_stream);
int mpo_ctx_synchronize(mpo_ctx* ctx);
int mpo_ctx_destroy(mpo_ctx* ctx);

/* ---- MPO handles (mpo.py:119-204 `Mpo`) ------------------------------- */
/* shapes: 4*d int64 (R, I, J, S per core); cores[k]: F-ordered FP64 data.
 * Validates like Mpo.__init__ (mpo.py:124-145). */
int mpo_dev_create(mpo_ctx* ctx, int d, const int64_t* shapes, const double* const* cores,
                   int from_host, mpo_dev** out);
/* the same from ONE packed buffer of F-ordered cores back to back (one H2D) */
int mpo_dev_create_packed(mpo_ctx* ctx, int d, const int64_t* shapes, const double* packed,
                          int from_host, mpo_dev** out);
/* every core into ONE packed buffer, F-ordered cores back to back (one D2H) */
int mpo_dev_copy_all(mpo_ctx* ctx, const mpo_dev* m, double* dst, int to_host);
int mpo_dev_num_cores(const mpo_dev* m, int* d);
int mpo_dev_shapes(const mpo_dev* m, int64_t* shapes /* 4*d */);
int mpo_dev_core_ptr(const mpo_dev* m, int k, const double** dev_ptr);
int mpo_dev_copy_core(mpo_ctx* ctx, const mpo_dev* m, int k, double* dst, int to_host);
int mpo_dev_free(mpo_dev* m);

/* ---- TNrSVD stages (rsvd.py) ------------------------------------------ */
/* rsvd.py:62-79 mpo_matmul; trans_* apply mpo_transpose (mpo.py:402) to the
 * operand without a copy. */
int mpo_matmul(mpo_ctx* ctx, const mpo_dev* a, int trans_a, const mpo_dev* b, int trans_b,
               mpo_dev** out);
/* mpo.py:402-410 mpo_transpose */
int mpo_transpose(mpo_ctx* ctx, const mpo_dev* a, mpo_dev** out);
/* rsvd.py:82-99 merge_leading_cores (count == 1 returns a copy) */
int mpo_merge_leading_cores(mpo_ctx* ctx, const mpo_dev* m, int count, mpo_dev** out);
/* rsvd.py:139-166 mpo_qr: Q handle + K x K factor R (column-major, host) */
int mpo_qr(mpo_ctx* ctx, const mpo_dev* y, double round_tol, int has_tol, mpo_dev** q,
           double* r_host);
/* rsvd.py:169-193 mpo_svd: W (K x K, column-major, host), s (K, host), tall V */
int mpo_svd(mpo_ctx* ctx, const mpo_dev* b, double round_tol, int has_tol, double* w_host,
            double* s_host, mpo_dev** v);
/* rsvd.py:196-214 subspace_iteration */
int mpo_subspace_iteration(mpo_ctx* ctx, const mpo_dev* a, const mpo_dev* o, int q,
                           double round_tol, int has_tol, mpo_dev** out);
/* rsvd.py:217-259 tnrsvd on an already merged operator `am` (rsvd.py:243)
 * with the caller's unit-rank sketch `o` (mpo.py:413-433; K = o's first
 * core column extent).  Writes the k_target leading singular values to
 * s_host and returns U and V (first cores carry the k_target column index,
 * sign convention of rsvd.py:251-255). */
int mpo_tnrsvd(mpo_ctx* ctx, const mpo_dev* am, const mpo_dev* o, int k_target, int q,
               double round_tol, int has_tol, mpo_dev** u, double* s_host, mpo_dev** v);

/* mpo.py:323-354 mpo_round (L2R QR sweep + R2L truncated-SVD sweep) */
int mpo_round(mpo_ctx* ctx, const mpo_dev* m, double rel_tol, mpo_dev** out);
/* mpo.py:264-294 mpo_add (block-diagonal core stacking) */
int mpo_add(mpo_ctx* ctx, const mpo_dev* a, const mpo_dev* b, mpo_dev** out);

/* ---- sparse -> MPO conversion (sparse.py:207-258, uncapped path) ------- */
/* row1/col1: 1-based int64 coordinates, val: FP64, n entries (explicit zeros
 * are dropped, sparse.py:234); factors: the PartitionPlan (partition.py:40). */
/* from_host = 0: row1/col1/val are device arrays that must stay valid until
 * mpo_conv_free (without explicit zeros the entry arrays i1, j1, values are
 * derived from them on demand); from_host = 1: host arrays, uploaded and
 * kept by the handle. */
int mpo_sparse_convert(mpo_ctx* ctx, const int64_t* row1, const int64_t* col1,
                       const double* val, int64_t n, int from_host, int d,
                       const int64_t* row_factors, const int64_t* col_factors, mpo_conv** out);
int mpo_conv_info(const mpo_conv* c, int64_t* nkept, int64_t* rank);
/* any output pointer may be NULL; sizes nkept (i1, j1, ti, values) and rank (uniq) */
int mpo_conv_copy(mpo_ctx* ctx, const mpo_conv* c, int64_t* i1, int64_t* j1, int64_t* ti,
                  double* values, int64_t* uniq, int to_host);
/* device pointers of the handle's arrays (owned by the handle, valid until
 * mpo_conv_free; any output may be NULL).  Requesting i1, j1 or values
 * materialises them if they were left derivable (no explicit zeros). */
int mpo_conv_ptrs(mpo_ctx* ctx, const mpo_conv* c, int64_t** i1, int64_t** j1, int64_t** ti,
                  double** values, int64_t** uniq);
/* block digits of core `level` (1..d-1), level-2 fastest (sparse.py:173-180, :249-250) */
int mpo_conv_level(mpo_ctx* ctx, const mpo_conv* c, int level, int64_t* row_digits,
                   int64_t* col_digits, int to_host);
/* dense core `level` (0..d-1) of the summed unit-rank terms (sparse.py:183-204
 * densified as Mpo.densify, mpo.py:184-197) */
int mpo_conv_dense_core(mpo_ctx* ctx, const mpo_conv* c, int level, double* dst, int to_host);
/* device MPO of the unit-rank terms of blocks [start, stop), dense cores
 * (one chunk of the capped accumulation, sparse.py:260-271) */
int mpo_conv_chunk(mpo_ctx* ctx, const mpo_conv* c, int64_t start, int64_t stop,
                   mpo_dev** out);
int mpo_conv_free(mpo_conv* c);

/* ---- multi-GPU conversion merge helpers (no reference counterpart: the
 *      exchange step of the nnz-sharded conversion) ------ */
/* sorted unique of n int64 keys in [0, max_key] (device in/out); *nuniq set */
int mpo_keys_unique(mpo_ctx* ctx, const int64_t* keys, int64_t n, int64_t max_key,
                    int64_t* uniq_out, int64_t* nuniq);
/* out[i] = index of q[i] in the sorted table (binary search; -1 if absent) */
int mpo_keys_lookup(mpo_ctx* ctx, const int64_t* table, int64_t ntab, const int64_t* q,
                    int64_t nq, int64_t* out);
/* out[i] = offset + lower_bound(table, q[i]) over the sorted table; with
 * exact != 0, -1 where q[i] is absent (device in/out).  Splitter positions
 * and range-local -> global block ids of the key-range exchange. */
int mpo_keys_search(mpo_ctx* ctx, const int64_t* table, int64_t ntab, const int64_t* q,
                    int64_t nq, int64_t offset, int exact, int64_t* out);
/* ti[i] = map[ti[i]] in place (device) */
int mpo_remap_ids(mpo_ctx* ctx, const int64_t* map, int64_t* ti, int64_t n);

/* ---- dense factorisations of device matrices (column-major) -----------
 * The local steps of the row-distributed TSQR / SVD of one tall unfolding
 * (paper_1707_07803_b200/distributed.py tsqr, tsqr_svd), replacing the
 * per-core np.linalg.qr at rsvd.py:106 and np.linalg.svd at rsvd.py:128 when
 * the unfolding's rows are sharded over GPUs. */
/* reduced QR A = Q R (m >= n; Householder, dgeqrf + dorgqr) */
int mpo_dense_qr(mpo_ctx* ctx, int64_t m, int64_t n, const double* a, int64_t lda, double* q,
                 int64_t ldq, double* r, int64_t ldr);
/* thin SVD A = U diag(s) Vt (m >= n; s descending, U orthonormal columns) */
int mpo_dense_svd(mpo_ctx* ctx, int64_t m, int64_t n, const double* a, int64_t lda, double* s,
                  double* u, int64_t ldu, double* vt, int64_t ldvt);
/* C = alpha op(A) op(B) + beta C (DMMA GEMM) */
int mpo_dense_gemm(mpo_ctx* ctx, int ta, int tb, int64_t m, int64_t n, int64_t k, double alpha,
                   const double* a, int64_t lda, const double* b, int64_t ldb, double beta,
                   double* c, int64_t ldc);

#ifdef __cplusplus
}
#endif

#endif /* MPO_B200_H */

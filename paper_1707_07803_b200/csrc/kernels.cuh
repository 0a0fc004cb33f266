// Host-side launchers of the sm_100a kernels (all stream-ordered, FP64,
// column-major).  Each launcher documents the reference operation it
// replaces.
#pragma once

#include "common.cuh"

namespace mpob {

// Optional per-kernel CUDA-event timing (bench.py's roofline): 0 =
// jacobi_gram, 1 = jacobi_eig, 2 = jacobi_apply, 3 = dgemm (+ its split-K
// reduction), 4 = QR panel, 5 = QR panel-reflector application (in-block /
// look-ahead update).  Each timed launch synchronises its stream (profiling
// runs only).
struct KernelProfile {
  static constexpr int N = 6;
  bool on = false;
  double ms[N] = {};
  double flops[N] = {};
  unsigned long long launches[N] = {};
  void add(int k, double t, double f) { ms[k] += t; flops[k] += f; launches[k] += 1; }
  void reset() { for (int k = 0; k < N; ++k) { ms[k] = 0; flops[k] = 0; launches[k] = 0; } }
};
// events around one launch on st when profiling (ProfScope p(st, 3, flops))
struct ProfScope {
  cudaStream_t st;
  int which;
  double flops;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  ProfScope(cudaStream_t s, int w, double f);
  ~ProfScope();
};
extern KernelProfile g_prof;

__host__ __device__ inline int64_t cdiv_dev(int64_t a, int64_t b) { return (a + b - 1) / b; }

// ---- dense building blocks (gemm.cu, core_ops.cu) -------------------------
void dgemm(cudaStream_t st, bool ta, bool tb, int64_t m, int64_t n, int64_t k, double alpha,
           const double* A, int64_t lda, const double* B, int64_t ldb, double beta, double* C,
           int64_t ldc, int64_t batch = 1, int64_t sA = 0, int64_t sB = 0, int64_t sC = 0);
void scale_matrix(cudaStream_t st, int64_t m, int64_t n, double alpha, double* C, int64_t ldc,
                  int64_t batch = 1, int64_t sC = 0);
void copy_matrix(cudaStream_t st, int64_t m, int64_t n, const double* A, int64_t lda, double* B,
                 int64_t ldb);
void set_identity(cudaStream_t st, int64_t m, int64_t n, double* A, int64_t lda);
void fill_zero(cudaStream_t st, double* p, int64_t n);
// out = in.transpose(perm) for F-ordered arrays of rank <= 6.
void permute(cudaStream_t st, const double* in, double* out, int rank, const int64_t* dims,
             const int* perm);
// Frobenius norm (deterministic two-level reduction) -> device scalar.
void frob_norm(cudaStream_t st, const double* x, int64_t n, double* out_dev);

// Per-core MPO product (rsvd.py:62-79):
//   N[a + Ra*c, i, k, b + Sa*d] = sum_j A[a,i,j,b] * B[c,j,k,d]
// Operands may be logically transposed (swap of axes 1 and 2,
// mpo.py:402-410) without a copy.
struct CoreView {
  const double* p;
  int64_t R, I, J, S;  // logical extents
  bool trans;          // physical storage is (R, J, I, S)
};
void core_product(cudaStream_t st, const CoreView& a, const CoreView& b, double* out);

// Householder QR of a column-major m x n matrix (qr.cu): on return A holds
// R in its upper triangle (k = min(m, n) rows) and Q (m x k) is written
// explicitly; replaces np.linalg.qr(mode="reduced") (LAPACK dgeqrf+dorgqr).
// defer_q: the explicit Q (dorgqr) is formed on a separate stream after the
// factorisation, overlapping whatever the caller issues next on st (R is
// ready in stream order as usual); the caller must join_deferred_q(st) before
// anything on st reads or frees Q.
void householder_qr(cudaStream_t st, int64_t m, int64_t n, double* A, int64_t lda, double* Q,
                    int64_t ldq, double* R, int64_t ldr, bool defer_q = false);
void join_deferred_q(cudaStream_t st);
// joins on scope exit (also when an exception unwinds past pending Q's)
struct DeferredQScope {
  cudaStream_t st;
  explicit DeferredQScope(cudaStream_t s) : st(s) {}
  ~DeferredQScope() { join_deferred_q(st); }
};
// The same factorisation keeping the compact-WY reflectors (no explicit Q),
// and C <- Q C for an m x ncols matrix C (qr.cu).
struct QrReflectors {
  static constexpr int NBO = 128;   // outer block width
  int64_t m = 0, k = 0;
  std::vector<int64_t> voff, wos;
  DBuf<double> V, T;
};
void householder_qr_keep(cudaStream_t st, int64_t m, int64_t n, double* A, int64_t lda,
                         double* R, int64_t ldr, QrReflectors& f);
void qr_apply_q(cudaStream_t st, const QrReflectors& f, double* C, int64_t ldc, int64_t ncols);
// X <- X Q for the nrows x m matrix X (rank-k update per outer block)
void qr_apply_q_right(cudaStream_t st, const QrReflectors& f, double* X, int64_t ldx, int64_t nrows);

// Thin SVD of a column-major m x n matrix (svd.cu).  Returns all min(m,n)
// singular values (descending, on the device) and the column-sorted
// factors:  M = Ucarry * Vh  where Ucarry = U * diag(s) (m x k) and
// Vh (k x n) has orthonormal rows.  Replaces np.linalg.svd(full_matrices=
// False) (LAPACK dgesdd) at rsvd.py:128 and :189.
struct SvdOut {
  DBuf<double> s;       // k
  DBuf<double> ucarry;  // m x k, column-major, ld = m  (U * diag(s))
  DBuf<double> vh;      // k x n, column-major, ld = k
  int64_t k = 0;
};
// trunc_rel > 0 (truncation SVDs): the caller's truncation level delta
// relative to ||M||_F.  Rotations whose coupling is below a noise floor of
// min(64 eps, 1e-2 trunc_rel) ||M||_F are skipped (singular values and the
// exact product U S Vh are unaffected; U = ucarry / s is then not
// orthonormal for noise-level s, so callers that need left vectors pass 0),
// and the sweeps may stop early once the couplings are O(1e-4) -- only
// while the floor sits >= 100x below delta.  0: full convergence.
void svd_thin(cudaStream_t st, int64_t m, int64_t n, const double* M, int64_t ldm, SvdOut& out,
              double trunc_rel = 0.0);
// One-CTA variants for matrices that fit shared memory (small.cu); false:
// not applicable (the blocked paths above take it).
bool small_qr(cudaStream_t st, int64_t m, int64_t n, const double* A, int64_t lda, double* Q,
              int64_t ldq, double* R, int64_t ldr);
bool small_svd(cudaStream_t st, int64_t m, int64_t n, const double* M, int64_t ldm, SvdOut& out,
               double trunc_rel);
// Inverse of a k x k upper-triangular matrix, and the certified lower
// bound 1 / ||U^{-1}||_F <= sigma_min(U) (rankcert.cu).
void tri_inv_upper(cudaStream_t st, int64_t k, const double* U, int64_t ldu, double* Out);
// inv_out (k x k, optional) receives U^{-1}.
double min_sv_lower_bound(cudaStream_t st, int64_t k, const double* U, int64_t ldu,
                          double target, double* inv_out = nullptr);
// Tail truncation of M = R'^T Q'^T (right: M = Q R') at level delta from R'
// (k x k upper triangular) and inv = R'^{-1} (rankcert.cu): t = the number
// of singular values _truncation_rank discards and C (k x (k - t)) an
// orthonormal basis of the complement of their left (right: right)
// singular vectors of R'.  false: not resolved inside the iterated block
// (the caller takes the full SVD).
// With build_c = false (and t > 0) C is not formed: H = the reflectors f of
// U_t, C = H [0; I_{k-t}], so X C = (X H)[:, t:] is a rank-t update of X.
struct TailCut {
  int64_t t = 0;
  DBuf<double> C;
  QrReflectors f;
  bool has_c = false;
};
bool tail_cut(cudaStream_t st, int64_t k, const double* Rt, int64_t ldr, const double* inv,
              double delta, bool right, TailCut& out, bool build_c = true);

}  // namespace mpob

namespace mpob {
// W = Ucarry diag(1/s), completed to orthonormal where s == 0 (k x k).
void svd_left_vectors(cudaStream_t st, int64_t k, const double* ucarry, int64_t ldu,
                      const double* s, double* W);
// y += alpha * x (n elements)
void dgemm_axpy(cudaStream_t st, int64_t n, double alpha, const double* x, double* y);
// out[(a + ra) + Ro*(m + M*(b + sb))] = in[a + Ri*(m + M*b)]  (mpo_add stacking)
void place_block(cudaStream_t st, const double* in, int64_t Ri, int64_t M, int64_t Si, double* out,
                 int64_t Ro, int64_t So, int64_t ra, int64_t sb);
// out[i, l, r] = in[i, l, r] * sign[l] for l < kt (tnrsvd finishing, rsvd.py:251-257)
void core0_finish(cudaStream_t st, const double* in, int64_t I1, int64_t K, int64_t R2,
                  int64_t kt, const double* sign_dev, double* out);

// A second (non-blocking) stream and eight events, created once per (host
// thread, main stream): lets one library call overlap independent work.
// Events 0-3 belong to the Jacobi sweeps (svd.cu), 4-7 to the QR (qr.cu).
struct SideStream {
  cudaStream_t main = nullptr, sv = nullptr;
  int device = -1;
  cudaStream_t hp = nullptr;   // highest-priority stream (latency-critical chains)
  cudaStream_t aux = nullptr;  // highest-priority helper (QR: compact-WY T assembly)
  cudaStream_t qs = nullptr;   // deferred explicit-Q formation (householder_qr defer_q)
  cudaEvent_t eqf = nullptr, eq = nullptr;   // factorisation done / Q formed
  bool q_pending = false;
  cudaEvent_t e[8] = {};
};
SideStream& side_stream(cudaStream_t main);
}  // namespace mpob

// Rank certificate for the truncation sweeps (rsvd.py:124-136 ->
// _truncation_rank, mpo.py:297-304).
//
// A truncating R2L step SVDs the unfolding M (R x N) of core k only to pick
// the smallest rank r whose discarded tail sum of squared singular values
// stays within delta^2.  When every singular value exceeds delta, that rank
// is min(R, N) = R (nothing is discarded) and any factorisation
// M = L Q with orthonormal rows Q represents the same tensor: the SVD
// (one-sided Jacobi, the dominant cost of config 2) is then unnecessary.
//
// The certificate: with M^T = Q' R' (the LQ of M, Householder), sigma_min(M)
// = sigma_min(R') >= 1 / ||R'^{-1}||_F.  The inverse of the R x R upper
// triangular R' is formed blockwise (32 x 32 diagonal blocks by back
// substitution, merged bottom-up with two DMMA GEMMs per pair of blocks,
// ~R^3/3 flops) and its Frobenius norm taken on the device.  A bound above
// a safety margin times delta proves the reference's rank (its dgesdd
// singular values are accurate to O(eps ||M||) << delta); anything else --
// including an ill-conditioned or singular R' (overflow, NaN) -- takes the
// SVD.  The represented tensor, and with it every later singular value and
// rank decision, is the same either way (the next core's unfolding changes
// by an orthogonal factor only).
#include <cmath>

#include "common.cuh"
#include "kernels.cuh"

namespace mpob {

namespace {

constexpr int TB = 32;

// Out[diagonal block b] = inverse of U's upper-triangular diagonal block b
// (back substitution, one thread per column of the inverse)
__global__ void __launch_bounds__(TB) diag_block_inv(const double* __restrict__ U, int64_t ldu,
                                                     int64_t k, double* __restrict__ Out,
                                                     int64_t ldo) {
  __shared__ double S[TB][TB + 1];
  __shared__ double X[TB][TB + 1];
  const int64_t o = (int64_t)blockIdx.x * TB;
  const int n = (int)min((int64_t)TB, k - o);
  const int t = threadIdx.x;
  for (int c = 0; c < n; ++c) {
    S[t][c] = t < n ? U[(o + t) + (o + c) * ldu] : 0.0;
    X[t][c] = 0.0;
  }
  __syncthreads();
  if (t < n) {
    const int j = t;   // column j of the inverse: S x = e_j, x_i = 0 for i > j
    for (int i = j; i >= 0; --i) {
      double acc = (i == j) ? 1.0 : 0.0;
      for (int l = i + 1; l <= j; ++l) acc -= S[i][l] * X[l][j];
      X[i][j] = acc / S[i][i];
    }
  }
  __syncthreads();
  for (int c = 0; c < n; ++c)
    if (t < n) Out[(o + t) + (o + c) * ldo] = X[t][c];
}

}  // namespace

// Inverse of the k x k upper-triangular U (ld ldu) into Out (k x k, ld k).
void tri_inv_upper(cudaStream_t st, int64_t k, const double* U, int64_t ldu, double* Out) {
  fill_zero(st, Out, k * k);
  const int nb = (int)cdiv(k, TB);
  diag_block_inv<<<nb, TB, 0, st>>>(U, ldu, k, Out, k);
  CK_LAUNCH();
  note_launch();
  DBuf<double> tmp((size_t)k * k, st);
  // bottom-up: [[A, B], [0, D]]^{-1} = [[A^{-1}, -A^{-1} B D^{-1}], [0, D^{-1}]]
  for (int64_t s = TB; s < k; s *= 2) {
    for (int64_t i = 0; i + s < k; i += 2 * s) {
      const int64_t n1 = s, n2 = std::min(s, k - i - s);
      // tmp = B D^{-1}  (n1 x n2)
      dgemm(st, false, false, n1, n2, n2, 1.0, U + i + (i + s) * ldu, ldu,
            Out + (i + s) + (i + s) * k, k, 0.0, tmp.get(), n1);
      // top-right = -A^{-1} tmp
      dgemm(st, false, false, n1, n2, n1, -1.0, Out + i + i * k, k, tmp.get(), n1, 0.0,
            Out + i + (i + s) * k, k);
    }
  }
}

static double host_frob(cudaStream_t st, const double* x, int64_t n, double* scratch) {
  frob_norm(st, x, n, scratch);
  double h = 0.0;
  CK(cudaMemcpyAsync(&h, scratch, sizeof(double), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return h;
}

// A certified lower bound on sigma_min(U), U k x k upper triangular (host
// value).  X = U^{-1}, sigma_min(U) = 1 / ||X||_2.
//   b1 = 1 / ||X||_F                       (within sqrt(k) of sigma_min)
// and, when b1 does not reach `target` (k >= 256), the tighter
//   b2 = 1 / sqrt(||G^8||_F^{1/8}),  G = X^T X      (within k^{1/32}),
// since lambda_max(G) <= ||G^m||_F^{1/m} <= k^{1/(2m)} lambda_max(G); G^8 by
// three squarings, each normalised by its Frobenius norm (the norms are
// carried as logarithms).  0 when U is singular or a norm overflows: the
// caller then factors by SVD.
double min_sv_lower_bound(cudaStream_t st, int64_t k, const double* U, int64_t ldu,
                          double target) {
  DBuf<double> inv((size_t)k * k, st), nrm(1, st);
  tri_inv_upper(st, k, U, ldu, inv.get());
  const double h = host_frob(st, inv.get(), k * k, nrm.get());
  if (!(h > 0.0) || !std::isfinite(h)) return 0.0;
  const double b1 = 1.0 / h;
  if (b1 > target || k < 256) return b1;
  DBuf<double> G((size_t)k * k, st), H((size_t)k * k, st);
  dgemm(st, true, false, k, k, k, 1.0, inv.get(), k, inv.get(), k, 0.0, G.get(), k);
  double logl = 0.0;   // log ||G^8||_F^{1/8} accumulated as sum of w_j log f_j
  double w = 1.0;
  double* a = G.get();
  double* b = H.get();
  for (int j = 0; j < 4; ++j) {
    const double f = host_frob(st, a, k * k, nrm.get());
    if (!(f > 0.0) || !std::isfinite(f)) return b1;
    logl += w * std::log(f);
    if (j == 3) break;
    scale_matrix(st, k, k, 1.0 / f, a, k);
    dgemm(st, false, false, k, k, k, 1.0, a, k, a, k, 0.0, b, k);
    std::swap(a, b);
    w *= 0.5;
  }
  const double b2 = std::exp(-0.5 * logl);   // 1 / sqrt(lambda bound)
  return std::max(b1, b2);
}

}  // namespace mpob

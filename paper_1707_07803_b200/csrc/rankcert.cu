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
#include <cstdio>
#include <cstdlib>
#include <vector>

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

// A[i, j] = A[j, i] for i > j (k x k, ld k): 32 x 32 tiles through shared memory
__global__ void __launch_bounds__(256) mirror_upper_kernel(int64_t k, double* __restrict__ A) {
  __shared__ double tile[32][33];
  const int64_t bi = blockIdx.y, bj = blockIdx.x;   // lower tile (bi, bj), bi >= bj
  if (bi < bj) return;
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;
  for (int r = ty; r < 32; r += 8) {
    const int64_t sr = bj * 32 + r, sc = bi * 32 + tx;   // source: upper tile (bj, bi)
    tile[r][tx] = (sr < k && sc < k) ? A[sr + sc * k] : 0.0;
  }
  __syncthreads();
  for (int r = ty; r < 32; r += 8) {
    const int64_t di = bi * 32 + tx, dj = bj * 32 + r;   // A[di, dj] = A[dj, di]
    if (di < k && dj < k && di > dj) A[di + dj * k] = tile[r][tx];
  }
}

// Out = X^T X (k x k, ld k) for a symmetric X (then Out = X^2) or an upper
// triangular X (tri): only the block rows' upper parts are multiplied
// (56 % of the flops of the full product for symmetric X, 17 % for
// triangular X at 8 block rows), the lower triangle is mirrored
void sym_gram(cudaStream_t st, int64_t k, const double* X, double* Out, bool tri) {
  const int64_t nb = 512;
  for (int64_t i0 = 0; i0 < k; i0 += nb) {
    const int64_t mi = std::min(nb, k - i0), n = k - i0, kd = tri ? i0 + mi : k;
    dgemm(st, true, false, mi, n, kd, 1.0, X + i0 * k, k, X + i0 * k, k, 0.0, Out + i0 + i0 * k, k);
  }
  const unsigned nt = (unsigned)cdiv(k, 32);
  mirror_upper_kernel<<<dim3(nt, nt), 256, 0, st>>>(k, Out);
  CK_LAUNCH();
  note_launch();
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
  // bottom-up: [[A, B], [0, D]]^{-1} = [[A^{-1}, -A^{-1} B D^{-1}], [0, D^{-1}]];
  // the full-size pairs of one level are one strided-batched GEMM each
  // (diagonal blocks at stride 2s (ld + 1)), a trailing partial pair alone
  for (int64_t s = TB; s < k; s *= 2) {
    const int64_t full = k / (2 * s);   // pairs with n2 == s
    if (full > 0) {
      const int64_t su = 2 * s * (ldu + 1), so = 2 * s * (k + 1), stp = s * s;
      dgemm(st, false, false, s, s, s, 1.0, U + s * ldu, ldu, Out + s + s * k, k, 0.0, tmp.get(),
            s, full, su, so, stp);
      dgemm(st, false, false, s, s, s, -1.0, Out, k, tmp.get(), s, 0.0, Out + s * k, k, full, so,
            stp, so);
    }
    const int64_t i = full * 2 * s;
    if (i + s < k) {
      const int64_t n1 = s, n2 = k - i - s;
      dgemm(st, false, false, n1, n2, n2, 1.0, U + i + (i + s) * ldu, ldu,
            Out + (i + s) + (i + s) * k, k, 0.0, tmp.get(), n1);
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
                          double target, double* inv_out) {
  DBuf<double> inv_own, nrm(1, st);
  double* inv = inv_out;
  if (!inv) {
    inv_own.alloc((size_t)k * k, st);
    inv = inv_own.get();
  }
  tri_inv_upper(st, k, U, ldu, inv);
  const double h = host_frob(st, inv, k * k, nrm.get());
  if (!(h > 0.0) || !std::isfinite(h)) return 0.0;
  const double b1 = 1.0 / h;
  // sigma_min <= sqrt(k) b1: a target above that cannot be certified (the
  // caller goes straight to the tail truncation)
  if (b1 > target || k < 256 || std::sqrt((double)k) * b1 <= target) return b1;
  DBuf<double> G((size_t)k * k, st), H((size_t)k * k, st);
  sym_gram(st, k, inv, G.get(), /*tri=*/true);
  // lambda_max(G) <= ||G^m||_F^{1/m} <= k^{1/(2m)} lambda_max(G): squarings
  // (each normalised by its Frobenius norm, the norms kept as logarithms)
  // until the bound passes or m = 8
  double logl = 0.0;   // log ||G^m||_F^{1/m}
  double w = 1.0;
  double* a = G.get();
  double* b = H.get();
  double best = b1;
  for (int j = 0; j < 4; ++j) {
    const double f = host_frob(st, a, k * k, nrm.get());
    if (!(f > 0.0) || !std::isfinite(f)) return best;
    logl += w * std::log(f);
    best = std::max(best, std::exp(-0.5 * logl));
    if (best > target || j == 3) break;
    scale_matrix(st, k, k, 1.0 / f, a, k);
    sym_gram(st, k, a, b, /*tri=*/false);
    std::swap(a, b);
    w *= 0.5;
  }
  return best;
}


// ---------------------------------------------------------------------------
// Tail truncation: when the certificate fails, only the singular values
// below (or near) delta decide _truncation_rank (mpo.py:297-304), and only
// their directions are discarded.  With M = R'^T Q'^T (the LQ above) the
// discarded right directions of M are Q' U_t, U_t the left singular vectors
// of R' for its smallest singular values, and the rounded unfolding is
//     M_r = M (I - V_t V_t^T) = (R'^T C)(Q' C)^T,   C C^T = I - U_t U_t^T,
// the same tensor as the reference's U_r S_r Vh_r in another gauge (every
// later singular value and rank is unchanged, as for the certificate).
//
// U_t and the smallest singular values come from subspace iteration with
// (R' R'^T)^{-1} = inv^T inv on a block of p vectors (two DMMA GEMMs + a
// QR per step) and Rayleigh-Ritz (QR of R'^T X, SVD of its p x p factor).
// The cut is taken from the Ritz values exactly as _truncation_rank takes
// it from the full spectrum (tail sums from the smallest value up) once it
// lies inside the block with a margin and the block has converged: the
// angle of the discarded directions shrinks by (a_t / a_p)^2 per step, so
// the discarded set is resolved to rounding (the same accuracy class as
// the reference's dgesdd subspace).  Anything else returns false and the
// caller takes the full SVD.

__device__ __forceinline__ uint64_t splitmix(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

// deterministic N(0,1) start block (Box-Muller on a counter hash)
__global__ void hash_normal_kernel(double* x, int64_t n, uint64_t seed) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t a = splitmix(seed ^ (2 * (uint64_t)i)), b = splitmix(seed ^ (2 * (uint64_t)i + 1));
    const double u1 = ((a >> 11) + 1) * (1.0 / 9007199254740993.0);
    const double u2 = (b >> 11) * (1.0 / 9007199254740992.0);
    x[i] = sqrt(-2.0 * log(u1)) * cospi(2.0 * u2);
  }
}

bool tail_cut(cudaStream_t st, int64_t k, const double* Rt, int64_t ldr, const double* inv,
              double delta, bool right, TailCut& out, bool build_c) {
  static const bool trace = std::getenv("MPO_B200_TRACE") != nullptr;
  for (int64_t p : {(int64_t)64, (int64_t)256}) {
    if (2 * p > k) break;
    DBuf<double> X((size_t)k * p, st), Y((size_t)k * p, st), Rx((size_t)p * p, st);
    {
      const int grid = (int)std::min<int64_t>(cdiv(k * p, 256), 1024);
      hash_normal_kernel<<<grid, 256, 0, st>>>(X.get(), k * p, 0x5eed0000ull + (uint64_t)k);
      CK_LAUNCH();
      note_launch();
    }
    std::vector<double> a(p), prev;
    SvdOut rr;
    int64_t t = -1;
    bool ok = false;
    const int maxit = p <= 64 ? 8 : 10;
    for (int it = 0; it < maxit && !ok; ++it) {
      // X <- orth((R' R'^T)^{-1} X) = orth(inv^T inv X)  (right: (R'^T R')^{-1} = inv inv^T)
      dgemm(st, right, false, k, p, k, 1.0, inv, k, X.get(), k, 0.0, Y.get(), k);
      dgemm(st, !right, false, k, p, k, 1.0, inv, k, Y.get(), k, 0.0, X.get(), k);
      householder_qr(st, k, p, X.get(), k, Y.get(), k, Rx.get(), p);
      std::swap(X, Y);
      // Rayleigh-Ritz: Z = R'^T X (right: R' X) = Qz Rz, Rz = Uz S Vz^T
      dgemm(st, !right, false, k, p, k, 1.0, Rt, ldr, X.get(), k, 0.0, Y.get(), k);
      {
        DBuf<double> Qz((size_t)k * p, st);
        householder_qr(st, k, p, Y.get(), k, Qz.get(), k, Rx.get(), p);
      }
      rr = SvdOut();
      // (trunc_rel 1: rotations below 64 eps ||Rz|| are skipped -- far below
      // the eps ||M|| accuracy the cut needs; the block's values span many decades)
      if (!small_svd(st, p, p, Rx.get(), p, rr, 1.0)) svd_thin(st, p, p, Rx.get(), p, rr, 1.0);
      std::vector<double> sd(p);
      CK(cudaMemcpyAsync(sd.data(), rr.s.get(), sizeof(double) * p, cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      for (int64_t j = 0; j < p; ++j) a[j] = sd[p - 1 - j];   // ascending
      for (double v : a)
        if (!std::isfinite(v)) return false;
      // the cut: the largest t whose smallest-first tail sum stays <= delta^2
      const double d2 = delta * delta;
      double acc = 0.0;
      t = 0;
      while (t < p && acc + a[t] * a[t] <= d2) { acc += a[t] * a[t]; ++t; }
      t = std::min<int64_t>(t, k - 1);   // _truncation_rank's floor of 1
      // converged when the discarded directions' residual contamination by
      // the kept ones outside the block, a_p (a_{t-1} / a_p)^{2(it+1)} from
      // a random start (a_{p-1} <= a_p bounds it from above), is a thousandth
      // of delta, and the cut did not move since the last step
      const double aj = a[t > 0 ? t - 1 : 0], ap = a[p - 1];
      const double decay = ap > 0.0 ? std::pow(aj / ap, 2.0 * (it + 1)) : 1.0;
      const double contam = ap * decay * std::sqrt((double)k) * 10.0;
      const bool same = !prev.empty() && prev[0] == (double)t;
      const bool inside = t <= p - 8;
      if (inside && it >= 1 && same && contam <= 1e-3 * delta) ok = true;
      prev.assign(1, (double)t);
      if (trace)
        std::fprintf(stderr, "[mpo_b200] tail_cut k=%lld p=%lld it=%d t=%lld a0=%.3e a_t-1=%.3e "
                     "a_t=%.3e a_p-1=%.3e delta=%.3e contam=%.2e%s\n", (long long)k, (long long)p,
                     it, (long long)t, a[0], a[t > 0 ? t - 1 : 0], a[std::min<int64_t>(t, p - 1)],
                     a[p - 1], delta, contam, ok ? " ok" : "");
      if (!inside) break;   // the cut is not inside the block: a wider one
      // steps still needed at the current rate (aj / ap)^2 per step: give up
      // early when they do not fit in the budget
      if (!ok && it >= 1 && aj > 0.0 && ap > aj) {
        const double need = std::log(1e-3 * delta / contam) / (2.0 * std::log(aj / ap));
        if (it + 1 + need > maxit) break;
      }
    }
    if (!ok) continue;
    out.t = t;
    const int64_t r = k - t;
    out.has_c = build_c || t == 0;
    if (out.has_c) out.C.alloc((size_t)k * r, st);
    if (t == 0) {
      set_identity(st, k, k, out.C.get(), k);
      return true;
    }
    // U_t = X Vz[:, p-t:p]  (the Ritz vectors of the t smallest values;
    // Vz^T = rr.vh, p x p, ld p)
    DBuf<double> Ut((size_t)k * t, st), Rt_((size_t)t * t, st);
    dgemm(st, false, true, k, t, p, 1.0, X.get(), k, rr.vh.get() + (p - t), p, 0.0, Ut.get(), k);
    // C = H [0; I_r], H the Householder reflectors of U_t
    householder_qr_keep(st, k, t, Ut.get(), k, Rt_.get(), t, out.f);
    if (!out.has_c) return true;
    fill_zero(st, out.C.get(), k * r);
    set_identity(st, r, r, out.C.get() + t, k);
    qr_apply_q(st, out.f, out.C.get(), k, r);
    return true;
  }
  return false;
}

}  // namespace mpob

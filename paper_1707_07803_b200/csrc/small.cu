// Single-CTA factorizations for the tiny-rank regime (config 1, the ends of
// every chain): a thin Householder QR and a QR-preconditioned one-sided
// Jacobi SVD of matrices that fit one CTA's shared memory, each ONE launch
// with the iteration converged on chip (no per-sweep host round trip).
// Same contracts as householder_qr (qr.cu) and svd_thin (svd.cu), which
// take everything larger:
//   QR  (rsvd.py:106, :132, :160 -> LAPACK dgeqrf + dorgqr): LAPACK's
//       reflector convention beta = -sign(alpha) ||x||, so Q and R match the
//       blocked path's (and the reference's) signs;
//   SVD (rsvd.py:128, :189 -> dgesdd): all min(m, n) <= 32 singular values,
//       descending with index tie-break, M = Ucarry Vh, Ucarry = U diag(s),
//       Vh with orthonormal rows (no division by s).
#include <cmath>

#include "common.cuh"
#include "kernels.cuh"

namespace mpob {

namespace {

constexpr int S_CT = 512;                // threads (16 warps)
constexpr int S_W = S_CT / 32;
constexpr int S_MAXE = 12288;            // doubles of the factored matrix in smem
constexpr int S_MAXK = 64;               // SVD: k = min(m, n) <= 64 (lane = row, two rows per lane above 32)
constexpr int S_MAXQ = 64;               // QR: kk = min(m, n) <= 64

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// H_j = I - tj v v^T (v = [1; x[j+1:m]]) applied by one warp to the nc <= 4
// columns Y + c * ldy, c = 0..3, at once: the four dots share the loads of x
// and reduce in one transposing butterfly (6 exchanges + 4 broadcasts instead
// of 4 x 5), then the four updates.
__device__ __forceinline__ void apply_reflector4(const double* x, double tj, int j, int m, double* Y,
                                                 int ldy, int nc) {
  const int lane = threadIdx.x & 31;
  double* y[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) y[u] = Y + (size_t)min(u, nc - 1) * ldy;
  double w[4];
#pragma unroll
  for (int u = 0; u < 4; ++u) w[u] = lane == 0 ? y[u][j] : 0.0;
  for (int i = j + 1 + lane; i < m; i += 32) {
    const double xi = x[i];
#pragma unroll
    for (int u = 0; u < 4; ++u) w[u] = fma(xi, y[u][i], w[u]);
  }
  const bool hi = lane & 16, mid = lane & 8;
  double k0 = (hi ? w[2] : w[0]) + __shfl_xor_sync(0xffffffffu, hi ? w[0] : w[2], 16);
  double k1 = (hi ? w[3] : w[1]) + __shfl_xor_sync(0xffffffffu, hi ? w[1] : w[3], 16);
  double k = (mid ? k1 : k0) + __shfl_xor_sync(0xffffffffu, mid ? k0 : k1, 8);
  k += __shfl_xor_sync(0xffffffffu, k, 4);
  k += __shfl_xor_sync(0xffffffffu, k, 2);
  k += __shfl_xor_sync(0xffffffffu, k, 1);
#pragma unroll
  for (int u = 0; u < 4; ++u) w[u] = __shfl_sync(0xffffffffu, k, 8 * u) * tj;
  if (lane == 0) {
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (u < nc) y[u][j] -= w[u];
  }
  for (int i = j + 1 + lane; i < m; i += 32) {
    const double xi = x[i];
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (u < nc) y[u][i] = fma(-w[u], xi, y[u][i]);
  }
}

// In-place Householder QR of the column-major m x n matrix A (ld m) in
// shared memory, kk = min(m, n) reflectors (dlarfg convention): R in the
// upper triangle, v_j below the diagonal (v_j[0] = 1 implicit), tau[j].
__device__ void block_qr(double* A, int m, int n, double* tau, double* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int kk = min(m, n);
  for (int j = 0; j < kk; ++j) {
    double* x = A + (size_t)j * m;
    // ||x[j+1:m]||^2 (fixed-order block reduction)
    double p = 0.0;
    for (int i = j + 1 + threadIdx.x; i < m; i += S_CT) p += x[i] * x[i];
    p = warp_sum(p);
    if (lane == 0) red[warp] = p;
    __syncthreads();
    if (threadIdx.x == 0) {
      double s2 = 0.0;
      for (int w = 0; w < S_W; ++w) s2 += red[w];
      const double alpha = x[j];
      double t = 0.0, scale = 0.0, beta = alpha;
      if (s2 > 0.0) {
        const double nrm = sqrt(alpha * alpha + s2);
        beta = alpha >= 0.0 ? -nrm : nrm;
        t = (beta - alpha) / beta;
        scale = 1.0 / (alpha - beta);
      }
      tau[j] = t;
      red[S_W] = scale;
      x[j] = beta;
    }
    __syncthreads();
    const double scale = red[S_W];
    if (tau[j] != 0.0)
      for (int i = j + 1 + threadIdx.x; i < m; i += S_CT) x[i] *= scale;
    __syncthreads();
    // apply H_j to the trailing columns: four columns per warp, or one per
    // warp when there is a warp for every column
    const double tj = tau[j];
    if (tj != 0.0) {
      const int per = n - j - 1 <= S_W ? 1 : 4;
      for (int c = j + 1 + per * warp; c < n; c += per * S_W)
        apply_reflector4(x, tj, j, m, A + (size_t)c * m, m, min(per, n - c));
    }
    __syncthreads();
  }
}

// C <- Q C for the m x nc column-major C (ld ldc) whose rows >= kk are
// zero on entry: the reflectors of block_qr applied backwards (dorgqr).
__device__ void block_apply_q(const double* A, int m, int kk, const double* tau, double* C,
                              int ldc, int nc) {
  const int warp = threadIdx.x >> 5;
  for (int j = kk - 1; j >= 0; --j) {
    const double tj = tau[j];
    if (tj != 0.0) {
      const double* x = A + (size_t)j * m;
      const int per = nc <= S_W ? 1 : 4;
      for (int c = per * warp; c < nc; c += per * S_W)
        apply_reflector4(x, tj, j, m, C + (size_t)c * ldc, ldc, min(per, nc - c));
    }
    __syncthreads();
  }
}

__global__ void __launch_bounds__(S_CT) small_qr_kernel(int m, int n, const double* __restrict__ Ain,
                                                        int64_t lda, double* __restrict__ Q,
                                                        int64_t ldq, double* __restrict__ R,
                                                        int64_t ldr) {
  extern __shared__ __align__(16) double sm[];
  double* A = sm;                            // m x n
  double* C = A + (size_t)m * n;             // m x kk (Q)
  double* tau = C + (size_t)m * min(m, n);
  double* red = tau + S_MAXQ;
  const int kk = min(m, n);
  for (int e = threadIdx.x; e < m * n; e += S_CT) A[e] = Ain[(e % m) + (int64_t)(e / m) * lda];
  for (int e = threadIdx.x; e < m * kk; e += S_CT) C[e] = (e % m == e / m) ? 1.0 : 0.0;
  __syncthreads();
  block_qr(A, m, n, tau, red);
  if (R)
    for (int e = threadIdx.x; e < kk * n; e += S_CT) {
      const int i = e % kk, c = e / kk;
      R[i + c * ldr] = i <= c ? A[i + (size_t)c * m] : 0.0;
    }
  if (Q) {
    block_apply_q(A, m, kk, tau, C, m, kk);
    for (int e = threadIdx.x; e < m * kk; e += S_CT) Q[(e % m) + (int64_t)(e / m) * ldq] = C[e];
  }
}

// One-sided Jacobi SVD of an m x n matrix, k = min(m, n) <= 64:
// QR of the tall orientation (M^T if wide), then cyclic round-robin Jacobi
// on the k x k factor X (16 warps rotate disjoint column pairs, one or two
// pairs per warp and round; lane = row, rows lane and lane + 32 when k > 32),
// converged on chip; then sort and the finishing products.
__global__ void __launch_bounds__(S_CT) small_svd_kernel(int m, int n, const double* __restrict__ M,
                                                         int64_t ldm, double* __restrict__ s_out,
                                                         double* __restrict__ ucarry,
                                                         double* __restrict__ vh,
                                                         double floorc) {
  extern __shared__ __align__(16) double sm[];
  const bool wide = m <= n;
  const int k = min(m, n), tm = wide ? n : m;
  const int KP = k <= 32 ? 32 : 64;          // padded order of X and V
  double* A = sm;                            // tm x k: the tall orientation, then reflectors
  double* Cb = A + (size_t)tm * k;           // tm x k: finishing product
  double* X = Cb + (size_t)tm * k;           // KP x KP
  double* V = X + KP * KP;                   // KP x KP
  double* tau = V + KP * KP;
  double* red = tau + S_MAXK;
  double* nrm = red + S_W + 1;
  __shared__ int perm[S_MAXK];
  __shared__ int s_rot, s_pair[S_MAXK / 2][2];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const bool two = KP > 32;                  // second row lane + 32
  for (int e = threadIdx.x; e < tm * k; e += S_CT) {
    const int i = e % tm, c = e / tm;   // A[i, c]
    A[e] = wide ? M[c + (int64_t)i * ldm] : M[i + (int64_t)c * ldm];
  }
  __syncthreads();
  block_qr(A, tm, k, tau, red);
  // X = R^T (wide: M = R^T Q^T) or R (tall: M = Q R), V = I, zero padded to KP
  for (int e = threadIdx.x; e < KP * KP; e += S_CT) {
    const int i = e % KP, c = e / KP;
    double v = 0.0;
    if (i < k && c < k) v = wide ? (c <= i ? A[c + (size_t)i * tm] : 0.0)
                                 : (i <= c ? A[i + (size_t)c * tm] : 0.0);
    X[e] = v;
    V[e] = (i == c) ? 1.0 : 0.0;
  }
  __syncthreads();
  const double eps = 2.220446049250313e-16;
  const double tol = 8.0 * eps * sqrt((double)k);
  // ||X||_F^2 (invariant under the rotations): couplings below
  // floorc ||X||_F x the larger column norm are skipped -- for truncation
  // SVDs (floorc = min(64 eps, 1e-2 delta/||X||), as svd.cu) they move no
  // singular value by more than the backward error of any SVD; otherwise
  // floorc = eps^2, which only keeps (near-)zero and denormal columns from
  // rotating forever
  if (warp == 0) {
    double f = 0.0;
    for (int c = 0; c < k; ++c) {
      f += X[lane + KP * c] * X[lane + KP * c];
      if (two) f += X[lane + 32 + KP * c] * X[lane + 32 + KP * c];
    }
    f = warp_sum(f);
    if (lane == 0) red[0] = f;
  }
  __syncthreads();
  const double fro2 = red[0];
  const int kp = (k + 1) & ~1;   // even number of slots for the tournament
  int sweep = 0;
  for (; sweep < 60; ++sweep) {
    if (threadIdx.x == 0) s_rot = 0;
    __syncthreads();
    for (int r = 0; r < kp - 1; ++r) {
      // round-robin pairing: slot 0 fixed, the rest rotate
      if (threadIdx.x < kp / 2) {
        const int t = threadIdx.x;
        auto slot = [&](int pos) { return pos == 0 ? 0 : 1 + (pos - 1 + r) % (kp - 1); };
        s_pair[t][0] = slot(t);
        s_pair[t][1] = slot(kp - 1 - t);
      }
      __syncthreads();
      for (int pi = warp; pi < kp / 2; pi += S_W) {
        const int p = min(s_pair[pi][0], s_pair[pi][1]);
        const int q = max(s_pair[pi][0], s_pair[pi][1]);
        if (q < k) {
          const double xp = X[lane + KP * p], xq = X[lane + KP * q];
          const double xp2 = two ? X[lane + 32 + KP * p] : 0.0, xq2 = two ? X[lane + 32 + KP * q] : 0.0;
          const double a = warp_sum(fma(xp, xp, xp2 * xp2)), b = warp_sum(fma(xq, xq, xq2 * xq2)),
                       c = warp_sum(fma(xp, xq, xp2 * xq2));
          if (c != 0.0 && fabs(c) > tol * sqrt(a) * sqrt(b) &&
              c * c > floorc * floorc * fro2 * fmax(a, b)) {
            const double zeta = (b - a) / (2.0 * c);
            const double t = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
            const double cs = 1.0 / sqrt(1.0 + t * t), sn = cs * t;
            X[lane + KP * p] = cs * xp - sn * xq;
            X[lane + KP * q] = sn * xp + cs * xq;
            const double vp = V[lane + KP * p], vq = V[lane + KP * q];
            V[lane + KP * p] = cs * vp - sn * vq;
            V[lane + KP * q] = sn * vp + cs * vq;
            if (two) {
              X[lane + 32 + KP * p] = cs * xp2 - sn * xq2;
              X[lane + 32 + KP * q] = sn * xp2 + cs * xq2;
              const double vp2 = V[lane + 32 + KP * p], vq2 = V[lane + 32 + KP * q];
              V[lane + 32 + KP * p] = cs * vp2 - sn * vq2;
              V[lane + 32 + KP * q] = sn * vp2 + cs * vq2;
            }
            if (lane == 0) s_rot = 1;
          }
        }
      }
      __syncthreads();
    }
    const int rot = s_rot;
    __syncthreads();   // every thread has read the flag before it is reset
    if (!rot) break;
  }
  const bool failed = sweep == 60;   // not converged: NaN singular values (the host raises)
  // singular values: column norms, descending, index tie-break
  if (threadIdx.x < KP) {
    const int col = threadIdx.x;
    double v = 0.0;
    for (int i = 0; i < KP; ++i) v += X[i + KP * col] * X[i + KP * col];
    nrm[col] = col < k ? sqrt(v) : -1.0;
  }
  __syncthreads();
  if (threadIdx.x < k) {
    const int col = threadIdx.x;
    const double v = nrm[col];
    int rank = 0;
    for (int j = 0; j < k; ++j) {
      const double u = nrm[j];
      rank += (u > v) || (u == v && j < col);
    }
    perm[rank] = col;
    s_out[rank] = failed ? nan("") : v;
  }
  __syncthreads();
  // finishing: wide  M = X Vs^T Q^T ... Ucarry = Ys (k x k), Vh = (Q [Vs; 0])^T
  //            tall  M = Q X:          Ucarry = Q [Ys; 0],   Vh = Vs^T
  const double* Fin = wide ? V : X;   // the factor that meets Q
  for (int e = threadIdx.x; e < tm * k; e += S_CT) {
    const int i = e % tm, c = e / tm;
    Cb[e] = i < k ? Fin[i + KP * perm[c]] : 0.0;
  }
  __syncthreads();
  block_apply_q(A, tm, k, tau, Cb, tm, k);
  if (wide) {
    for (int e = threadIdx.x; e < k * k; e += S_CT) {
      const int i = e % k, c = e / k;
      ucarry[i + (int64_t)c * m] = X[i + KP * perm[c]];
    }
    for (int e = threadIdx.x; e < k * n; e += S_CT) {
      const int r = e % k, c = e / k;   // vh[r, c] = (Q Vs)[c, r]
      vh[r + (int64_t)c * k] = Cb[c + (size_t)r * tm];
    }
  } else {
    for (int e = threadIdx.x; e < m * k; e += S_CT) ucarry[e] = Cb[e];
    for (int e = threadIdx.x; e < k * k; e += S_CT) {
      const int r = e % k, c = e / k;   // vh[r, c] = Vs[c, r]
      vh[r + (int64_t)c * k] = V[c + KP * perm[r]];
    }
  }
}

size_t qr_smem(int64_t m, int64_t n) {
  const int64_t kk = std::min(m, n);
  return sizeof(double) * (size_t)(m * n + m * kk + S_MAXQ + S_W + 1);
}
size_t svd_smem(int64_t m, int64_t n) {
  const int64_t k = std::min(m, n), tm = std::max(m, n);
  const int64_t kpad = k <= 32 ? 32 : 64;
  return sizeof(double) * (size_t)(2 * tm * k + 2 * kpad * kpad + S_MAXK + S_W + 1 + S_MAXK);
}

void set_attrs() {
  static std::once_flag once[kMaxDevices];
  once_per_device(once, [] {
    CK(cudaFuncSetAttribute(small_qr_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            200 * 1024));
    CK(cudaFuncSetAttribute(small_svd_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            220 * 1024));
  });
}

}  // namespace

bool small_qr(cudaStream_t st, int64_t m, int64_t n, const double* A, int64_t lda, double* Q,
              int64_t ldq, double* R, int64_t ldr) {
  static const bool off = std::getenv("MPO_B200_SMALL") && std::atoi(std::getenv("MPO_B200_SMALL")) == 0;
  if (off || m < 1 || n < 1 || std::min(m, n) > S_MAXQ || m * n > S_MAXE ||
      qr_smem(m, n) > 200 * 1024)
    return false;
  set_attrs();
  small_qr_kernel<<<1, S_CT, qr_smem(m, n), st>>>((int)m, (int)n, A, lda, Q, ldq, R, ldr);
  CK_LAUNCH();
  note_launch();
  return true;
}

bool small_svd(cudaStream_t st, int64_t m, int64_t n, const double* M, int64_t ldm, SvdOut& out,
               double trunc_rel) {
  static const bool off = std::getenv("MPO_B200_SMALL") && std::atoi(std::getenv("MPO_B200_SMALL")) == 0;
  const int64_t k = std::min(m, n), tm = std::max(m, n);
  if (off || k < 1 || k > S_MAXK || tm * k > S_MAXE || svd_smem(m, n) > 220 * 1024) return false;
  set_attrs();
  out.k = k;
  out.s.alloc(k, st);
  out.ucarry.alloc((size_t)m * k, st);
  out.vh.alloc((size_t)k * n, st);
  const double eps = 2.220446049250313e-16;
  const double floorc = trunc_rel > 0.0 ? std::min(64.0 * eps, 1e-2 * trunc_rel) : eps * eps;
  small_svd_kernel<<<1, S_CT, svd_smem(m, n), st>>>((int)m, (int)n, M, ldm, out.s.get(),
                                                   out.ucarry.get(), out.vh.get(), floorc);
  CK_LAUNCH();
  note_launch();
  return true;
}

}  // namespace mpob

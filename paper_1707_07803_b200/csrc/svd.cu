// Thin SVD on sm_100a, replacing LAPACK dgesdd behind
// np.linalg.svd(full_matrices=False) at rsvd.py:128 (truncation sweep) and
// rsvd.py:189 (first-core SVD of Algorithm 4).
//
// Algorithm: QR preconditioning (Householder QR of the tall orientation,
// qr.cu) followed by one-sided block Jacobi (Hestenes) on the k x k
// triangular factor X.  Columns are grouped in blocks of JB = 16; each
// round of the round-robin tournament pairs every block with another, and
// one CTA per pair
//   1. forms the 32 x 32 Gram matrix of its two column blocks (DMMA),
//   2. diagonalises it in shared memory with cyclic two-sided Jacobi
//      (rotations accumulated into J), and
//   3. applies J to the X and V column blocks (DMMA).
// A sweep is nb-1 rounds; iteration stops when a whole sweep performs no
// rotation (every pair has |x_p.x_q| <= tol ||x_p|| ||x_q||), which gives
// singular values to absolute accuracy O(eps ||M||) like dgesdd.  Singular
// values are the final column norms, sorted descending with index
// tie-break (deterministic).  No atomics anywhere.
#include "common.cuh"
#include "kernels.cuh"

namespace mpob {

namespace {

constexpr int JB = 16;          // columns per Jacobi block
constexpr int P2 = 2 * JB;      // columns per pair
constexpr int CH = 64;          // rows per streamed chunk
constexpr int CLD = P2 + 4;     // chunk row stride (doubles): conflict-free fragments
constexpr int GLD = P2 + 1;
constexpr int JT = 256;

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile(
      "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 "
      "{%0, %1}, {%2}, {%3}, {%0, %1};\n"
      : "+d"(c[0]), "+d"(c[1])
      : "d"(a), "d"(b));
}

__device__ __forceinline__ void pair_of_round(int nb, int r, int i, int& x, int& y) {
  // circle method: slot 0 fixed, slots 1..nb-1 rotate by r
  auto slot = [&](int j) { return j == 0 ? 0 : 1 + ((j - 1 + r) % (nb - 1)); };
  x = slot(i);
  y = slot(nb - 1 - i);
}

struct RoundArgs {
  double* X;     // rows x ncols_pad, ld = ldx
  int64_t ldx, rows;
  double* V;     // vrows x ncols_pad, ld = ldv
  int64_t ldv, vrows;
  int nb, round;
  double tol;
  int* flag;     // set to 1 when any rotation happened
};

// stream the 2*JB columns of blocks (bx, by) through shared memory
__device__ __forceinline__ int64_t gcol(int c, int bx, int by) {
  return c < JB ? (int64_t)bx * JB + c : (int64_t)by * JB + (c - JB);
}

__global__ void __launch_bounds__(JT) jacobi_round_kernel(RoundArgs a) {
  __shared__ double G[P2 * GLD];
  __shared__ double J[P2 * GLD];
  __shared__ double chunk[CH * CLD];
  __shared__ double rc[P2 / 2], rs[P2 / 2];
  __shared__ int rp[P2 / 2], rq[P2 / 2];
  __shared__ int s_any, s_skip;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  int bx, by;
  pair_of_round(a.nb, a.round, blockIdx.x, bx, by);

  // ---- 1. Gram matrix of the 32 columns (DMMA over row chunks) ----
  const int ti = warp >> 1, tj0 = (warp & 1) * 2;
  double acc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
  for (int64_t r0 = 0; r0 < a.rows; r0 += CH) {
    __syncthreads();
    for (int idx = t; idx < CH * P2; idx += JT) {
      int r = idx % CH, c = idx / CH;
      int64_t gr = r0 + r;
      chunk[r * CLD + c] = gr < a.rows ? a.X[gr + gcol(c, bx, by) * a.ldx] : 0.0;
    }
    __syncthreads();
#pragma unroll 4
    for (int k0 = 0; k0 < CH; k0 += 4) {
      const double* row = chunk + (k0 + (lane & 3)) * CLD + (lane >> 2);
      double av = row[ti * 8];
      dmma(acc[0], av, row[tj0 * 8]);
      dmma(acc[1], av, row[(tj0 + 1) * 8]);
    }
  }
  {
    const int gi = ti * 8 + (lane >> 2);
#pragma unroll
    for (int u = 0; u < 2; ++u)
#pragma unroll
      for (int e = 0; e < 2; ++e) G[gi * GLD + (tj0 + u) * 8 + 2 * (lane & 3) + e] = acc[u][e];
  }
  for (int idx = t; idx < P2 * P2; idx += JT) J[(idx / P2) * GLD + idx % P2] = (idx / P2 == idx % P2) ? 1.0 : 0.0;
  if (t == 0) { s_any = 0; s_skip = 1; }
  __syncthreads();
  // symmetrise (the two halves come from different DMMA tiles; use the
  // upper one for both so the inner problem is exactly symmetric)
  for (int idx = t; idx < P2 * P2; idx += JT) {
    int i = idx / P2, j = idx % P2;
    if (i > j) G[i * GLD + j] = G[j * GLD + i];
  }
  __syncthreads();
  // convergence test over all column pairs of the two blocks
  for (int idx = t; idx < P2 * P2; idx += JT) {
    int i = idx / P2, j = idx % P2;
    if (i < j) {
      // sqrt before multiplying: G_ii * G_jj underflows for graded columns
      double gij = G[i * GLD + j], d = sqrt(G[i * GLD + i]) * sqrt(G[j * GLD + j]);
      if (d > 0.0 && fabs(gij) > a.tol * d) s_skip = 0;
    }
  }
  __syncthreads();
  if (s_skip) return;

  // ---- 2. cyclic two-sided Jacobi on G (parallel circle ordering) ----
  for (int sweep = 0; sweep < 12; ++sweep) {
    int any = 0;
    for (int r = 0; r < P2 - 1; ++r) {
      if (t < P2 / 2) {
        int p, q;
        pair_of_round(P2, r, t, p, q);
        if (p > q) { int tmp = p; p = q; q = tmp; }
        double gpp = G[p * GLD + p], gqq = G[q * GLD + q], gpq = G[p * GLD + q];
        double c = 1.0, s = 0.0;
        const double dd = sqrt(gpp) * sqrt(gqq);
        if (dd > 0.0 && fabs(gpq) > a.tol * dd) {
          double zeta = (gqq - gpp) / (2.0 * gpq);
          double tt = (zeta >= 0.0 ? 1.0 : -1.0) / (fabs(zeta) + sqrt(1.0 + zeta * zeta));
          c = 1.0 / sqrt(1.0 + tt * tt);
          s = tt * c;
        }
        rp[t] = p; rq[t] = q; rc[t] = c; rs[t] = s;
      }
      __syncthreads();
      // column update of G and J: (col_p, col_q) <- (c col_p - s col_q, s col_p + c col_q)
      for (int idx = t; idx < (P2 / 2) * P2; idx += JT) {
        int pr = idx / P2, j = idx % P2;
        double c = rc[pr], s = rs[pr];
        if (s != 0.0) {
          int p = rp[pr], q = rq[pr];
          double gp = G[j * GLD + p], gq = G[j * GLD + q];
          G[j * GLD + p] = c * gp - s * gq;
          G[j * GLD + q] = s * gp + c * gq;
          double jp = J[j * GLD + p], jq = J[j * GLD + q];
          J[j * GLD + p] = c * jp - s * jq;
          J[j * GLD + q] = s * jp + c * jq;
        }
      }
      __syncthreads();
      // row update of G
      for (int idx = t; idx < (P2 / 2) * P2; idx += JT) {
        int pr = idx / P2, j = idx % P2;
        double c = rc[pr], s = rs[pr];
        if (s != 0.0) {
          int p = rp[pr], q = rq[pr];
          double gp = G[p * GLD + j], gq = G[q * GLD + j];
          G[p * GLD + j] = c * gp - s * gq;
          G[q * GLD + j] = s * gp + c * gq;
        }
      }
      __syncthreads();
      if (t < P2 / 2 && rs[t] != 0.0) {
        int p = rp[t], q = rq[t];
        G[p * GLD + q] = 0.0;
        G[q * GLD + p] = 0.0;
        s_any = 1;
      }
      __syncthreads();
      any |= s_any;
      __syncthreads();
      if (t == 0) s_any = 0;
    }
    if (!any) break;
  }
  if (t == 0) *a.flag = 1;

  // re-orthogonalise J (one Newton-Schulz step J <- J (3I - J^T J) / 2):
  // hundreds of accumulated plane rotations drift O(n_rot * eps) from
  // orthogonal, which would otherwise build up in V over the sweeps
  {
    double* E = G;  // G is no longer needed
    __syncthreads();
    for (int idx = t; idx < P2 * P2; idx += JT) {
      int i = idx / P2, j = idx % P2;
      double acc = 0.0;
      for (int l = 0; l < P2; ++l) acc = fma(J[l * GLD + i], J[l * GLD + j], acc);
      E[i * GLD + j] = acc - (i == j ? 1.0 : 0.0);
    }
    __syncthreads();
    double nv[P2 * P2 / JT];
#pragma unroll
    for (int e = 0; e < P2 * P2 / JT; ++e) {
      int idx = t + e * JT, i = idx / P2, j = idx % P2;
      double acc = 0.0;
      for (int l = 0; l < P2; ++l) acc = fma(J[i * GLD + l], E[l * GLD + j], acc);
      nv[e] = J[i * GLD + j] - 0.5 * acc;
    }
    __syncthreads();
#pragma unroll
    for (int e = 0; e < P2 * P2 / JT; ++e) {
      int idx = t + e * JT;
      J[(idx / P2) * GLD + idx % P2] = nv[e];
    }
    __syncthreads();
  }

  // ---- 3. apply J to the X and V column blocks (DMMA) ----
  // B fragments of J stay in registers: bj[ks][nt] = J[4ks + (lane&3)][8nt + (lane>>2)]
  double bj[8][4];
#pragma unroll
  for (int ks = 0; ks < 8; ++ks)
#pragma unroll
    for (int nt = 0; nt < 4; ++nt) bj[ks][nt] = J[(4 * ks + (lane & 3)) * GLD + 8 * nt + (lane >> 2)];
  for (int which = 0; which < 2; ++which) {
    double* M = which == 0 ? a.X : a.V;
    const int64_t ld = which == 0 ? a.ldx : a.ldv;
    const int64_t rows = which == 0 ? a.rows : a.vrows;
    for (int64_t r0 = 0; r0 < rows; r0 += CH) {
      __syncthreads();
      for (int idx = t; idx < CH * P2; idx += JT) {
        int r = idx % CH, c = idx / CH;
        int64_t gr = r0 + r;
        chunk[r * CLD + c] = gr < rows ? M[gr + gcol(c, bx, by) * ld] : 0.0;
      }
      __syncthreads();
      double o[4][2] = {{0, 0}, {0, 0}, {0, 0}, {0, 0}};
      const double* arow = chunk + (8 * warp + (lane >> 2)) * CLD + (lane & 3);
#pragma unroll
      for (int ks = 0; ks < 8; ++ks) {
        double av = arow[4 * ks];
#pragma unroll
        for (int nt = 0; nt < 4; ++nt) dmma(o[nt], av, bj[ks][nt]);
      }
      __syncwarp();
      double* orow = chunk + (8 * warp + (lane >> 2)) * CLD + 2 * (lane & 3);
#pragma unroll
      for (int nt = 0; nt < 4; ++nt) { orow[8 * nt] = o[nt][0]; orow[8 * nt + 1] = o[nt][1]; }
      __syncthreads();
      for (int idx = t; idx < CH * P2; idx += JT) {
        int r = idx % CH, c = idx / CH;
        int64_t gr = r0 + r;
        if (gr < rows) M[gr + gcol(c, bx, by) * ld] = chunk[r * CLD + c];
      }
    }
  }
}

// per-column norms (one warp per column, fixed reduction order)
__global__ void col_norms_kernel(const double* X, int64_t rows, int64_t ld, int64_t ncols,
                                 double* out) {
  const int lane = threadIdx.x & 31;
  const int64_t col = blockIdx.x * (int64_t)(blockDim.x / 32) + (threadIdx.x >> 5);
  if (col >= ncols) return;
  double s = 0.0;
  for (int64_t r = lane; r < rows; r += 32) { double x = X[r + col * ld]; s = fma(x, x, s); }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) out[col] = sqrt(s);
}

// single-CTA bitonic sort of (value desc, index asc); n <= 8192 padded to pow2
__global__ void sort_desc_kernel(const double* vals, int n, int npow2, double* sorted,
                                 int* perm) {
  extern __shared__ unsigned char smem[];
  double* v = reinterpret_cast<double*>(smem);
  int* ix = reinterpret_cast<int*>(v + npow2);
  for (int i = threadIdx.x; i < npow2; i += blockDim.x) {
    v[i] = i < n ? vals[i] : -1.0;
    ix[i] = i;
  }
  __syncthreads();
  for (int k = 2; k <= npow2; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < npow2; i += blockDim.x) {
        int l = i ^ j;
        if (l > i) {
          // "before(a, b)": a has larger value, or equal value and smaller index
          bool dir = (i & k) == 0;
          double vi = v[i], vl = v[l];
          int ii = ix[i], il = ix[l];
          bool l_before_i = (vl > vi) || (vl == vi && il < ii);
          if (l_before_i == dir) {
            v[i] = vl; v[l] = vi; ix[i] = il; ix[l] = ii;
          }
        }
      }
      __syncthreads();
    }
  }
  for (int i = threadIdx.x; i < n; i += blockDim.x) { sorted[i] = v[i]; perm[i] = ix[i]; }
}

// B[:, j] = A[0:rows, perm[j]]
__global__ void gather_cols_kernel(const double* A, int64_t lda, int64_t rows, const int* perm,
                                   int64_t ncols, double* B, int64_t ldb) {
  const int64_t total = rows * ncols;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    int64_t i = idx % rows, j = idx / rows;
    B[i + j * ldb] = A[i + (int64_t)perm[j] * lda];
  }
}

// X (k x kp) = lower triangle source transposed: X[i][j] = R[j][i] for j <= i (R upper k x k)
__global__ void tri_transpose_kernel(const double* R, int64_t ldr, int64_t k, int64_t kp,
                                     double* X, int upper) {
  const int64_t total = k * kp;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    int64_t i = idx % k, j = idx / k;
    double v = 0.0;
    if (j < k) {
      if (upper) v = (i <= j) ? R[i + j * ldr] : 0.0;      // X = R
      else v = (j <= i) ? R[j + i * ldr] : 0.0;            // X = R^T
    }
    X[i + j * k] = v;
  }
}

inline int gridn(int64_t n) {
  return (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(n, 256), 148 * 16));
}

}  // namespace

// Jacobi on the k x k matrix X (in place, ld = k, kp >= k padded columns
// present and zero).  V (kp x kp) accumulates the rotations.  Returns sweeps.
static int jacobi_sweeps(cudaStream_t st, double* X, int64_t k, int64_t kp, double* V) {
  set_identity(st, kp, kp, V, kp);
  const int nb = (int)(kp / JB);
  const double eps = 2.220446049250313e-16;
  const double tol = 8.0 * eps * sqrt((double)std::max<int64_t>(k, 1));
  DBuf<int> flag(1, st);
  int h_flag = 0, sweeps = 0;
  for (int sweep = 0; sweep < 60; ++sweep) {
    CK(cudaMemsetAsync(flag.get(), 0, sizeof(int), st));
    for (int r = 0; r < nb - 1; ++r) {
      RoundArgs a{X, k, k, V, kp, kp, nb, r, tol, flag.get()};
      jacobi_round_kernel<<<nb / 2, JT, 0, st>>>(a);
      CK_LAUNCH();
    }
    note_launch(nb - 1);
    CK(cudaMemcpyAsync(&h_flag, flag.get(), sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    ++sweeps;
    if (!h_flag) break;
  }
  return sweeps;
}

void svd_thin(cudaStream_t st, int64_t m, int64_t n, const double* M, int64_t ldm, SvdOut& out) {
  const int64_t k = std::min(m, n);
  out.k = k;
  if (k <= 0) return;
  const int64_t kp = cdiv(k, P2) * P2;
  const bool wide = m <= n;            // factor M^T = Q T  (n x m, tall)
  const int64_t tm = wide ? n : m;     // tall orientation rows
  DBuf<double> A((size_t)tm * k, st), Q((size_t)tm * k, st), R((size_t)k * k, st);
  if (wide) {
    int64_t dims[2] = {m, n};
    int perm[2] = {1, 0};
    if (ldm == m) permute(st, M, A.get(), 2, dims, perm);
    else {
      DBuf<double> tmp((size_t)m * n, st);
      copy_matrix(st, m, n, M, ldm, tmp.get(), m);
      permute(st, tmp.get(), A.get(), 2, dims, perm);
    }
  } else {
    copy_matrix(st, m, n, M, ldm, A.get(), m);
  }
  householder_qr(st, tm, k, A.get(), tm, Q.get(), tm, R.get(), k);
  // X = T^T (wide) or T (tall), padded to kp columns
  DBuf<double> X((size_t)k * kp, st), V((size_t)kp * kp, st);
  tri_transpose_kernel<<<gridn(k * kp), 256, 0, st>>>(R.get(), k, k, kp, X.get(), wide ? 0 : 1);
  CK_LAUNCH();
  note_launch();
  jacobi_sweeps(st, X.get(), k, kp, V.get());
  // singular values = column norms, sorted
  DBuf<double> norms(kp, st);
  col_norms_kernel<<<(int)cdiv(kp, 8), 256, 0, st>>>(X.get(), k, k, kp, norms.get());
  CK_LAUNCH();
  int np2 = 1;
  while (np2 < kp) np2 <<= 1;
  if (np2 > 8192) throw ValueError("svd: k > 8192 not supported by the single-CTA sort");
  DBuf<int> perm(kp, st);
  out.s.alloc(k, st);
  size_t ssmem = (size_t)np2 * (sizeof(double) + sizeof(int));
  if (ssmem > 48 * 1024)
    CK(cudaFuncSetAttribute(sort_desc_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ssmem));
  sort_desc_kernel<<<1, 1024, ssmem, st>>>(norms.get(), (int)kp, np2, norms.get(), perm.get());
  CK_LAUNCH();
  CK(cudaMemcpyAsync(out.s.get(), norms.get(), sizeof(double) * k, cudaMemcpyDeviceToDevice, st));
  note_launch(2);
  // sorted Y = X[:, perm] (k x k) and Vs = V[0:k, perm]
  DBuf<double> Ys((size_t)k * k, st), Vs((size_t)k * k, st);
  gather_cols_kernel<<<gridn(k * k), 256, 0, st>>>(X.get(), k, k, perm.get(), k, Ys.get(), k);
  CK_LAUNCH();
  gather_cols_kernel<<<gridn(k * k), 256, 0, st>>>(V.get(), kp, k, perm.get(), k, Vs.get(), k);
  CK_LAUNCH();
  note_launch(2);
  out.ucarry.alloc((size_t)m * k, st);
  out.vh.alloc((size_t)k * n, st);
  if (wide) {
    // M = X Q^T, X Vs = Ys:  Ucarry = Ys (m = k rows),  Vh = Vs^T Q^T = (Q Vs)^T
    copy_matrix(st, k, k, Ys.get(), k, out.ucarry.get(), m);
    dgemm(st, true, true, k, n, k, 1.0, Vs.get(), k, Q.get(), tm, 0.0, out.vh.get(), k);
  } else {
    // M = Q X:  Ucarry = Q Ys,  Vh = Vs^T
    dgemm(st, false, false, m, k, k, 1.0, Q.get(), tm, Ys.get(), k, 0.0, out.ucarry.get(), m);
    int64_t dims[2] = {k, k};
    int pr[2] = {1, 0};
    permute(st, Vs.get(), out.vh.get(), 2, dims, pr);
  }
}

}  // namespace mpob

namespace mpob {

namespace {

// W[:, j] = Ucarry[:, j] / s_j; columns with s_j == 0 are completed to an
// orthonormal set by Gram-Schmidt against unit vectors (single CTA, k small).
__global__ void left_vectors_kernel(int k, const double* U, int64_t ldu, const double* s,
                                    double* W) {
  extern __shared__ double cand[];
  __shared__ double red[32];
  __shared__ int s_ok;
  const int t = threadIdx.x;
  for (int j = 0; j < k; ++j) {
    double sj = s[j];
    if (sj > 0.0) {
      for (int i = t; i < k; i += blockDim.x) W[i + (int64_t)j * k] = U[i + j * ldu] / sj;
      __syncthreads();
      continue;
    }
    if (t == 0) s_ok = 0;
    __syncthreads();
    for (int e = 0; e < k && !s_ok; ++e) {
      for (int i = t; i < k; i += blockDim.x) cand[i] = (i == e) ? 1.0 : 0.0;
      __syncthreads();
      for (int p = 0; p < j; ++p) {       // two passes of classical GS per previous column
        for (int pass = 0; pass < 2; ++pass) {
          double d = 0.0;
          for (int i = t; i < k; i += blockDim.x) d += W[i + (int64_t)p * k] * cand[i];
          for (int o = 16; o > 0; o >>= 1) d += __shfl_xor_sync(0xffffffffu, d, o);
          if ((t & 31) == 0) red[t >> 5] = d;
          __syncthreads();
          if (t == 0) { double a = 0; for (int w = 0; w < (int)(blockDim.x >> 5); ++w) a += red[w]; red[0] = a; }
          __syncthreads();
          d = red[0];
          __syncthreads();
          for (int i = t; i < k; i += blockDim.x) cand[i] -= d * W[i + (int64_t)p * k];
          __syncthreads();
        }
      }
      double nn = 0.0;
      for (int i = t; i < k; i += blockDim.x) nn += cand[i] * cand[i];
      for (int o = 16; o > 0; o >>= 1) nn += __shfl_xor_sync(0xffffffffu, nn, o);
      if ((t & 31) == 0) red[t >> 5] = nn;
      __syncthreads();
      if (t == 0) { double a = 0; for (int w = 0; w < (int)(blockDim.x >> 5); ++w) a += red[w]; red[0] = sqrt(a); }
      __syncthreads();
      double nrm = red[0];
      if (nrm > 0.5) {
        for (int i = t; i < k; i += blockDim.x) W[i + (int64_t)j * k] = cand[i] / nrm;
        if (t == 0) s_ok = 1;
      }
      __syncthreads();
    }
  }
}

}  // namespace

void svd_left_vectors(cudaStream_t st, int64_t k, const double* ucarry, int64_t ldu,
                      const double* s, double* W) {
  if (k <= 0) return;
  if (k > 4096) throw ValueError("left singular vectors: k too large");
  left_vectors_kernel<<<1, 256, sizeof(double) * k, st>>>((int)k, ucarry, ldu, s, W);
  CK_LAUNCH();
  note_launch();
}

}  // namespace mpob

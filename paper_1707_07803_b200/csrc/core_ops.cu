// Elementwise / data-movement kernels of the TNrSVD path: the per-core MPO
// product (rsvd.py:62-79), F-order permutations (the reshape/transpose
// bookkeeping of rsvd.py:97, :159-160, :192), copies, scaling and the
// deterministic Frobenius norm of rsvd.py:123.
#include <deque>

#include "common.cuh"
#include "kernels.cuh"

namespace mpob {

namespace {

inline int grid_for(int64_t n, int threads = 256) {
  return (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(n, threads), 148 * 16));
}

__global__ void scale_kernel(int64_t m, int64_t n, double alpha, double* C, int64_t ldc,
                             int64_t batch, int64_t sC) {
  const int64_t total = m * n * batch;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    int64_t b = idx / (m * n), r = idx % (m * n);
    double* p = C + b * sC + (r % m) + (r / m) * ldc;
    *p = alpha == 0.0 ? 0.0 : alpha * *p;
  }
}

__global__ void copy_kernel(int64_t m, int64_t n, const double* __restrict__ A, int64_t lda,
                            double* __restrict__ B, int64_t ldb) {
  const int64_t total = m * n;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    int64_t i = idx % m, j = idx / m;
    B[i + j * ldb] = A[i + j * lda];
  }
}

__global__ void identity_kernel(int64_t m, int64_t n, double* A, int64_t lda) {
  const int64_t total = m * n;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    int64_t i = idx % m, j = idx / m;
    A[i + j * lda] = (i == j) ? 1.0 : 0.0;
  }
}

// Permutation of an F-ordered array, after unit axes are dropped and axes
// that stay adjacent are merged (host side).  A tile is 32 "x" positions
// (the input-fastest axis, or the first two input axes when the fastest is
// shorter than 32) by 32 "y" positions (the output-fastest axis, or the
// first two output axes), staged through shared memory so global reads run
// along x and global writes along y, both coalesced; the remaining axes are
// decomposed once per tile, not per element.
constexpr int TP = 32;
struct PermAxis2 {
  int64_t n1, n2;      // extents of the first / second axis of the group
  int64_t c2;          // positions of the second axis per tile (1 if single)
  int64_t is1, is2;    // input strides
  int64_t os1, os2;    // output strides
  int64_t tiles;
  bool comp;           // two-axis group
};
struct PermArgs {
  PermAxis2 X, Y;
  int nrest;
  int64_t rdim[4], ris[4], ros[4];  // remaining axes: extent, in/out strides
  int64_t ntiles;
};

struct PermIdx {
  int64_t in, out;
  bool ok;
};
__device__ __forceinline__ PermIdx perm_pos(const PermAxis2& g, int64_t b, int u) {
  PermIdx r;
  if (g.comp) {
    const int64_t a1 = u % g.n1, a2 = b * g.c2 + u / g.n1;
    r.ok = (u < g.n1 * g.c2) && a2 < g.n2;
    r.in = a1 * g.is1 + a2 * g.is2;
    r.out = a1 * g.os1 + a2 * g.os2;
  } else {
    const int64_t a1 = b * TP + u;
    r.ok = a1 < g.n1;
    r.in = a1 * g.is1;
    r.out = a1 * g.os1;
  }
  return r;
}

__global__ void __launch_bounds__(256) permute_tiled_kernel(const double* __restrict__ in,
                                                            double* __restrict__ out, PermArgs a) {
  __shared__ double tile[TP][TP + 1];
  const int tx = threadIdx.x & 31, ty = threadIdx.x >> 5;   // 32 x 8 threads
  for (int64_t t = blockIdx.x; t < a.ntiles; t += gridDim.x) {
    int64_t rem = t;
    const int64_t bx = rem % a.X.tiles; rem /= a.X.tiles;
    const int64_t by = rem % a.Y.tiles; rem /= a.Y.tiles;
    int64_t ib = 0, ob = 0;
    for (int q = 0; q < a.nrest; ++q) {
      const int64_t c = rem % a.rdim[q];
      rem /= a.rdim[q];
      ib += c * a.ris[q];
      ob += c * a.ros[q];
    }
    const PermIdx px = perm_pos(a.X, bx, tx);   // x position of this lane (reads)
    const PermIdx py = perm_pos(a.Y, by, tx);   // y position of this lane (writes)
    __syncthreads();
#pragma unroll
    for (int r = 0; r < TP; r += 8) {
      const PermIdx yy = perm_pos(a.Y, by, ty + r);
      if (px.ok && yy.ok) tile[ty + r][tx] = in[ib + px.in + yy.in];
    }
    __syncthreads();
#pragma unroll
    for (int r = 0; r < TP; r += 8) {
      const PermIdx xx = perm_pos(a.X, bx, ty + r);
      if (py.ok && xx.ok) out[ob + py.out + xx.out] = tile[tx][ty + r];
    }
  }
}

// fallback for permutations that keep a short input-fastest axis first
struct PermArgsG {
  int rank;
  int64_t odims[6];
  int64_t istride[6];
  int64_t total;
};
__global__ void permute_generic_kernel(const double* __restrict__ in, double* __restrict__ out,
                                       PermArgsG a) {
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < a.total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    int64_t rem = idx, off = 0;
#pragma unroll
    for (int q = 0; q < 6; ++q) {
      if (q < a.rank) {
        int64_t c = rem % a.odims[q];
        rem /= a.odims[q];
        off += c * a.istride[q];
      }
    }
    out[idx] = in[off];
  }
}

// contiguous runs (the output-fastest axis is the input-fastest axis)
__global__ void __launch_bounds__(256) permute_runs_kernel(const double* __restrict__ in,
                                                           double* __restrict__ out, PermArgs a) {
  const int64_t run = a.X.n1, tiles_x = a.X.tiles;
  for (int64_t t = blockIdx.x; t < a.ntiles; t += gridDim.x) {
    int64_t rem = t;
    const int64_t bx = rem % tiles_x; rem /= tiles_x;
    int64_t ib = 0, ob = 0;
    for (int q = 0; q < a.nrest; ++q) {
      const int64_t c = rem % a.rdim[q];
      rem /= a.rdim[q];
      ib += c * a.ris[q];
      ob += c * a.ros[q];
    }
    const int64_t x = bx * 256 + threadIdx.x;
    if (x < run) out[ob + x] = in[ib + x];
  }
}

// N[a + Ra*c, i, k, b + Sa*d] = sum_j A[a,i,j,b] * B[c,j,k,d]; one output
// element per thread (write-bound: 2J flops per 8-byte store), A and B
// cores are small and stay in L1/L2.
struct ProdArgs {
  const double* A;
  const double* B;
  double* N;
  int64_t Ra, I, J, Sa, Rb, K, Sb;
  int64_t aI, aJ, aS;  // element strides of A's logical axes i, j, b (a stride 1)
  int64_t bJ, bK, bS;  // element strides of B's logical axes j, k, d (c stride 1)
  int64_t total;
};

__global__ void core_product_kernel(ProdArgs p) {
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < p.total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    int64_t r = idx;
    const int64_t a = r % p.Ra; r /= p.Ra;
    const int64_t c = r % p.Rb; r /= p.Rb;
    const int64_t i = r % p.I; r /= p.I;
    const int64_t k = r % p.K; r /= p.K;
    const int64_t b = r % p.Sa; r /= p.Sa;
    const int64_t d = r;
    const double* pa = p.A + a + i * p.aI + b * p.aS;
    const double* pb = p.B + c + k * p.bK + d * p.bS;
    double s = 0.0;
    for (int64_t j = 0; j < p.J; ++j) s = fma(pa[j * p.aJ], pb[j * p.bJ], s);
    p.N[idx] = s;
  }
}

// deterministic sum of squares: per-block partials then one block
__global__ void sumsq_partial(const double* __restrict__ x, int64_t n, double* part) {
  __shared__ double sh[256];
  double s = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    s = fma(x[i], x[i], s);
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) part[blockIdx.x] = sh[0];
}

__global__ void sumsq_final(const double* part, int n, double* out) {
  __shared__ double sh[256];
  double s = 0.0;
  for (int i = threadIdx.x; i < n; i += blockDim.x) s += part[i];
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) *out = sqrt(sh[0]);
}

}  // namespace

void scale_matrix(cudaStream_t st, int64_t m, int64_t n, double alpha, double* C, int64_t ldc,
                  int64_t batch, int64_t sC) {
  if (m <= 0 || n <= 0 || batch <= 0 || alpha == 1.0) return;
  scale_kernel<<<grid_for(m * n * batch), 256, 0, st>>>(m, n, alpha, C, ldc, batch, sC);
  CK_LAUNCH();
  note_launch();
}

void copy_matrix(cudaStream_t st, int64_t m, int64_t n, const double* A, int64_t lda, double* B,
                 int64_t ldb) {
  if (m <= 0 || n <= 0) return;
  if (lda == m && ldb == m) {
    CK(cudaMemcpyAsync(B, A, sizeof(double) * m * n, cudaMemcpyDeviceToDevice, st));
    return;
  }
  copy_kernel<<<grid_for(m * n), 256, 0, st>>>(m, n, A, lda, B, ldb);
  CK_LAUNCH();
  note_launch();
}

void set_identity(cudaStream_t st, int64_t m, int64_t n, double* A, int64_t lda) {
  if (m <= 0 || n <= 0) return;
  identity_kernel<<<grid_for(m * n), 256, 0, st>>>(m, n, A, lda);
  CK_LAUNCH();
  note_launch();
}

void fill_zero(cudaStream_t st, double* p, int64_t n) {
  if (n > 0) CK(cudaMemsetAsync(p, 0, sizeof(double) * n, st));
}

void permute(cudaStream_t st, const double* in, double* out, int rank, const int64_t* dims,
             const int* perm) {
  if (rank < 1 || rank > 6) throw ValueError("permute rank must be 1..6");
  int64_t total = 1;
  for (int q = 0; q < rank; ++q) total *= dims[q];
  if (total == 0) return;
  // canonical form: drop unit axes, merge input axes k, k+1 that are also
  // consecutive in the output
  int64_t n[6];
  int p[6];        // output axis q <- canonical input axis p[q]
  int nr = 0;
  {
    int map[6];
    int64_t nd[6];
    int kept = 0;
    for (int k = 0; k < rank; ++k) {
      map[k] = -1;
      if (dims[k] != 1) { map[k] = kept; nd[kept++] = dims[k]; }
    }
    int op[6], no = 0;
    for (int q = 0; q < rank; ++q)
      if (map[perm[q]] >= 0) op[no++] = map[perm[q]];
    // merge: output-consecutive pairs (k, k+1) of input axes
    int grp[6];
    for (int k = 0; k < kept; ++k) grp[k] = k;
    for (int q = 0; q + 1 < no; ++q)
      if (op[q + 1] == op[q] + 1) grp[op[q + 1]] = grp[op[q]];
    int cid[6];
    for (int k = 0; k < kept; ++k) {
      if (grp[k] == k) { cid[k] = nr; n[nr++] = nd[k]; }
      else { cid[k] = cid[grp[k]]; n[cid[k]] *= nd[k]; }
    }
    int np = 0;
    for (int q = 0; q < no; ++q)
      if (grp[op[q]] == op[q]) p[np++] = cid[op[q]];
  }
  if (nr <= 1) {
    CK(cudaMemcpyAsync(out, in, sizeof(double) * total, cudaMemcpyDeviceToDevice, st));
    return;
  }
  int64_t is[6], os[6];
  {
    int64_t s = 1;
    for (int k = 0; k < nr; ++k) { is[k] = s; s *= n[k]; }
    s = 1;
    for (int q = 0; q < nr; ++q) { os[p[q]] = s; s *= n[p[q]]; }
  }
  auto launch_generic = [&]() {
    PermArgsG g{};
    g.rank = nr;
    g.total = total;
    for (int q = 0; q < 6; ++q) { g.odims[q] = 1; g.istride[q] = 0; }
    for (int q = 0; q < nr; ++q) { g.odims[q] = n[p[q]]; g.istride[q] = is[p[q]]; }
    permute_generic_kernel<<<(int)std::max<int64_t>(1, std::min<int64_t>(cdiv(total, 256), 148 * 16)),
                             256, 0, st>>>(in, out, g);
    CK_LAUNCH();
    note_launch();
  };
  PermArgs a{};
  bool used[6] = {false, false, false, false, false, false};
  auto rest_and_launch = [&](bool runs) {
    a.nrest = 0;
    a.ntiles = a.X.tiles * (runs ? 1 : a.Y.tiles);
    for (int k = 0; k < nr; ++k) {
      if (used[k]) continue;
      a.rdim[a.nrest] = n[k];
      a.ris[a.nrest] = is[k];
      a.ros[a.nrest] = os[k];
      a.ntiles *= n[k];
      ++a.nrest;
    }
    const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(a.ntiles, 148 * 16));
    if (runs) permute_runs_kernel<<<blocks, 256, 0, st>>>(in, out, a);
    else permute_tiled_kernel<<<blocks, 256, 0, st>>>(in, out, a);
    CK_LAUNCH();
    note_launch();
  };
  if (p[0] == 0) {
    // runs along the input-fastest axis
    if (n[0] < 64) { launch_generic(); return; }
    a.X.n1 = n[0];
    a.X.tiles = cdiv(n[0], 256);
    used[0] = true;
    rest_and_launch(true);
    return;
  }
  // X group: input axis 0 (+ axis 1 when axis 0 is short and axis 1 is not
  // the output-fastest axis)
  auto set_group = [&](PermAxis2& g, int k1, int k2, bool is_x) {
    g.n1 = n[k1];
    g.is1 = is[k1];
    g.os1 = os[k1];
    g.comp = k2 >= 0;
    used[k1] = true;
    if (g.comp) {
      g.n2 = n[k2];
      g.is2 = is[k2];
      g.os2 = os[k2];
      g.c2 = std::max<int64_t>(1, TP / g.n1);
      g.tiles = cdiv(g.n2, g.c2);
      used[k2] = true;
    } else {
      g.n2 = 1; g.c2 = 1; g.is2 = 0; g.os2 = 0;
      g.tiles = cdiv(g.n1, TP);
    }
    (void)is_x;
  };
  const int y1 = p[0];
  int x2 = -1, y2 = -1;
  if (n[0] < TP && nr > 2 && y1 != 1) x2 = 1;
  if (n[y1] < TP && nr > 2 && p[1] != 0 && p[1] != x2) y2 = p[1];
  set_group(a.X, 0, x2, true);
  set_group(a.Y, y1, y2, false);
  rest_and_launch(false);
}

void frob_norm(cudaStream_t st, const double* x, int64_t n, double* out_dev) {
  const int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(n, 256), 296));
  DBuf<double> part(blocks, st);
  sumsq_partial<<<blocks, 256, 0, st>>>(x, n, part.get());
  CK_LAUNCH();
  sumsq_final<<<1, 256, 0, st>>>(part.get(), blocks, out_dev);
  CK_LAUNCH();
  note_launch(2);
}

void core_product(cudaStream_t st, const CoreView& a, const CoreView& b, double* out) {
  if (a.J != b.I) throw ValueError("inner dims differ per core");
  ProdArgs p;
  p.A = a.p;
  p.B = b.p;
  p.N = out;
  p.Ra = a.R; p.I = a.I; p.J = a.J; p.Sa = a.S;
  p.Rb = b.R; p.K = b.J; p.Sb = b.S;
  // A physical (R, I, J, S) or (R, J, I, S) when transposed
  if (!a.trans) { p.aI = a.R; p.aJ = a.R * a.I; }
  else { p.aJ = a.R; p.aI = a.R * a.J; }
  p.aS = a.R * a.I * a.J;
  // B logical (Rb, J, K, Sb)
  if (!b.trans) { p.bJ = b.R; p.bK = b.R * b.I; }
  else { p.bK = b.R; p.bJ = b.R * b.J; }
  p.bS = b.R * b.I * b.J;
  p.total = p.Ra * p.Rb * p.I * p.K * p.Sa * p.Sb;
  if (p.total == 0) return;
  core_product_kernel<<<grid_for(p.total), 256, 0, st>>>(p);
  CK_LAUNCH();
  note_launch();
}

}  // namespace mpob

namespace mpob {
namespace {
__global__ void core0_finish_kernel(const double* in, int64_t I1, int64_t K, int64_t R2,
                                    int64_t kt, const double* sign, double* out) {
  const int64_t total = I1 * kt * R2;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    int64_t i = idx % I1, l = (idx / I1) % kt, r = idx / (I1 * kt);
    out[idx] = in[i + I1 * (l + K * r)] * sign[l];
  }
}
__global__ void axpy_kernel(int64_t n, double alpha, const double* x, double* y) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    y[i] += alpha * x[i];
}
__global__ void place_kernel(const double* in, int64_t Ri, int64_t M, int64_t Si, double* out,
                             int64_t Ro, int64_t So, int64_t ra, int64_t sb) {
  const int64_t total = Ri * M * Si;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    int64_t a = idx % Ri, m = (idx / Ri) % M, b = idx / (Ri * M);
    out[(a + ra) + Ro * (m + M * (b + sb))] = in[idx];
  }
}
}  // namespace

void dgemm_axpy(cudaStream_t st, int64_t n, double alpha, const double* x, double* y) {
  if (n <= 0) return;
  axpy_kernel<<<grid_for(n), 256, 0, st>>>(n, alpha, x, y);
  CK_LAUNCH();
  note_launch();
}

void place_block(cudaStream_t st, const double* in, int64_t Ri, int64_t M, int64_t Si, double* out,
                 int64_t Ro, int64_t So, int64_t ra, int64_t sb) {
  const int64_t total = Ri * M * Si;
  if (total <= 0) return;
  (void)So;
  place_kernel<<<grid_for(total), 256, 0, st>>>(in, Ri, M, Si, out, Ro, So, ra, sb);
  CK_LAUNCH();
  note_launch();
}

void core0_finish(cudaStream_t st, const double* in, int64_t I1, int64_t K, int64_t R2,
                  int64_t kt, const double* sign_dev, double* out) {
  const int64_t total = I1 * kt * R2;
  if (total <= 0) return;
  core0_finish_kernel<<<grid_for(total), 256, 0, st>>>(in, I1, K, R2, kt, sign_dev, out);
  CK_LAUNCH();
  note_launch();
}

SideStream& side_stream(cudaStream_t main) {
  // keyed by (device, main stream): the legacy/per-thread default stream has
  // the same handle on every device, and the side streams belong to one
  thread_local std::deque<SideStream> cache;   // deque: stable references
  const int dev = current_device();
  for (auto& x : cache)
    if (x.main == main && x.device == dev) return x;
  SideStream x;
  x.main = main;
  x.device = dev;
  CK(cudaStreamCreateWithFlags(&x.sv, cudaStreamNonBlocking));
  int lo = 0, hi = 0;
  CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
  CK(cudaStreamCreateWithPriority(&x.hp, cudaStreamNonBlocking, hi));
  CK(cudaStreamCreateWithPriority(&x.aux, cudaStreamNonBlocking, hi));
  CK(cudaStreamCreateWithFlags(&x.qs, cudaStreamNonBlocking));
  CK(cudaEventCreateWithFlags(&x.eqf, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&x.eq, cudaEventDisableTiming));
  for (auto& e : x.e) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  cache.push_back(x);
  return cache.back();
}

}  // namespace mpob

// FP64 GEMM on the sm_100a DMMA pipe (mma.sync m8n8k4 f64 -> SASS DMMA).
//
// C = alpha * op(A) * op(B) + beta * C, column-major, optional strided batch
// and deterministic split-K (partials reduced in a fixed order, no atomics,
// so repeated runs are bitwise identical -- SPEC.md:240 determinism).
// Used for every dense contraction of the sweeps: R-factor absorption
// (rsvd.py:108, :136), the blocked-Householder trailing updates that replace
// LAPACK dgeqrf/dorgqr (rsvd.py:106, :132, :160), the Jacobi SVD's Q*V
// back-transform (rsvd.py:128) and the leading-core merge (rsvd.py:95).
#include <algorithm>
#include <cstdlib>
#include <map>
#include <mutex>
#include <string>
#include <tuple>

#include "common.cuh"
#include "kernels.cuh"

namespace mpob {

namespace {

constexpr int BM = 64, BN = 64, BK = 16, PAD = 4, THREADS = 128;
constexpr int LDS = BM + PAD;  // 68 doubles: conflict-free fragment reads

__device__ __forceinline__ void dmma_8x8x4(double (&c)[2], double a, double b) {
  asm volatile(
      "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 "
      "{%0, %1}, {%2}, {%3}, {%0, %1};\n"
      : "+d"(c[0]), "+d"(c[1])
      : "d"(a), "d"(b));
}

struct GemmArgs {
  int64_t m, n, k;
  const double* A;
  int64_t lda, sA;
  const double* B;
  int64_t ldb, sB;
  double* C;
  int64_t ldc, sC;
  double alpha, beta;
  int ta, tb;
  int64_t kchunk;   // K range per split
  double* work;     // split-K partials (nsplit * batch * m * n) or null
};

template <int TA, int TB>
__global__ void __launch_bounds__(THREADS) dgemm_kernel(GemmArgs g) {
  __shared__ double As[2][BK][LDS];
  __shared__ double Bs[2][BK][LDS];

  const int64_t tiles_m = cdiv_dev(g.m, BM);
  const int64_t tm = blockIdx.x % tiles_m, tn = blockIdx.x / tiles_m;
  const int split = blockIdx.y;
  const int64_t bat = blockIdx.z;
  const int64_t m0 = tm * BM, n0 = tn * BN;
  const int64_t kb = split * g.kchunk;
  const int64_t ke = min(g.k, kb + g.kchunk);
  const double* A = g.A + bat * g.sA;
  const double* B = g.B + bat * g.sB;

  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int wm = warp & 1, wn = warp >> 1;

  double ra[8], rb[8];
  auto load_tile = [&](int64_t k0) {
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      int i, kk;
      if (!TA) { i = t & 63; kk = (t >> 6) + 2 * r; } else { kk = t & 15; i = (t >> 4) + 8 * r; }
      int64_t gi = m0 + i, gk = k0 + kk;
      double v = 0.0;
      if (gi < g.m && gk < ke) v = TA ? A[gk + gi * g.lda] : A[gi + gk * g.lda];
      ra[r] = v;
    }
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      int j, kk;
      if (!TB) { kk = t & 15; j = (t >> 4) + 8 * r; } else { j = t & 63; kk = (t >> 6) + 2 * r; }
      int64_t gj = n0 + j, gk = k0 + kk;
      double v = 0.0;
      if (gj < g.n && gk < ke) v = TB ? B[gj + gk * g.ldb] : B[gk + gj * g.ldb];
      rb[r] = v;
    }
  };
  auto store_tile = [&](int buf) {
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      int i, kk;
      if (!TA) { i = t & 63; kk = (t >> 6) + 2 * r; } else { kk = t & 15; i = (t >> 4) + 8 * r; }
      As[buf][kk][i] = ra[r];
    }
#pragma unroll
    for (int r = 0; r < 8; ++r) {
      int j, kk;
      if (!TB) { kk = t & 15; j = (t >> 4) + 8 * r; } else { j = t & 63; kk = (t >> 6) + 2 * r; }
      Bs[buf][kk][j] = rb[r];
    }
  };

  double acc[4][4][2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;

  int buf = 0;
  if (kb < ke) {
    load_tile(kb);
    store_tile(0);
  }
  __syncthreads();
  for (int64_t k0 = kb; k0 < ke; k0 += BK) {
    const bool more = k0 + BK < ke;
    if (more) load_tile(k0 + BK);
#pragma unroll
    for (int k4 = 0; k4 < BK / 4; ++k4) {
      double af[4], bf[4];
      const int kr = k4 * 4 + (lane & 3);
#pragma unroll
      for (int mi = 0; mi < 4; ++mi) af[mi] = As[buf][kr][wm * 32 + mi * 8 + (lane >> 2)];
#pragma unroll
      for (int ni = 0; ni < 4; ++ni) bf[ni] = Bs[buf][kr][wn * 32 + ni * 8 + (lane >> 2)];
#pragma unroll
      for (int mi = 0; mi < 4; ++mi)
#pragma unroll
        for (int ni = 0; ni < 4; ++ni) dmma_8x8x4(acc[mi][ni], af[mi], bf[ni]);
    }
    if (more) {
      store_tile(buf ^ 1);
      __syncthreads();
      buf ^= 1;
    }
  }

  // epilogue
  const int row = lane >> 2, col = (lane & 3) * 2;
  if (g.work) {
    double* W = g.work + ((int64_t)split * gridDim.z + bat) * g.m * g.n;
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
      for (int ni = 0; ni < 4; ++ni)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          int64_t gi = m0 + wm * 32 + mi * 8 + row, gj = n0 + wn * 32 + ni * 8 + col + e;
          if (gi < g.m && gj < g.n) W[gi + gj * g.m] = acc[mi][ni][e];
        }
    return;
  }
  double* C = g.C + bat * g.sC;
  // all C reads are issued before any C write (the compiler cannot prove the
  // addresses distinct, so an interleaved read-modify-write would serialise
  // on the full memory latency of every element)
  if (g.beta != 0.0) {
    double old[4][4][2];
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
      for (int ni = 0; ni < 4; ++ni)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          int64_t gi = m0 + wm * 32 + mi * 8 + row, gj = n0 + wn * 32 + ni * 8 + col + e;
          old[mi][ni][e] = (gi < g.m && gj < g.n) ? __ldcg(C + gi + gj * g.ldc) : 0.0;
        }
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
      for (int ni = 0; ni < 4; ++ni)
#pragma unroll
        for (int e = 0; e < 2; ++e) acc[mi][ni][e] = g.alpha * acc[mi][ni][e] + g.beta * old[mi][ni][e];
  } else {
#pragma unroll
    for (int mi = 0; mi < 4; ++mi)
#pragma unroll
      for (int ni = 0; ni < 4; ++ni)
#pragma unroll
        for (int e = 0; e < 2; ++e) acc[mi][ni][e] *= g.alpha;
  }
#pragma unroll
  for (int mi = 0; mi < 4; ++mi)
#pragma unroll
    for (int ni = 0; ni < 4; ++ni)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        int64_t gi = m0 + wm * 32 + mi * 8 + row, gj = n0 + wn * 32 + ni * 8 + col + e;
        if (gi < g.m && gj < g.n) C[gi + gj * g.ldc] = acc[mi][ni][e];
      }
}

__global__ void splitk_reduce(const double* __restrict__ W, int nsplit, int64_t batch, int64_t m,
                              int64_t n, double alpha, double beta, double* C, int64_t ldc,
                              int64_t sC) {
  const int64_t total = batch * m * n;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    int64_t b = idx / (m * n), r = idx % (m * n);
    int64_t i = r % m, j = r / m;
    double s = 0.0;
    for (int p = 0; p < nsplit; ++p) s += W[((int64_t)p * batch + b) * m * n + r];
    double* c = C + b * sC + i + j * ldc;
    double v = alpha * s;
    if (beta != 0.0) v += beta * *c;
    *c = v;
  }
}

}  // namespace

namespace {
// MPO_B200_GEMM_STATS=1: per-shape call counts and flops, printed at exit
// (diagnostics: which GEMM shapes the sweeps spend their DGEMM time on)
struct GemmStats {
  std::mutex mu;
  // (m, n, k, batch, ta, tb) -> (calls, device ms: each call timed with events)
  std::map<std::tuple<int64_t, int64_t, int64_t, int64_t, int, int>, std::pair<int64_t, double>>
      calls;
  ~GemmStats() {
    if (calls.empty()) return;
    std::vector<std::pair<double, std::string>> rows;
    double tot = 0.0, small = 0.0;
    for (auto& kv : calls) {
      auto [m, n, k, b, ta, tb] = kv.first;
      const double f = 2.0 * m * n * k * b * kv.second.first, ms = kv.second.second;
      tot += ms;
      if (f / kv.second.first < 2e9) small += ms;
      char buf[200];
      snprintf(buf, sizeof(buf),
               "gemm %c%c m=%lld n=%lld k=%lld batch=%lld calls=%lld gflop=%.2f ms=%.3f tflops=%.1f",
               ta ? 'T' : 'N', tb ? 'T' : 'N', (long long)m, (long long)n, (long long)k,
               (long long)b, (long long)kv.second.first, f / 1e9, ms, ms > 0 ? f / ms / 1e9 : 0.0);
      rows.emplace_back(ms, buf);
    }
    std::sort(rows.begin(), rows.end(), [](auto& x, auto& y) { return x.first > y.first; });
    fprintf(stderr, "[mpo_b200] gemm total %.1f ms over %zu shapes; calls under 2 GFLOP: %.1f ms\n",
            tot, calls.size(), small);
    for (size_t i = 0; i < rows.size() && i < 60; ++i) fprintf(stderr, "[mpo_b200] %s\n", rows[i].second.c_str());
  }
};

GemmStats& gemm_stats() {
  static GemmStats g;
  return g;
}
}  // namespace

void dgemm(cudaStream_t st, bool ta, bool tb, int64_t m, int64_t n, int64_t k, double alpha,
           const double* A, int64_t lda, const double* B, int64_t ldb, double beta, double* C,
           int64_t ldc, int64_t batch, int64_t sA, int64_t sB, int64_t sC) {
  if (m <= 0 || n <= 0 || batch <= 0) return;
  static const bool stats = std::getenv("MPO_B200_GEMM_STATS") != nullptr;
  struct StatTimer {   // MPO_B200_GEMM_STATS: per-shape call count and device time
    bool on;
    cudaStream_t st;
    std::tuple<int64_t, int64_t, int64_t, int64_t, int, int> key;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    ~StatTimer() {
      if (!on) return;
      cudaEventRecord(e1, st);
      cudaEventSynchronize(e1);
      float ms = 0.0f;
      cudaEventElapsedTime(&ms, e0, e1);
      cudaEventDestroy(e0);
      cudaEventDestroy(e1);
      std::lock_guard<std::mutex> lk(gemm_stats().mu);
      auto& v = gemm_stats().calls[key];
      v.first += 1;
      v.second += ms;
    }
  } stat{stats, st, {m, n, k, batch, (int)ta, (int)tb}};
  if (stats) {
    CK(cudaEventCreate(&stat.e0));
    CK(cudaEventCreate(&stat.e1));
    CK(cudaEventRecord(stat.e0, st));
  }
  if (k <= 0) {
    scale_matrix(st, m, n, beta, C, ldc, batch, sC);
    return;
  }
  ProfScope prof(st, 3, 2.0 * (double)m * n * k * batch);
  GemmArgs g{m, n, k, A, lda, sA, B, ldb, sB, C, ldc, sC, alpha, beta, ta, tb, k, nullptr};
  const int64_t tiles = cdiv(m, BM) * cdiv(n, BN);
  // split-K when the output grid cannot fill the 148 SMs and K is long
  int nsplit = 1;
  const int64_t ctas = tiles * batch;
  if (ctas < 148 && k >= 512) {
    nsplit = (int)std::min<int64_t>(std::max<int64_t>(1, 296 / ctas), k / 256);
    nsplit = std::max(1, std::min(nsplit, 64));
  }
  DBuf<double> work;
  if (nsplit > 1) {
    g.kchunk = cdiv(cdiv(k, nsplit), BK) * BK;
    nsplit = (int)cdiv(k, g.kchunk);
  }
  if (nsplit > 1) {
    work.alloc((size_t)nsplit * batch * m * n, st);
    g.work = work.get();
  }
  if (batch > 65535) throw ValueError("gemm batch too large");
  dim3 grid((unsigned)tiles, (unsigned)nsplit, (unsigned)batch);
  if (!ta && !tb) dgemm_kernel<0, 0><<<grid, THREADS, 0, st>>>(g);
  else if (!ta && tb) dgemm_kernel<0, 1><<<grid, THREADS, 0, st>>>(g);
  else if (ta && !tb) dgemm_kernel<1, 0><<<grid, THREADS, 0, st>>>(g);
  else dgemm_kernel<1, 1><<<grid, THREADS, 0, st>>>(g);
  CK_LAUNCH();
  note_launch();
  if (nsplit > 1) {
    int64_t total = batch * m * n;
    int blocks = (int)std::min<int64_t>(cdiv(total, 256), 148 * 8);
    splitk_reduce<<<blocks, 256, 0, st>>>(work.get(), nsplit, batch, m, n, alpha, beta, C, ldc, sC);
    CK_LAUNCH();
    note_launch();
  }
}

}  // namespace mpob

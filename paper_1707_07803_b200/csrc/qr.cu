// Blocked Householder QR on sm_100a, replacing LAPACK dgeqrf + dorgqr behind
// np.linalg.qr(mode="reduced") at rsvd.py:106 (left-to-right sweep),
// rsvd.py:132 (exact RQ sweep) and rsvd.py:160 (first-core QR).
//
// Panel factorisation: one cooperative kernel per nb-column panel.  The
// panel's rows are split over up to 148 co-resident CTAs, each keeping its
// row chunk in shared memory; every column needs two grid-wide reductions
// (norm, then v^T A_panel), done as per-CTA partials summed in a fixed order
// (deterministic, no atomics).  The kernel also forms the compact-WY factor
// T (LAPACK dlarft) from V^T V.  Trailing updates and the explicit Q
// (dorgqr) are DMMA GEMMs (gemm.cu).  Householder convention as dlarfg:
// beta = -sign(alpha) * ||x||, tau = (beta - alpha) / beta.
#include <cooperative_groups.h>
#include <cstdlib>

#include "common.cuh"
#include "kernels.cuh"

namespace cg = cooperative_groups;

namespace mpob {

namespace {

constexpr int QR_NB = 32;
constexpr int QR_THREADS = 256;

struct PanelArgs {
  double* A;       // panel top-left (row j0, col j0)
  int64_t lda;
  int64_t mp;      // panel height (m - j0)
  int w;           // panel width
  int rpc;         // rows per CTA
  double* V;       // mp x w explicit reflectors (unit diagonal, zeros above)
  int64_t ldv;
  double* T;       // w x w compact-WY factor (column-major)
  double* tau;     // w
  double* part;    // G partial norms
  double* wpart;   // G x w partial v^T A
  double* vtv;     // G x w x w partial V^T V
  double* alpha;   // 1 slot (diagonal element of the current column)
};

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// dlarft (forward, columnwise) in shared memory, one column per step with
// the i < j entries in parallel: T(0:j, j) = -tau_j T(0:j,0:j) S(0:j, j),
// S = V^T V (strict upper part used).  Writes T (w x w, column-major) and
// tau to global memory.  Called by all threads of one CTA.
//
// Formulated column-parallel: for true reflectors (tau_j = 2 / v_j^T v_j)
// T^{-1} = diag(1/tau) + striu(V^T V), so column i of T is the
// back-substitution x_i = tau_i, x_r = -tau_r sum_{l=r+1..i} S(r,l) x_l
// (r = i-1 .. 0) -- one thread per column, no barriers between steps; a
// tau_r = 0 (H_r = I) zeroes row and column r exactly as the recurrence does.
__device__ void build_t_factor(const double* S, double* sT, const double* tau_in, int w,
                               double* T, double* tau_out) {
  const int t = threadIdx.x;
  if (t < w) {
    const int i = t;
    double* x = sT + i * w;
    for (int r = i + 1; r < w; ++r) x[r] = 0.0;
    x[i] = tau_in[i];
    for (int r = i - 1; r >= 0; --r) {
      double acc = 0.0;
      for (int l = r + 1; l <= i; ++l) acc = fma(S[r + l * w], x[l], acc);
      x[r] = -tau_in[r] * acc;
    }
  }
  __syncthreads();
  for (int idx = t; idx < w * w; idx += blockDim.x) T[idx] = sT[idx];
  for (int idx = t; idx < w; idx += blockDim.x) tau_out[idx] = tau_in[idx];
}

__device__ __forceinline__ void dmma884(double (&c)[2], double a, double b) {
  asm volatile(
      "mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 "
      "{%0, %1}, {%2}, {%3}, {%0, %1};\n"
      : "+d"(c[0]), "+d"(c[1])
      : "d"(a), "d"(b));
}

// out[a + b*w] = sum_r V[r][a] V[r][b] for a < b (else 0) over this CTA's nr
// rows of the explicit reflectors held column-major in smem (ld rows).  On
// the DMMA pipe: 16 8x8 tiles, two per warp, K = rows in steps of 4.
__device__ void vtv_partial_dmma(const double* V, int ld, int nr, int w, double* out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int ti = warp >> 1, tj0 = (warp & 1) * 2;
  double acc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
  const int ia = ti * 8 + (lane >> 2);
  for (int k0 = 0; k0 < nr; k0 += 4) {
    const int kk = k0 + (lane & 3);
    const bool kin = kk < nr;
    const double av = (kin && ia < w) ? V[kk + ia * ld] : 0.0;
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int jb = (tj0 + u) * 8 + (lane >> 2);
      const double bv = (kin && jb < w) ? V[kk + jb * ld] : 0.0;
      dmma884(acc[u], av, bv);
    }
  }
#pragma unroll
  for (int u = 0; u < 2; ++u)
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int b = (tj0 + u) * 8 + 2 * (lane & 3) + e;
      if (ia < w && b < w) out[ia + b * w] = ia < b ? acc[u][e] : 0.0;
    }
}

__global__ void __launch_bounds__(QR_THREADS) qr_panel_kernel(PanelArgs p) {
  extern __shared__ double chunk[];  // rpc x w, column-major: chunk[r + col*ld]
  __shared__ double red[QR_THREADS / 32];
  __shared__ double s_scal, s_tau, s_beta;
  __shared__ double s_w[QR_NB];
  cg::grid_group grid = cg::this_grid();
  const int G = gridDim.x, c = blockIdx.x, t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int w = p.w;
  const int64_t r0 = (int64_t)c * p.rpc;
  const int64_t rem = p.mp - r0;
  const int nr = rem <= 0 ? 0 : (int)(rem < p.rpc ? rem : p.rpc);

  const int ld = p.rpc;
  for (int idx = t; idx < nr * w; idx += QR_THREADS) {
    int r = idx % nr, col = idx / nr;
    chunk[r + col * ld] = p.A[(r0 + r) + col * p.lda];
  }
  __syncthreads();

  for (int jj = 0; jj < w; ++jj) {
    // phase 1: partial ||x||^2 strictly below the diagonal
    double s = 0.0;
    for (int r = t; r < nr; r += QR_THREADS) {
      int64_t gr = r0 + r;
      if (gr > jj) { double x = chunk[r + jj * ld]; s = fma(x, x, s); }
      if (gr == jj) *p.alpha = chunk[r + jj * ld];
    }
    s = warp_sum(s);
    if (lane == 0) red[warp] = s;
    __syncthreads();
    if (t == 0) {
      double tot = 0.0;
      for (int i = 0; i < QR_THREADS / 32; ++i) tot += red[i];
      p.part[c] = tot;
    }
    __threadfence();
    grid.sync();
    // phase 2: reflector (every CTA computes the same scalars)
    if (t == 0) {
      double sig = 0.0;
      for (int i = 0; i < G; ++i) sig += p.part[i];
      double al = *p.alpha;
      double tau = 0.0, beta = al, scal = 0.0;
      if (sig != 0.0) {
        double nrm = sqrt(fma(al, al, sig));
        beta = al >= 0.0 ? -nrm : nrm;
        tau = (beta - al) / beta;
        scal = 1.0 / (al - beta);
      }
      s_tau = tau; s_beta = beta; s_scal = scal;
      if (c == 0) p.tau[jj] = tau;
    }
    __syncthreads();
    const double tau = s_tau, scal = s_scal;
    for (int r = t; r < nr; r += QR_THREADS) {
      int64_t gr = r0 + r;
      if (gr > jj) chunk[r + jj * ld] *= scal;
    }
    __syncthreads();
    // partial w_t = sum_r v_r A[r, jj+1+t] over r >= jj (v_jj = 1)
    const int ncols = w - jj - 1;
    for (int col = warp; col < ncols; col += QR_THREADS / 32) {
      double acc = 0.0;
      for (int r = lane; r < nr; r += 32) {
        int64_t gr = r0 + r;
        if (gr >= jj) {
          double v = (gr == jj) ? 1.0 : chunk[r + jj * ld];
          acc = fma(v, chunk[r + (jj + 1 + col) * ld], acc);
        }
      }
      acc = warp_sum(acc);
      if (lane == 0) p.wpart[(int64_t)c * w + col] = acc;
    }
    __threadfence();
    grid.sync();
    if (ncols > 0) {
      for (int col = t; col < ncols; col += QR_THREADS) {
        double tot = 0.0;
        for (int i = 0; i < G; ++i) tot += p.wpart[(int64_t)i * w + col];
        s_w[col] = tot * tau;
      }
      __syncthreads();
      // rank-1 update of the remaining panel columns (no integer division:
      // each thread keeps its rows and walks the columns)
      for (int r = t; r < nr; r += QR_THREADS) {
        const int64_t gr = r0 + r;
        if (gr < jj) continue;
        const double v = (gr == jj) ? 1.0 : chunk[r + jj * ld];
        double* rowp = chunk + r + (jj + 1) * ld;
        for (int col = 0; col < ncols; ++col) rowp[col * ld] -= v * s_w[col];
      }
    }
    // diagonal of R
    for (int r = t; r < nr; r += QR_THREADS)
      if (r0 + r == jj) chunk[r + jj * ld] = s_beta;
    __syncthreads();
  }

  // write back R / V parts; explicit V with unit diagonal; partial V^T V
  for (int idx = t; idx < nr * w; idx += QR_THREADS) {
    int r = idx % nr, col = idx / nr;
    int64_t gr = r0 + r;
    double x = chunk[r + col * ld];
    p.A[gr + col * p.lda] = x;
    double v = gr > col ? x : (gr == col ? 1.0 : 0.0);
    p.V[gr + (int64_t)col * p.ldv] = v;
    chunk[r + col * ld] = v;
  }
  __syncthreads();
  vtv_partial_dmma(chunk, ld, nr, w, p.vtv + (int64_t)c * w * w);
  __threadfence();
  grid.sync();
  if (c == 0) {
    // dlarft (forward, columnwise): T(0:j, j) = -tau_j T(0:j,0:j) V(:,0:j)^T v_j
    __shared__ double sv[QR_NB * QR_NB];
    __shared__ double st_[QR_NB * QR_NB];
    __shared__ double stau[QR_NB];
    for (int idx = t; idx < w * w; idx += QR_THREADS) {
      double tot = 0.0;
      for (int i = 0; i < G; ++i) tot += p.vtv[(int64_t)i * w * w + idx];
      sv[idx] = tot;  // sv[a + b*w] = v_a . v_b (a < b)
    }
    for (int idx = t; idx < w; idx += QR_THREADS) stau[idx] = p.tau[idx];
    __syncthreads();
    build_t_factor(sv, st_, stau, w, p.T, p.tau);
  }
}

// Cluster variant of the panel factorisation: the panel's rows are split
// over the CTAs of ONE thread-block cluster (<= 16 SMs); the two reductions
// per column go through distributed shared memory and cluster barriers
// (~0.2 us) instead of global memory and grid-wide barriers.
struct ClusterPanelArgs {
  double* A;
  int64_t lda;
  int64_t mp;
  int w;
  int rpc;
  int ld;          // shared-memory leading dimension (cluster_panel_ld)
  double* V;
  int64_t ldv;
  double* T;
  double* tau;
};

// cluster panel threads: 16 warps; the dot phase splits each 4-column group's
// rows over QRC / 256 warps, the rank-1 update gives every thread <= 1 row of
// a 512-row CTA slice
constexpr int QRC = 512;
constexpr int QRC_H = QRC / 256;   // row halves per column group in the dot phase

// Remote shared-memory stores that signal the destination CTA's mbarrier
// (st.async ... mbarrier::complete_tx): the per-column exchange needs no
// fence -- cluster.sync()'s release is a MEMBAR.ALL.GPU per warp, which was
// 40 % of the panel's stall samples (profiles/r02_panel_membar.txt).
__device__ __forceinline__ uint32_t smem_addr(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ uint32_t cluster_addr(uint32_t local, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local), "r"(rank));
  return r;
}
__device__ __forceinline__ void st_async_2f64(uint32_t dst, double a, double b, uint32_t mbar) {
  asm volatile(
      "st.async.weak.shared::cluster.mbarrier::complete_tx::bytes.v2.b64 [%0], {%1, %2}, [%3];"
      ::"r"(dst), "l"(__double_as_longlong(a)), "l"(__double_as_longlong(b)), "r"(mbar)
      : "memory");
}
__device__ __forceinline__ void mbar_init(uint32_t mbar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(mbar), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint32_t mbar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mbar), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint32_t mbar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_LOOP:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@p bra WAIT_DONE;\n"
      "bra WAIT_LOOP;\n"
      "WAIT_DONE:\n"
      "}\n" ::"r"(mbar), "r"(parity)
      : "memory");
}

// -DMPO_QR_PROF: clock64 phase totals of cluster rank 0's thread 0, printed per launch
#ifdef MPO_QR_PROF
#define QPROF(i) do { if (t == 0 && c == 0) { long long now_ = clock64(); pacc[i] += now_ - plast; plast = now_; } } while (0)
#else
#define QPROF(i) do { } while (0)
#endif

// T = (diag(1/tau) + striu(S))^{-1} by one warp, lane i owning column i in
// registers: x_i = tau_i, x_r = -tau_r sum_{l=r+1..i} S(r,l) x_l (r = i-1..0)
// run in lockstep over r = 31..0 with x_l = 0 for l > i (dlarft, forward
// columnwise; a tau_r = 0 zeroes row and column r as the recurrence does).
// S is 32 x 32 (ld 32), zero outside the strict upper w x w part.
__device__ void build_t_factor_warp(const double* S, const double* tau_in, int w, double* T,
                                    double* tau_out) {
  const int lane = threadIdx.x & 31;
  double x[QR_NB];
#pragma unroll
  for (int r = QR_NB - 1; r >= 0; --r) {
    double a0 = 0.0, a1 = 0.0, a2 = 0.0, a3 = 0.0;
#pragma unroll
    for (int l = r + 1; l < QR_NB; ++l) {
      const double sv = S[r + l * QR_NB];
      if (((l - r - 1) & 3) == 0) a0 = fma(sv, x[l], a0);
      else if (((l - r - 1) & 3) == 1) a1 = fma(sv, x[l], a1);
      else if (((l - r - 1) & 3) == 2) a2 = fma(sv, x[l], a2);
      else a3 = fma(sv, x[l], a3);
    }
    const double tr = r < w ? tau_in[r] : 0.0;
    x[r] = r == lane ? tr : (r < lane ? -tr * ((a0 + a1) + (a2 + a3)) : 0.0);
  }
  if (lane < w) {
#pragma unroll
    for (int r = 0; r < QR_NB; ++r)
      if (r < w) T[r + lane * w] = x[r];
    tau_out[lane] = tau_in[lane];
  }
}

// (A three-stage blocked variant on the whole CTA measured 3.4K instead of
// 8.8K cycles under the clock64 profile but made every panel launch 7 us
// longer in the regular build; not kept.)
// out (32 x 32, ld 32) = strict upper part of V^T V over this CTA's nr rows,
// V = the explicit reflectors (unit diagonal, zeros above) held column-major
// in smem (ld rows); zero elsewhere.  DMMA: warp (ti, tj) of 4 x 4 owns one
// 8x8 tile (the 10 with ti <= tj compute), K = rows in steps of 4 on two
// accumulators.  Called by all 16 warps.
__device__ void vtv_partial_dmma32(const double* V, int ld, int nr, int w, double* out) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int ti = warp >> 2, tj = warp & 3;
  double acc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
  const int ia = ti * 8 + (lane >> 2), jb = tj * 8 + (lane >> 2);
  if (ti <= tj && ti * 8 < w && tj * 8 < w) {
    const double* pa = V + (lane & 3) + ia * ld;
    const double* pb = V + (lane & 3) + jb * ld;
    const bool ain = ia < w, bin = jb < w;
    for (int k0 = 0; k0 < nr; k0 += 8) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int kk = k0 + 4 * h + (lane & 3);
        const bool kin = kk < nr;
        const double av = (kin && ain) ? pa[k0 + 4 * h] : 0.0;
        const double bv = (kin && bin) ? pb[k0 + 4 * h] : 0.0;
        dmma884(acc[h], av, bv);
      }
    }
  }
#pragma unroll
  for (int e = 0; e < 2; ++e) {
    const int b = tj * 8 + 2 * (lane & 3) + e;
    out[ia + b * QR_NB] = (ia < w && b < w && ia < b) ? acc[0][e] + acc[1][e] : 0.0;
  }
}

__global__ void __launch_bounds__(QRC) qr_panel_cluster_kernel(ClusterPanelArgs p) {
  extern __shared__ double chunk[];  // rpc x w, column-major
  __shared__ double s_w[QR_NB];
  __shared__ double s_vtv[QR_NB * QR_NB];
  __shared__ double s_tau[QR_NB], s_scal[QR_NB], s_beta[QR_NB];
  // per-rank partials by column parity: [parity][rank][column][dot, row-jj entry]
  __shared__ __align__(16) double s_red[2][16 * QR_NB * 2];
  __shared__ double s_dpart[QRC_H][QR_NB];
  __shared__ __align__(8) unsigned long long s_mbar[2];
  cg::cluster_group cluster = cg::this_cluster();
  const int CS = (int)cluster.num_blocks(), c = (int)cluster.block_rank();
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int w = p.w, ld = p.ld;
  const int64_t r0 = (int64_t)c * p.rpc;
  const int64_t rem = p.mp - r0;
  const int nr = rem <= 0 ? 0 : (int)(rem < p.rpc ? rem : p.rpc);
  if (t == 0) {
    mbar_init(smem_addr(&s_mbar[0]), 1);
    mbar_init(smem_addr(&s_mbar[1]), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  for (int col = warp; col < w; col += QRC / 32)
    for (int r = lane; r < nr; r += 32) chunk[r + col * ld] = p.A[(r0 + r) + col * p.lda];
  // remote addresses of this rank's slot in rank `warp`'s buffers / mbarriers
  uint32_t rem_red[2] = {0, 0}, rem_mb[2] = {0, 0};
  if (warp < CS) {
#pragma unroll
    for (int b = 0; b < 2; ++b) {
      rem_red[b] = cluster_addr(smem_addr(&s_red[b][(c * QR_NB + lane) * 2]), warp);
      rem_mb[b] = cluster_addr(smem_addr(&s_mbar[b]), warp);
    }
  }
  cluster.sync();   // every rank's mbarriers are initialised before the first remote store
#ifdef MPO_QR_PROF
  long long pacc[16] = {0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0, 0}, plast = clock64(), pstart = plast;
#endif
  // One exchange per column: the norm of column jj and the dots x^T a_c of
  // its sub-diagonal part with every later panel column are reduced together
  // (plus the owner's row-jj entries), since with v = [1; scal x] the
  // reflector's w_c = tau (a_jj,c + scal x^T a_c).  Warp rk of every rank
  // stores the rank's partials into slot c of rank rk's buffer with st.async,
  // which counts the bytes on rank rk's mbarrier; a rank waits on its own
  // mbarrier only.  Buffers and mbarriers alternate by column parity: rank B's
  // buffer jj&1 is rewritten for column jj+2 by a rank A that has received
  // B's column-(jj+1) partials, which B sent after it finished reading
  // column jj's.  Column jj stays unscaled in shared memory (x, and a_jj on
  // the diagonal); scal and beta are applied at the write-back.
  //
  // One pass over the slice per column: warp (grp, half) owns 4 columns and
  // half of the rows; it applies reflector jj to its columns (and, redundantly,
  // to the next pivot column p = jj + 1) and accumulates the dots of the
  // updated pivot column with its updated columns for the next exchange.
  const int grp = warp % 8, half = warp / 8, col0 = grp * 4;
  double* piv = chunk + (size_t)ld * w;   // [2][ld]: the current pivot column, by parity
  for (int jj = -1; jj < w; ++jj) {
    const int pv = jj + 1;               // pivot whose dots this pass produces
    const int ncp = w - pv;              // columns pv .. w-1 (slot 0: its norm)
    if (jj >= 0) {
      const int ncols = w - jj;          // slot 0: column jj itself (its norm)
      const bool owner = jj >= r0 && jj < r0 + nr;
      const uint32_t mb = smem_addr(&s_mbar[jj & 1]);
      if (t == 0) mbar_expect_tx(mb, (uint32_t)(CS * ncols * 16));
      QPROF(0);
      __syncthreads();
      QPROF(1);
      if (warp < CS && lane < ncols) {
        double d = 0.0;
#pragma unroll
        for (int h = 0; h < QRC_H; ++h) d += s_dpart[h][lane];
        const double rowv = !owner ? 0.0 : (lane == 0 ? piv[(jj & 1) * ld + (jj - r0)]
                                                      : chunk[(jj - r0) + (jj + lane) * ld]);
        st_async_2f64((jj & 1) ? rem_red[1] : rem_red[0], d, rowv, (jj & 1) ? rem_mb[1] : rem_mb[0]);
      }
      QPROF(2);
      if (warp == 0) {
        // one warp derives the reflector: lane u sums column u's partials in a
        // fixed (pairwise, rank-ordered) tree, lane 0's are the norm and a_jj
        mbar_wait(mb, (jj >> 1) & 1);
        QPROF(3);
        const double* red = s_red[jj & 1] + lane * 2;
        double2 v[16];
#pragma unroll
        for (int i = 0; i < 16; ++i)
          v[i] = i < CS ? *reinterpret_cast<const double2*>(red + i * QR_NB * 2) : make_double2(0.0, 0.0);
#pragma unroll
        for (int s = 1; s < 16; s <<= 1)
#pragma unroll
          for (int i = 0; i < 16; i += 2 * s) { v[i].x += v[i + s].x; v[i].y += v[i + s].y; }
        const double dt = v[0].x, rt = v[0].y;
        const double sig = __shfl_sync(0xffffffffu, dt, 0), al = __shfl_sync(0xffffffffu, rt, 0);
        double tau = 0.0, beta = al, scal = 0.0;
        if (sig != 0.0) {
          const double nrm = sqrt(fma(al, al, sig));
          beta = al >= 0.0 ? -nrm : nrm;
          tau = (beta - al) / beta;
          scal = 1.0 / (al - beta);
        }
        if (lane == 0) { s_tau[jj] = tau; s_scal[jj] = scal; s_beta[jj] = beta; }
        else if (lane < ncols) s_w[lane] = tau * fma(scal, dt, rt);
      }
      QPROF(4);
      __syncthreads();
      QPROF(5);
    }
    if (ncp > 0 && col0 < ncp) {
      // reflector jj (none for jj = -1): v = [1; scal x], w as s_w.  The
      // updated pivot column goes to piv[pv & 1] (rows >= jj), not in place:
      // every group reads its old values in this pass.  Group 0 moves column
      // jj from piv[jj & 1] to its final home in the slice as it reads it.
      const bool refl = jj >= 0, g0 = col0 == 0;
      const double scal = refl ? s_scal[jj] : 0.0;
      const double wp = refl ? s_w[1] : 0.0;
      const int nu = min(4, ncp - col0);   // this group's live columns
      double wu[4], acc[4] = {0.0, 0.0, 0.0, 0.0};
      double* cp[4];                       // dead columns alias the last live one (loads only)
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        wu[u] = (refl && u < nu) ? s_w[1 + col0 + u] : 0.0;
        cp[u] = chunk + (pv + col0 + min(u, nu - 1)) * ld;
      }
      const double* xj = piv + (jj & 1) * ld;
      double* xhome = chunk + (refl ? jj : 0) * ld;
      double* ynew = piv + (pv & 1) * ld;
      const double* yp = chunk + pv * ld;
      // two 32-row blocks per trip, every load ahead of the arithmetic and
      // the stores (the compiler cannot hoist loads over the stores itself).
      // Blocks that are full and entirely below row pv (all but the slice's
      // last block and cluster rank 0's first) take a predicate-free path:
      // the pass is bound by instruction issue, not by shared-memory bandwidth.
      const int ir0 = (int)r0;
      constexpr int RS = 32 * QRC_H;        // row stride between a warp's blocks
      auto slow_trip = [&](int rb) {
        double x[2], yo[2], a[2][4];
        bool live[2];
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          const int r = rb + RS * k;
          live[k] = r < nr;
          const int rr = live[k] ? r : rb;
          x[k] = refl ? xj[rr] : 0.0;
          yo[k] = yp[rr];
#pragma unroll
          for (int u = 0; u < 4; ++u) a[k][u] = cp[u][rr];
        }
#pragma unroll
        for (int k = 0; k < 2; ++k) {
          const int r = rb + RS * k;
          const int gr = ir0 + r;
          if (!live[k]) continue;
          if (gr < jj) {
            if (g0 && gr == jj - 1) xhome[r] = x[k];
            continue;
          }
          const double v = !refl ? 0.0 : (gr > jj ? x[k] * scal : 1.0);
          const double y = fma(-v, wp, yo[k]);
#pragma unroll
          for (int u = 0; u < 4; ++u) a[k][u] = fma(-v, wu[u], a[k][u]);
          if (g0) {
            a[k][0] = y;
            ynew[r] = y;
            if (refl) xhome[r] = x[k];
          } else if (refl) {
            cp[0][r] = a[k][0];
          }
          if (refl) {
            if (nu > 1) cp[1][r] = a[k][1];
            if (nu > 2) cp[2][r] = a[k][2];
            if (nu > 3) cp[3][r] = a[k][3];
          }
          if (gr > pv) {
#pragma unroll
            for (int u = 0; u < 4; ++u) acc[u] = fma(y, a[k][u], acc[u]);
          }
        }
      };
      int rb = lane + 32 * half;
      // leading trips that touch rows <= pv (cluster rank 0 only)
      for (; rb < nr && ir0 + (rb - lane) <= pv; rb += 2 * RS) slow_trip(rb);
      if (refl) {
        // full blocks entirely below row pv: running pointers, no predicates
        const double* px = xj + rb;
        const double* py = yp + rb;
        double *p0 = cp[0] + rb, *p1 = cp[1] + rb, *p2 = cp[2] + rb, *p3 = cp[3] + rb;
        double *pyn = ynew + rb, *pxh = xhome + rb;
        const double nscal = -scal;
        for (; (rb - lane) + RS + 32 <= nr; rb += 2 * RS) {
          const double x0 = px[0], x1 = px[RS], y0 = py[0], y1 = py[RS];
          double a00 = p0[0], a01 = p1[0], a02 = p2[0], a03 = p3[0];
          double a10 = p0[RS], a11 = p1[RS], a12 = p2[RS], a13 = p3[RS];
          const double v0 = x0 * nscal, v1 = x1 * nscal;   // -v
          const double yy0 = fma(v0, wp, y0), yy1 = fma(v1, wp, y1);
          a00 = fma(v0, wu[0], a00); a01 = fma(v0, wu[1], a01);
          a02 = fma(v0, wu[2], a02); a03 = fma(v0, wu[3], a03);
          a10 = fma(v1, wu[0], a10); a11 = fma(v1, wu[1], a11);
          a12 = fma(v1, wu[2], a12); a13 = fma(v1, wu[3], a13);
          if (g0) {
            a00 = yy0; a10 = yy1;
            pyn[0] = yy0; pyn[RS] = yy1;
            pxh[0] = x0; pxh[RS] = x1;
          } else {
            p0[0] = a00; p0[RS] = a10;
          }
          if (nu > 1) { p1[0] = a01; p1[RS] = a11; }
          if (nu > 2) { p2[0] = a02; p2[RS] = a12; }
          if (nu > 3) { p3[0] = a03; p3[RS] = a13; }
          acc[0] = fma(yy0, a00, acc[0]); acc[1] = fma(yy0, a01, acc[1]);
          acc[2] = fma(yy0, a02, acc[2]); acc[3] = fma(yy0, a03, acc[3]);
          acc[0] = fma(yy1, a10, acc[0]); acc[1] = fma(yy1, a11, acc[1]);
          acc[2] = fma(yy1, a12, acc[2]); acc[3] = fma(yy1, a13, acc[3]);
          px += 2 * RS; py += 2 * RS; p0 += 2 * RS; p1 += 2 * RS; p2 += 2 * RS; p3 += 2 * RS;
          pyn += 2 * RS; pxh += 2 * RS;
        }
      }
      for (; rb < nr; rb += 2 * RS) slow_trip(rb);
      // transposing butterfly: 4 sums over 32 lanes in 6 exchanges; lane
      // 8u ends with column col0 + u
      const bool hi = lane & 16, mid = lane & 8;
      double k0 = (hi ? acc[2] : acc[0]) + __shfl_xor_sync(0xffffffffu, hi ? acc[0] : acc[2], 16);
      double k1 = (hi ? acc[3] : acc[1]) + __shfl_xor_sync(0xffffffffu, hi ? acc[1] : acc[3], 16);
      double k = (mid ? k1 : k0) + __shfl_xor_sync(0xffffffffu, mid ? k0 : k1, 8);
      k += __shfl_xor_sync(0xffffffffu, k, 4);
      k += __shfl_xor_sync(0xffffffffu, k, 2);
      k += __shfl_xor_sync(0xffffffffu, k, 1);
      if ((lane & 7) == 0 && col0 + (lane >> 3) < ncp) s_dpart[half][col0 + (lane >> 3)] = k;
    }
    QPROF(6);
  }
  __syncthreads();
  // the last pivot column's rows >= w - 2 are still in piv
  for (int r = t; r < nr; r += QRC)
    if (r0 + r >= w - 2) chunk[r + (w - 1) * ld] = piv[((w - 1) & 1) * ld + r];
  __syncthreads();
  // write back R / the scaled reflectors, and V (unit diagonal, zeros above)
  for (int col = warp; col < w; col += QRC / 32) {
    const double scal = s_scal[col], beta = s_beta[col];
    for (int r = lane; r < nr; r += 32) {
      const int64_t gr = r0 + r;
      const double x = chunk[r + col * ld];
      const double a = gr > col ? x * scal : (gr == col ? beta : x);
      p.A[gr + col * p.lda] = a;
      const double v = gr > col ? a : (gr == col ? 1.0 : 0.0);
      p.V[gr + (int64_t)col * p.ldv] = v;
      chunk[r + col * ld] = v;
    }
  }
  __syncthreads();
  QPROF(8);
  vtv_partial_dmma32(chunk, ld, nr, w, s_vtv);
  QPROF(9);
  cluster.sync();
  QPROF(10);
  if (c == 0) {
    // sum the V^T V partials (fixed rank order) in place, then dlarft
    for (int idx = t; idx < QR_NB * QR_NB; idx += QRC) {
      if ((idx & (QR_NB - 1)) >= (idx / QR_NB) || (idx / QR_NB) >= w) continue;   // strict upper part only
      double tot = 0.0;
      double xv[16];   // all remote loads in flight, then the rank-order sum
#pragma unroll
      for (int i = 0; i < 16; ++i) xv[i] = i < CS ? cluster.map_shared_rank(s_vtv, i)[idx] : 0.0;
#pragma unroll
      for (int i = 0; i < 16; ++i) tot += xv[i];
      s_vtv[idx] = tot;
    }
  }
  QPROF(11);
  cluster.sync();  // the partials are read: the other ranks may exit
  QPROF(12);
  if (c == 0 && warp == 0) build_t_factor_warp(s_vtv, s_tau, w, p.T, p.tau);
  QPROF(13);
#ifdef MPO_QR_PROF
  if (t == 0 && c == 0)
    printf("qrprof mp=%lld w=%d nr=%d CS=%d: fusedtail %lld syncA %lld push %lld wait %lld scal %lld syncC %lld fused %lld (unused %lld) | wb %lld vtv %lld cs1 %lld gather %lld cs2 %lld buildT %lld total %lld\n",
           (long long)p.mp, w, nr, CS, pacc[0], pacc[1], pacc[2], pacc[3], pacc[4], pacc[5], pacc[6], pacc[7],
           pacc[8], pacc[9], pacc[10], pacc[11], pacc[12], pacc[13], clock64() - pstart);
#endif
}

// Application of inner panels' reflectors to a column range in ONE launch:
//   A_r <- (I - V_i T_i V_i^T)^T A_r = A_r - V_i T_i^T (V_i^T A_r),  i = 0 .. npan-1 in order,
// instead of three skinny GEMMs per panel (K = panel height for an output of
// 32 x <= 128: 7-13 us each on the panel chain).  Used for the in-block update
// (one panel, the rest of its outer block) and for the look-ahead ("near")
// update of the next outer block's columns with all of a block's panels --
// which then needs only the panels' own T factors, not the assembled outer T.
// Column slabs of 8 x clusters of R CTAs along the rows: a CTA forms its rows'
// part of W = V_i^T A_r (wi x 8, DMMA, fragments straight from L2), the cluster
// all-gathers the partials with st.async on each rank's mbarrier (fixed
// rank-order sum; buffers and mbarriers alternate by panel parity), then every
// CTA applies A_r -= V_i (T_i^T W) to its rows.
constexpr int IB_MAXP = 16;       // panels per launch (an outer block of 8-column panels)
struct InblockArgs {
  const double* V;   // mp x (sum of widths), ld ldv: unit diagonals, zeros above
  int64_t ldv;
  const double* T;   // panel i's wi x wi upper triangular factor at T + toff[i], ld wi
  double* A;         // mp x rem, ld lda
  int64_t lda;
  int64_t mp;
  int rem;
  int rpc;           // rows per CTA
  int npan;
  int voff[IB_MAXP]; // first column of panel i in V
  int wid[IB_MAXP];  // its width (<= 32)
  int toff[IB_MAXP];
};
constexpr int IBT = 512;          // 16 warps: 4 reflector-column tiles x 4 row quarters
constexpr int IB_MAXR = 16;       // cluster size along the rows (non-portable above 8)
constexpr int IB_SMEM = 2 * IB_MAXR * QR_NB * 8 * (int)sizeof(double);
__global__ void __launch_bounds__(IBT, 2) qr_inblock_cluster_kernel(InblockArgs p) {
  extern __shared__ double s_all[];        // [2][IB_MAXR][QR_NB * 8] gathered partials, by parity
  __shared__ double s_part[4][QR_NB * 8];  // row-quarter partials, then T (same size)
  __shared__ double s_W[QR_NB * 8], s_W2[QR_NB * 8];
  __shared__ __align__(8) unsigned long long s_mbar[2];
  double* s_T = &s_part[0][0];
  cg::cluster_group cluster = cg::this_cluster();
  const int R = (int)cluster.num_blocks(), q = (int)cluster.block_rank();
  const int slab = blockIdx.x / R;
  const int t = threadIdx.x, lane = t & 31, warp = t >> 5;
  const int n0 = slab * 8, ncol = min(8, p.rem - n0);
  const int64_t rbeg = (int64_t)q * p.rpc, rend = min(p.mp, rbeg + p.rpc);
  if (t == 0) {
    mbar_init(smem_addr(&s_mbar[0]), 1);
    mbar_init(smem_addr(&s_mbar[1]), 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  cluster.sync();   // mbarriers initialised cluster-wide before any remote store
  for (int ph = 0; ph < p.npan; ++ph) {
    const int wi = p.wid[ph];
    const double* Vp = p.V + (int64_t)p.voff[ph] * p.ldv;
    const uint32_t mb = smem_addr(&s_mbar[ph & 1]);
    double* all = s_all + (ph & 1) * (IB_MAXR * QR_NB * 8);
    if (t == 0) mbar_expect_tx(mb, (uint32_t)(R * QR_NB * 8 * 8));
    // W partial: warp (mt, kq) = reflector columns 8 mt.., quarter kq of the rows
    {
      const int mt = warp & 3, kq = warp >> 2;
      const int64_t nrows = rend - rbeg, qlen = (((nrows + 3) / 4 + 3) & ~(int64_t)3);
      const int64_t lo = min(rbeg + kq * qlen, rend), hi = min(lo + qlen, rend);
      const int mc = mt * 8 + (lane >> 2), nc = lane >> 2;
      const bool mok = mc < wi, nok = nc < ncol;
      const double* pv = Vp + (int64_t)mc * p.ldv + (lane & 3);
      const double* pa = p.A + (int64_t)(n0 + nc) * p.lda + (lane & 3);
      double acc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
      if (mt * 8 < wi)
        for (int64_t k0 = lo; k0 < hi; k0 += 32) {
          double av[8], bv[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) {
            const int64_t kk = k0 + 4 * u + (lane & 3);
            const bool in = kk < hi;
            av[u] = (in && mok) ? pv[k0 + 4 * u] : 0.0;
            bv[u] = (in && nok) ? pa[k0 + 4 * u] : 0.0;
          }
#pragma unroll
          for (int u = 0; u < 8; ++u) dmma884(acc[u & 1], av[u], bv[u]);
        }
#pragma unroll
      for (int e = 0; e < 2; ++e)
        s_part[kq][(mt * 8 + (lane >> 2)) * 8 + 2 * (lane & 3) + e] = acc[0][e] + acc[1][e];
    }
    __syncthreads();
    if (t < QR_NB * 8) {
      const double wsum = (s_part[0][t] + s_part[1][t]) + (s_part[2][t] + s_part[3][t]);
      const uint32_t dst = smem_addr(&all[q * (QR_NB * 8) + t]);
      for (int rk = 0; rk < R; ++rk)
        asm volatile("st.async.weak.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];"
                     ::"r"(cluster_addr(dst, rk)), "l"(__double_as_longlong(wsum)),
                     "r"(cluster_addr(mb, rk)) : "memory");
    }
    __syncthreads();   // the partials are consumed: their buffer takes T
    {
      const double* Tp = p.T + p.toff[ph];
      for (int idx = t; idx < QR_NB * QR_NB; idx += IBT) {
        const int i = idx & (QR_NB - 1), j = idx / QR_NB;
        s_T[idx] = (i < wi && j < wi) ? Tp[i + j * wi] : 0.0;
      }
    }
    mbar_wait(mb, (ph >> 1) & 1);
    if (t < QR_NB * 8) {
      double tot = 0.0;
      for (int rk = 0; rk < R; ++rk) tot += all[rk * (QR_NB * 8) + t];
      s_W[t] = tot;
    }
    __syncthreads();
    if (t < QR_NB * 8) {   // W2 = T^T W
      const int j = t >> 3, n = t & 7;
      double a0 = 0.0, a1 = 0.0;
      for (int i = 0; i < QR_NB; i += 2) {
        a0 = fma(s_T[i + j * QR_NB], s_W[i * 8 + n], a0);
        a1 = fma(s_T[i + 1 + j * QR_NB], s_W[(i + 1) * 8 + n], a1);
      }
      s_W2[t] = a0 + a1;
    }
    __syncthreads();
    // A_r -= V W2 on this CTA's rows, 8-row tiles per warp
    {
      const int m = lane >> 2, kq = lane & 3;
      double bw[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) bw[u] = s_W2[(4 * u + kq) * 8 + m];   // B[k][n = m]
      for (int64_t rt = rbeg + 8 * warp; rt < rend; rt += 8 * (IBT / 32)) {
        const int64_t row = rt + m;
        const bool rok = row < rend;
        double av[8];
#pragma unroll
        for (int u = 0; u < 8; ++u)
          av[u] = (rok && 4 * u + kq < wi) ? Vp[row + (int64_t)(4 * u + kq) * p.ldv] : 0.0;
        double cold[2];
#pragma unroll
        for (int e = 0; e < 2; ++e)
          cold[e] = (rok && 2 * kq + e < ncol) ? p.A[row + (int64_t)(n0 + 2 * kq + e) * p.lda] : 0.0;
        double acc[2][2] = {{0.0, 0.0}, {0.0, 0.0}};
#pragma unroll
        for (int u = 0; u < 8; ++u) dmma884(acc[u & 1], av[u], bw[u]);
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int n = 2 * kq + e;
          if (rok && n < ncol) p.A[row + (int64_t)(n0 + n) * p.lda] = cold[e] - (acc[0][e] + acc[1][e]);
        }
      }
    }
    __syncthreads();   // this CTA's rows of A_r are updated before the next panel reads them
  }
}

__global__ void extract_r_kernel(int64_t k, int64_t n, const double* A, int64_t lda, double* R,
                                 int64_t ldr) {
  const int64_t total = k * n;
  for (int64_t idx = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; idx < total;
       idx += (int64_t)gridDim.x * blockDim.x) {
    int64_t i = idx % k, j = idx / k;
    R[i + j * ldr] = (i <= j) ? A[i + j * lda] : 0.0;
  }
}

// one-time kernel attribute setup: C++11 magic statics make these
// thread-safe (the batched path calls in from several host threads)
int panel_smem_limit() {
  static std::once_flag once[kMaxDevices];   // per device (function attributes are)
  static int lims[kMaxDevices];
  const int dev = current_device() & (kMaxDevices - 1);
  std::call_once(once[dev], [dev] {
    int l;
    CK(cudaDeviceGetAttribute(&l, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    cudaFuncAttributes fa;
    CK(cudaFuncGetAttributes(&fa, qr_panel_kernel));
    l -= (int)fa.sharedSizeBytes + 1024;
    CK(cudaFuncSetAttribute(qr_panel_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, l));
    lims[dev] = l;
  });
  return lims[dev];
}

int cluster_smem_limit() {
  static std::once_flag once[kMaxDevices];
  static int lims[kMaxDevices];
  const int dev = current_device() & (kMaxDevices - 1);
  std::call_once(once[dev], [dev] {
    int l;
    CK(cudaDeviceGetAttribute(&l, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev));
    cudaFuncAttributes fa;
    CK(cudaFuncGetAttributes(&fa, qr_panel_cluster_kernel));
    l -= (int)fa.sharedSizeBytes + 1024;
    CK(cudaFuncSetAttribute(qr_panel_cluster_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            l));
    CK(cudaFuncSetAttribute(qr_panel_cluster_kernel,
                            cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    lims[dev] = l;
  });
  return lims[dev];
}

int max_coresident_panel_ctas(size_t smem) {
  int dev, nsm, per;
  CK(cudaGetDevice(&dev));
  CK(cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, dev));
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per, qr_panel_kernel, QR_THREADS, smem));
  return std::max(1, per) * nsm;
}

// rows per CTA of the cluster panel, and the shared-memory leading dimension
// of its slice: the smallest ld >= rpc with ld = 4 (mod 16), so the DMMA
// fragment loads of V^T V (4 consecutive rows x 8 columns per warp) take the
// minimal two wavefronts instead of an 8-way bank conflict
int64_t cluster_panel_rpc(int64_t mp) { return cdiv(std::max<int64_t>(64, cdiv(mp, 16)), 8) * 8; }
int64_t cluster_panel_ld(int64_t rpc) { return rpc + ((4 - rpc % 16) + 16) % 16; }

// widest panel (<= wmax columns) whose rows fit the panel kernels' shared
// memory: very tall, narrow matrices (e.g. the 196608 x 48 first core of
// config 3's B) are factored in narrower panels
int panel_width(int64_t mp, int wmax) {
  // prefer the cluster panel (16 CTAs, DSMEM reductions): the widest panel
  // (>= 8 columns) whose rows fit 16 CTAs' shared memory -- a 16384-row
  // panel of 32 columns does not, 16 columns do; the cooperative-grid panel
  // (one grid barrier per reduction) is several times slower per column
  const int64_t crpc = cluster_panel_rpc(mp);
  for (int w = wmax; w >= 8; w = (w + 1) / 2)
    if (cluster_panel_ld(crpc) * (w + 2) * (int64_t)sizeof(double) <= cluster_smem_limit()) return w;
  const int64_t rpc = std::max<int64_t>(32, cdiv(mp, 148));
  int w = wmax;
  while (w > 1 && rpc * w * (int64_t)sizeof(double) > panel_smem_limit()) w = (w + 1) / 2;
  return w;
}

}  // namespace

// one panel of width w at A (mp rows, ld lda): reflectors to V (ld ldv),
// compact-WY factor to T (w x w), tau to tau
static void factor_panel(cudaStream_t st, double* A, int64_t lda, int64_t mp, int w, double* V,
                         int64_t ldv, double* T, double* tau, double* part, double* wpart,
                         double* vtv, double* alpha) {
  ProfScope prof(st, 4, 4.0 * (double)mp * w * w);   // panel Householder work
  // preferred: one thread-block cluster (<= 16 CTAs, DSMEM reductions)
  const int64_t crpc = cluster_panel_rpc(mp), cld = cluster_panel_ld(crpc);
  const size_t csmem = (size_t)cld * (w + 2) * sizeof(double);   // slice + two pivot columns
  if ((int64_t)csmem <= cluster_smem_limit()) {
    const int CS = (int)cdiv(mp, crpc);
    ClusterPanelArgs ca{A, lda, mp, w, (int)crpc, (int)cld, V, ldv, T, tau};
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(CS);
    cfg.blockDim = dim3(QRC);
    cfg.dynamicSmemBytes = csmem;
    cfg.stream = st;
    cudaLaunchAttribute attr[1];
    attr[0].id = cudaLaunchAttributeClusterDimension;
    attr[0].val.clusterDim.x = CS;
    attr[0].val.clusterDim.y = 1;
    attr[0].val.clusterDim.z = 1;
    cfg.attrs = attr;
    cfg.numAttrs = 1;
    CK(cudaLaunchKernelEx(&cfg, qr_panel_cluster_kernel, ca));
  } else {
    const int gmax = 148;
    int64_t rpc = std::max<int64_t>(32, cdiv(mp, gmax));
    size_t smem = (size_t)rpc * w * sizeof(double);
    if ((int64_t)smem > panel_smem_limit())
      throw ValueError("QR panel too tall for the cooperative panel kernel");
    int G = (int)cdiv(mp, rpc);
    if (G > max_coresident_panel_ctas(smem)) throw CudaError("QR panel grid not co-resident");
    PanelArgs pa{A, lda, mp, w, (int)rpc, V, ldv, T, tau, part, wpart, vtv, alpha};
    void* args[] = {&pa};
    CK(cudaLaunchCooperativeKernel((void*)qr_panel_kernel, dim3(G), dim3(QR_THREADS), args, smem,
                                   st));
  }
  note_launch();
}

// A_r (mp x rem) <- A_r - V_i T_i^T (V_i^T A_r), i = 0 .. npan-1, for panels
// i of widths wid[i] at columns voff[i] of V (ld ldv, full height mp: zeros
// above each unit diagonal) with T_i at T + toff[i]; one clustered launch
// (qr_inblock_cluster_kernel)
static void panels_apply(cudaStream_t st, const double* V, int64_t ldv, const double* T, int npan,
                         const int* voff, const int* wid, const int* toff, double* A, int64_t lda,
                         int64_t mp, int64_t rem) {
  // <= 8 CTAs along the rows, 16 for tall panels (512-row slices)
  static std::once_flag once[kMaxDevices];
  once_per_device(once, [] {
    CK(cudaFuncSetAttribute(qr_inblock_cluster_kernel,
                            cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    CK(cudaFuncSetAttribute(qr_inblock_cluster_kernel,
                            cudaFuncAttributeMaxDynamicSharedMemorySize, IB_SMEM));
  });
  double wsum = 0.0;
  for (int i = 0; i < npan; ++i) wsum += wid[i];
  ProfScope prof(st, 5, 4.0 * (double)mp * wsum * (double)rem);
  const int maxr = mp > 4096 ? IB_MAXR : 8;
  const int64_t rows = cdiv(cdiv(mp, (int64_t)maxr), (int64_t)8) * 8;
  const int64_t rpc = std::max<int64_t>(128, rows);
  const int R = (int)cdiv(mp, rpc);
  const int nslab = (int)cdiv(rem, (int64_t)8);
  InblockArgs a{};
  a.V = V; a.ldv = ldv; a.T = T; a.A = A; a.lda = lda; a.mp = mp; a.rem = (int)rem;
  a.rpc = (int)rpc; a.npan = npan;
  for (int i = 0; i < npan; ++i) { a.voff[i] = voff[i]; a.wid[i] = wid[i]; a.toff[i] = toff[i]; }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(R * nslab);
  cfg.blockDim = dim3(IBT);
  cfg.dynamicSmemBytes = IB_SMEM;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = R;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  CK(cudaLaunchKernelEx(&cfg, qr_inblock_cluster_kernel, a));
  note_launch();
}

// Two-level blocked Householder QR: panels of QR_NB = 32 columns are
// factored inside outer blocks of NBO = 128 columns; the panel's reflectors
// update only the rest of their outer block, and the trailing matrix is
// updated once per outer block with K = 128 DMMA GEMMs (compute-bound rather
// than one rank-32 HBM pass per panel).  The outer block's T is assembled
// from the panels' T's: T = [[T1, -T1 (V1^T V2) T2], [0, T2]].
static void householder_qr_impl(cudaStream_t st, int64_t m, int64_t n, double* A, int64_t lda,
                                double* Q, int64_t ldq, double* R, int64_t ldr,
                                QrReflectors* keep, bool defer_q = false) {
  constexpr int NBO = QrReflectors::NBO;
  const int64_t k = std::min(m, n);
  if (k <= 0) return;
  const int64_t nob = cdiv(k, NBO);
  // per outer block: V (mp x wo, ld mp, zero above the unit diagonal) and T (wo x wo)
  std::vector<int64_t> voff(nob), wos(nob);
  int64_t vtotal = 0;
  for (int64_t b = 0; b < nob; ++b) {
    const int64_t j0 = b * NBO;
    wos[b] = std::min<int64_t>(NBO, k - j0);
    voff[b] = vtotal;
    vtotal += (m - j0) * wos[b];
  }
  DBuf<double> V((size_t)vtotal, st), T((size_t)nob * NBO * NBO, st), tau(k + QR_NB, st);
  fill_zero(st, V.get(), vtotal);
  fill_zero(st, T.get(), nob * NBO * NBO);
  const int gmax = 148;
  DBuf<double> part(gmax, st), wpart((size_t)gmax * QR_NB, st),
      vtv((size_t)gmax * QR_NB * QR_NB, st), alpha(1, st);
  // one compact-WY T slot per inner panel of an outer block (indexed by the
  // panel's first column): the outer T is assembled on the aux stream while
  // the panel chain moves on, so a panel's T must outlive the next panels
  DBuf<double> TpAll((size_t)NBO * QR_NB * QR_NB, st), S((size_t)NBO * NBO, st),
      tmp((size_t)NBO * QR_NB, st);
  DBuf<double> W, W2;
  // look-ahead (see the trailing update below) for matrices with > 2 outer blocks
  static const bool lookahead = std::getenv("MPO_B200_QR_LOOKAHEAD")
                                    ? std::atoi(std::getenv("MPO_B200_QR_LOOKAHEAD")) != 0
                                    : true;
  const bool la = lookahead && nob > 2 && n > 2 * NBO;
  SideStream* sd = la ? &side_stream(st) : nullptr;
  cudaEvent_t ev_panel = la ? sd->e[4] : nullptr, ev_far = la ? sd->e[5] : nullptr;
  cudaEvent_t ev_v = la ? sd->e[6] : nullptr, ev_t = la ? sd->e[7] : nullptr;
  // the outer-T assembly (off the panel chain's critical path) runs here
  cudaStream_t ts = la ? sd->aux : st;
  // the panel chain (panels, in-block updates, near updates) runs on the
  // highest-priority stream so its small launches are scheduled ahead of
  // the far updates' CTAs
  cudaStream_t ps = la ? sd->hp : st;
  auto ensure = [&](int64_t sz) {
    if ((int64_t)W.size() < sz) { W.alloc((size_t)sz, ps); W2.alloc((size_t)sz, ps); }
  };
  DBuf<double> Ws, Ws2;
  if (la) {
    CK(cudaEventRecord(ev_panel, st));              // A, V, T initialised
    CK(cudaStreamWaitEvent(sd->sv, ev_panel, 0));
    CK(cudaStreamWaitEvent(ps, ev_panel, 0));
    CK(cudaStreamWaitEvent(ts, ev_panel, 0));
    Ws.alloc((size_t)NBO * n, sd->sv);
    Ws2.alloc((size_t)NBO * n, sd->sv);
  }
  static const bool fused_inblock = std::getenv("MPO_B200_QR_INBLOCK")
                                        ? std::atoi(std::getenv("MPO_B200_QR_INBLOCK")) != 0
                                        : true;
  // taller panels leave > 1024 rows to each CTA of a 16-CTA row cluster: the
  // split-K GEMMs over all SMs are faster there (row-sharded TSQR's local QRs)
  constexpr int64_t kFusedApplyMaxRows = 16384;
  static const bool fused_near = std::getenv("MPO_B200_QR_NEAR")
                                     ? std::atoi(std::getenv("MPO_B200_QR_NEAR")) != 0
                                     : true;
  for (int64_t b = 0; b < nob; ++b) {
    const int64_t j0 = b * NBO, wo = wos[b], mp = m - j0;
    double* Vo = V.get() + voff[b];
    double* To = T.get() + b * NBO * NBO;   // ld wo
    int pan_off[IB_MAXP], pan_w[IB_MAXP], pan_t[IB_MAXP], npan = 0;   // this block's panels
    bool pan_ok = true;
    for (int64_t i0 = 0, wi = 0; i0 < wo; i0 += wi) {
      const int64_t jj = j0 + i0, mpi = m - jj;
      wi = std::min<int64_t>(panel_width(mpi, QR_NB), wo - i0);
      double* Tpi = TpAll.get() + i0 * QR_NB * QR_NB;
      if (npan < IB_MAXP && wi <= QR_NB) {
        pan_off[npan] = (int)i0; pan_w[npan] = (int)wi; pan_t[npan] = (int)(i0 * QR_NB * QR_NB);
        ++npan;
      } else {
        pan_ok = false;
      }
      factor_panel(ps, A + jj + jj * lda, lda, mpi, wi, Vo + i0 + i0 * mp, mp, Tpi,
                   tau.get() + jj, part.get(), wpart.get(), vtv.get(), alpha.get());
      if (la) {
        CK(cudaEventRecord(ev_v, ps));
        CK(cudaStreamWaitEvent(ts, ev_v, 0));
      }
      // place the panel's T on the diagonal of the outer T (aux stream)
      copy_matrix(ts, wi, wi, Tpi, wi, To + i0 + i0 * wo, wo);
      if (i0 > 0) {
        // To[0:i0, i0:i0+wi] = -To[0:i0, 0:i0] (V[:, 0:i0]^T V[:, i0:i0+wi]) Tp
        dgemm(ts, true, false, i0, wi, mp, 1.0, Vo, mp, Vo + i0 * mp, mp, 0.0, S.get(), i0);
        dgemm(ts, false, false, i0, wi, i0, 1.0, To, wo, S.get(), i0, 0.0, tmp.get(), i0);
        dgemm(ts, false, false, i0, wi, wi, -1.0, tmp.get(), i0, Tpi, wi, 0.0, To + i0 * wo, wo);
      }
      // update the rest of this outer block with the panel's reflectors
      const int64_t rem = wo - (i0 + wi);
      if (rem > 0) {
        double* Ar = A + jj + (jj + wi) * lda;
        const double* Vi = Vo + i0 + i0 * mp;
        if (fused_inblock && wi <= QR_NB && mpi <= kFusedApplyMaxRows) {
          const int z = 0, wv = (int)wi;
          panels_apply(ps, Vi, mp, Tpi, 1, &z, &wv, &z, Ar, lda, mpi, rem);
        } else {
          ensure(wi * rem);
          dgemm(ps, true, false, wi, rem, mpi, 1.0, Vi, mp, Ar, lda, 0.0, W.get(), wi);
          dgemm(ps, true, false, wi, rem, wi, 1.0, Tpi, wi, W.get(), wi, 0.0, W2.get(), wi);
          dgemm(ps, false, false, mpi, rem, wi, -1.0, Vi, mp, W2.get(), wi, 1.0, Ar, lda);
        }
      }
    }
    // trailing update of columns j0+wo .. n-1 with the outer block:
    // A -= V T^T (V^T A).  With look-ahead, only the next outer block's
    // columns ("near") are updated here; the rest ("far") go to the side
    // stream and overlap the next block's latency-bound panels (<= 16 SMs).
    // Main waits for far(b-1) before near(b): the near columns were part of
    // far(b-1)'s range.
    if (la) CK(cudaEventRecord(ev_t, ts));   // the outer T of this block is assembled
    const int64_t nt = n - (j0 + wo);
    const int64_t near = nt <= 0 ? 0 : (la ? std::min<int64_t>(nt, NBO) : nt), far = nt - near;
    // near update straight from the panels' own (V_i, T_i), one launch: the
    // panel chain does not wait for the assembled outer T
    const bool near_fused = fused_inblock && fused_near && pan_ok && near > 0 && near <= NBO &&
                            mp <= kFusedApplyMaxRows;
    if (la && !(nt > 0 && near_fused)) CK(cudaStreamWaitEvent(ps, ev_t, 0));
    if (nt > 0) {
      double* At = A + j0 + (j0 + wo) * lda;
      if (la) {
        CK(cudaEventRecord(ev_panel, ps));   // block b's V is ready
        if (b > 0) CK(cudaStreamWaitEvent(ps, ev_far, 0));
      }
      if (near_fused) {
        panels_apply(ps, Vo, mp, TpAll.get(), npan, pan_off, pan_w, pan_t, At, lda, mp, near);
        // the next block's panels overwrite the T slots the assembly reads
        if (la) CK(cudaStreamWaitEvent(ps, ev_t, 0));
      } else {
        ensure(wo * near);
        dgemm(ps, true, false, wo, near, mp, 1.0, Vo, mp, At, lda, 0.0, W.get(), wo);
        dgemm(ps, true, false, wo, near, wo, 1.0, To, wo, W.get(), wo, 0.0, W2.get(), wo);
        dgemm(ps, false, false, mp, near, wo, -1.0, Vo, mp, W2.get(), wo, 1.0, At, lda);
      }
      if (far > 0) {
        cudaStream_t sv = sd->sv;
        double* Af = At + near * lda;
        CK(cudaStreamWaitEvent(sv, ev_panel, 0));
        CK(cudaStreamWaitEvent(sv, ev_t, 0));
        dgemm(sv, true, false, wo, far, mp, 1.0, Vo, mp, Af, lda, 0.0, Ws.get(), wo);
        dgemm(sv, true, false, wo, far, wo, 1.0, To, wo, Ws.get(), wo, 0.0, Ws2.get(), wo);
        dgemm(sv, false, false, mp, far, wo, -1.0, Vo, mp, Ws2.get(), wo, 1.0, Af, lda);
        CK(cudaEventRecord(ev_far, sv));
      }
    }
  }
  if (la) {   // main continues after the last far and the last panel-chain work
    CK(cudaStreamWaitEvent(st, ev_far, 0));
    CK(cudaEventRecord(ev_panel, ps));
    CK(cudaStreamWaitEvent(st, ev_panel, 0));
    ps = st;   // workspace (re)allocations below are ordered on the main stream
  }
  if (R) {
    extract_r_kernel<<<(int)std::max<int64_t>(1, std::min<int64_t>(cdiv(k * n, 256), 2368)), 256,
                       0, st>>>(k, n, A, lda, R, ldr);
    CK_LAUNCH();
    note_launch();
  }
  if (keep) {
    keep->m = m;
    keep->k = k;
    keep->voff = voff;
    keep->wos = wos;
    keep->V = std::move(V);
    keep->T = std::move(T);
  }
  if (!Q) return;
  // dorgqr: Q = H_1 ... H_k [I; 0], outer blocks applied last to first (a
  // block's reflectors act only on rows j0.. and, for [I; 0], on columns j0..)
  cudaStream_t qst = st;
  SideStream* sq = nullptr;
  static const bool defer_env = std::getenv("MPO_B200_QR_DEFERQ")
                                    ? std::atoi(std::getenv("MPO_B200_QR_DEFERQ")) != 0
                                    : true;
  if (defer_q && defer_env && !keep) {
    // on the Q stream, behind the factorisation; V and T are released there
    sq = &side_stream(st);
    CK(cudaEventRecord(sq->eqf, st));
    CK(cudaStreamWaitEvent(sq->qs, sq->eqf, 0));
    qst = sq->qs;
    V.set_stream(qst);
    T.set_stream(qst);
  }
  DBuf<double> Wq, Wq2;
  if (sq) {
    Wq.alloc((size_t)NBO * k, qst);
    Wq2.alloc((size_t)NBO * k, qst);
  }
  set_identity(qst, m, k, Q, ldq);
  for (int64_t b = nob - 1; b >= 0; --b) {
    const int64_t j0 = b * NBO, wo = wos[b], mp = m - j0, nq = k - j0;
    const double* Vo = (keep ? keep->V.get() : V.get()) + voff[b];
    const double* To = (keep ? keep->T.get() : T.get()) + b * NBO * NBO;
    double* Qb = Q + j0 + j0 * ldq;
    if (!sq) ensure(wo * nq);
    double* w1 = sq ? Wq.get() : W.get();
    double* w2 = sq ? Wq2.get() : W2.get();
    dgemm(qst, true, false, wo, nq, mp, 1.0, Vo, mp, Qb, ldq, 0.0, w1, wo);
    dgemm(qst, false, false, wo, nq, wo, 1.0, To, wo, w1, wo, 0.0, w2, wo);
    dgemm(qst, false, false, mp, nq, wo, -1.0, Vo, mp, w2, wo, 1.0, Qb, ldq);
  }
  if (sq) {
    CK(cudaEventRecord(sq->eq, qst));
    sq->q_pending = true;
  }
}

void join_deferred_q(cudaStream_t st) {
  SideStream& sd = side_stream(st);
  if (!sd.q_pending) return;
  cudaStreamWaitEvent(st, sd.eq, 0);   // no throw: also runs from destructors
  sd.q_pending = false;
}

void householder_qr(cudaStream_t st, int64_t m, int64_t n, double* A, int64_t lda, double* Q,
                    int64_t ldq, double* R, int64_t ldr, bool defer_q) {
  if (small_qr(st, m, n, A, lda, Q, ldq, R, ldr)) return;   // one CTA (small.cu)
  householder_qr_impl(st, m, n, A, lda, Q, ldq, R, ldr, nullptr, defer_q);
}

void householder_qr_keep(cudaStream_t st, int64_t m, int64_t n, double* A, int64_t lda,
                         double* R, int64_t ldr, QrReflectors& f) {
  householder_qr_impl(st, m, n, A, lda, nullptr, 0, R, ldr, &f);
}

// C <- Q C for the m x ncols matrix C (Q = H_1 ... H_k from householder_qr_keep):
// the dorgqr recurrence on an arbitrary right-hand side, so Q times a
// k-column block costs one reflector sweep instead of forming Q and a GEMM
void qr_apply_q(cudaStream_t st, const QrReflectors& f, double* C, int64_t ldc, int64_t ncols) {
  constexpr int NBO = QrReflectors::NBO;
  const int64_t nob = (int64_t)f.wos.size();
  if (ncols <= 0 || nob == 0) return;
  DBuf<double> W((size_t)NBO * ncols, st), W2((size_t)NBO * ncols, st);
  for (int64_t b = nob - 1; b >= 0; --b) {
    const int64_t j0 = b * NBO, wo = f.wos[b], mp = f.m - j0;
    const double* Vo = f.V.get() + f.voff[b];
    const double* To = f.T.get() + b * NBO * NBO;
    double* Cb = C + j0;
    dgemm(st, true, false, wo, ncols, mp, 1.0, Vo, mp, Cb, ldc, 0.0, W.get(), wo);
    dgemm(st, false, false, wo, ncols, wo, 1.0, To, wo, W.get(), wo, 0.0, W2.get(), wo);
    dgemm(st, false, false, mp, ncols, wo, -1.0, Vo, mp, W2.get(), wo, 1.0, Cb, ldc);
  }
}

// X <- X Q for the nrows x m matrix X: X H_b = X - (X V_b) T_b V_b^T on the
// columns j0.. of each outer block, first block to last
void qr_apply_q_right(cudaStream_t st, const QrReflectors& f, double* X, int64_t ldx,
                      int64_t nrows) {
  constexpr int NBO = QrReflectors::NBO;
  const int64_t nob = (int64_t)f.wos.size();
  if (nrows <= 0 || nob == 0) return;
  DBuf<double> W((size_t)NBO * nrows, st), W2((size_t)NBO * nrows, st);
  for (int64_t b = 0; b < nob; ++b) {
    const int64_t j0 = b * NBO, wo = f.wos[b], mp = f.m - j0;
    const double* Vo = f.V.get() + f.voff[b];
    const double* To = f.T.get() + b * NBO * NBO;
    double* Xb = X + j0 * ldx;
    dgemm(st, false, false, nrows, wo, mp, 1.0, Xb, ldx, Vo, mp, 0.0, W.get(), nrows);
    dgemm(st, false, false, nrows, wo, wo, 1.0, W.get(), nrows, To, wo, 0.0, W2.get(), nrows);
    dgemm(st, false, true, nrows, mp, wo, -1.0, W2.get(), nrows, Vo, mp, 1.0, Xb, ldx);
  }
}

}  // namespace mpob

// Sparse -> MPO conversion structure, bucketed fast path (sm_100a).
//
// Same result as the onesweep pipeline in convert.cu -- np.unique(key,
// return_inverse=True) of the kept block keys, sparse.py:234-250 -- with
// about half the DRAM traffic, by sorting MSD-first into buckets that fit one
// CTA's shared memory and finishing each bucket on chip:
//
//   K1 fast_hist     per 16K-entry tile: histogram of the bucket (key >> s)
//                    of every kept entry, kept count          read col (+row), val
//   K2 fast_scan_*   per-bucket tile offsets, bucket starts, kept offsets
//   K3 fast_scatter  per tile: key, bucket, 64-bit item (low key | position),
//                    staged by bucket in shared memory, written as runs into
//                    the bucket regions                        read row, col, val;
//                                                              write 8 B / entry
//   K4 fast_bucket   per bucket (<= 16K entries, taken in bucket order from a
//                    ticket), 32 warps: for the square 2^k plans a stable
//                    counting pass on the block-column bits (ballot
//                    multisplit, warp-private counters) groups each block
//                    column's items in fast_scatter (tile) order -- for
//                    row-sorted input already ordered by block row except
//                    where two entries of one column met in one tile -- then
//                    only groups with a key inversion are re-sorted (one
//                    warp each); other plans and oversize groups take stable
//                    10-bit LSD passes.  Head flags -> local block ids,
//                    decoupled look-back over the preceding buckets (the
//                    whole CTA polls 1024 predecessors per step, relaxed
//                    loads) for the global id offset, then uniq (coalesced)
//                    and ti[position]                          read 8 B, write
//                                                              8 B/block + 8 B
// Compulsory traffic is 32 B/entry + 8 B/block; this path
// moves ~64 B/entry + 8 B/block plus the random ti scatter.  Ties between
// equal keys are never ordered by anything observable (ids only), so the
// in-tile slot order (shared-memory atomics) does not affect the output,
// which is bit-identical to the reference's.
//
// Without explicit zeros the per-entry (i1, j1, values) arrays are not
// written here at all: they are derivable from the input (i1 = (row-1) % I1,
// values = val) and are materialised on demand (ensure_entries).
#include "common.cuh"
#include "convert.cuh"
#include "kernels.cuh"
#ifdef MPO_CONV_PROF
#include <cstdio>
#include <cstdlib>
#include <cstring>
#endif

namespace mpob {

namespace {

constexpr int F_CT = 512;                 // tile CTAs (K1, K3)
constexpr int F_IT = 32;
constexpr int F_TILE = F_CT * F_IT;       // 16384 entries per tile
constexpr int F_MAXB = 4096;              // buckets
constexpr int B_CT = 1024;                // bucket CTAs (K4), one per SM (measured: the same
constexpr int B_MINB = 1;                 // as two 512-thread CTAs on half-size buckets)
constexpr int B_W = B_CT / 32;
constexpr int B_IT = 16;
constexpr int B_CAP = B_CT * B_IT;        // 16384 entries per bucket
constexpr int B_RB = 10;
constexpr int B_R = 1 << B_RB;            // local digit bins

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}
constexpr unsigned long long ST_AGG = 1ull << 62, ST_PRE = 2ull << 62,
                             ST_VAL = (1ull << 62) - 1;
// status words carry their whole payload (flag | value), so the look-back
// polls with relaxed L2 loads (an acquire load would invalidate L1 on every
// poll) and publishes with a release store
__device__ __forceinline__ unsigned long long ld_relaxed(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// x / d without a 64-bit division: a shift for powers of two, a 32-bit
// division when both fit (row/col indices below 2^32)
struct FastDiv {
  uint64_t d;
  int sh;   // >= 0: power of two
};
FastDiv make_div(int64_t d) {
  FastDiv f{(uint64_t)d, -1};
  if ((d & (d - 1)) == 0) { f.sh = 0; while (((uint64_t)1 << f.sh) < (uint64_t)d) ++f.sh; }
  return f;
}
__device__ __forceinline__ uint64_t fdiv(const FastDiv& f, uint64_t x) {
  if (f.sh >= 0) return x >> f.sh;
  if ((x >> 32) == 0 && (f.d >> 32) == 0) return (uint32_t)x / (uint32_t)f.d;
  return x / f.d;
}

struct KeyMap {
  FastDiv I1, J1;
  int64_t nrb;
  int s;          // bucket = key >> s
  int bc_shift;   // >= 0: bucket = bc >> bc_shift (no row needed); -1: full key
};

__device__ __forceinline__ uint64_t entry_key(const KeyMap& m, int64_t r1, int64_t c1) {
  const uint64_t br = fdiv(m.I1, (uint64_t)(r1 - 1)), bc = fdiv(m.J1, (uint64_t)(c1 - 1));
  return br + (uint64_t)m.nrb * bc;
}

// ---------------- K1 -------------------------------------------------------
__global__ void __launch_bounds__(F_CT, 2) fast_hist(const int64_t* __restrict__ row1,
                                                  const int64_t* __restrict__ col1,
                                                  const double* __restrict__ val, int64_t n,
                                                  KeyMap m, int nb, bool zero_aware,
                                                  uint16_t* __restrict__ thist,
                                                  unsigned* __restrict__ tkept) {
  // zero_aware = false: every entry counted as kept (fast_scatter checks the
  // values and flags a rerun with zero_aware = true if any is zero)
  __shared__ unsigned h[F_MAXB];
  __shared__ unsigned wsum[F_CT / 32];
  for (int i = threadIdx.x; i < nb; i += F_CT) h[i] = 0;
  __syncthreads();
  const int64_t base = blockIdx.x * (int64_t)F_TILE;
  unsigned c = 0;
  constexpr int U = 8;   // loads in flight per thread
#pragma unroll 1
  for (int it0 = 0; it0 < F_IT; it0 += U) {
    int64_t cv[U];
    double vv[U];
    int64_t rv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = base + (it0 + u) * F_CT + threadIdx.x;
      const bool ok = i < n;
      cv[u] = ok ? col1[i] : 1;
      vv[u] = ok ? (zero_aware ? val[i] : 1.0) : 0.0;
      rv[u] = (ok && m.bc_shift < 0) ? row1[i] : 1;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (vv[u] != 0.0) {
        unsigned b;
        if (m.bc_shift >= 0) b = (unsigned)(fdiv(m.J1, (uint64_t)(cv[u] - 1)) >> m.bc_shift);
        else b = (unsigned)(entry_key(m, rv[u], cv[u]) >> m.s);
        atomicAdd(&h[b], 1u);
        ++c;
      }
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned t = 0;
    for (int w = 0; w < F_CT / 32; ++w) t += wsum[w];
    tkept[blockIdx.x] = t;
  }
  uint16_t* out = thist + (int64_t)blockIdx.x * nb;
  for (int i = threadIdx.x; i < nb; i += F_CT) out[i] = (uint16_t)h[i];
}

// ---------------- K2 -------------------------------------------------------
// per bucket (lane), 32 warps over contiguous tile segments, 8 loads in
// flight per lane: tile prefix of the bucket counts (toff, without the
// bucket start) and the bucket totals
__global__ void __launch_bounds__(1024) fast_scan_tiles(const uint16_t* __restrict__ thist,
                                                        int ntiles, int nb,
                                                        uint16_t* __restrict__ toff,
                                                        unsigned* __restrict__ tot) {
  __shared__ unsigned ssum[32][33];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int b = blockIdx.x * 32 + lane;
  const int seg = (ntiles + 31) / 32;
  const int t0 = warp * seg, t1 = min(ntiles, t0 + seg);
  constexpr int U = 8;
  unsigned s = 0;
  if (b < nb) {
    int t = t0;
    for (; t + U <= t1; t += U) {
      unsigned v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) v[u] = thist[(int64_t)(t + u) * nb + b];
#pragma unroll
      for (int u = 0; u < U; ++u) s += v[u];
    }
    for (; t < t1; ++t) s += thist[(int64_t)t * nb + b];
  }
  ssum[warp][lane] = s;
  __syncthreads();
  unsigned run = 0;
  for (int w = 0; w < warp; ++w) run += ssum[w][lane];
  if (b < nb) {
    int t = t0;
    for (; t + U <= t1; t += U) {
      unsigned v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) v[u] = thist[(int64_t)(t + u) * nb + b];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        toff[(int64_t)(t + u) * nb + b] = (uint16_t)run;
        run += v[u];
      }
    }
    for (; t < t1; ++t) {
      const int64_t o = (int64_t)t * nb + b;
      const unsigned v = thist[o];
      toff[o] = (uint16_t)run;
      run += v;
    }
    if (warp == 31) tot[b] = run;
  }
}

// bucket starts (exclusive scan of the totals), the largest bucket, kept
// offsets per tile and the kept total: one CTA
__global__ void __launch_bounds__(1024) fast_scan_buckets(const unsigned* __restrict__ tot, int nb,
                                                          const unsigned* __restrict__ tkept,
                                                          int ntiles,
                                                          int64_t* __restrict__ bstart,
                                                          int64_t* __restrict__ tkoff,
                                                          int64_t* __restrict__ info) {
  __shared__ int64_t sh[1024];
  __shared__ unsigned smax[32];
  auto scan = [&](auto get, auto put, int count, int64_t* total) {
    int64_t carry = 0;
    for (int base = 0; base < count; base += 1024) {
      const int i = base + threadIdx.x;
      const int64_t v = i < count ? get(i) : 0;
      sh[threadIdx.x] = v;
      __syncthreads();
      for (int o = 1; o < 1024; o <<= 1) {
        const int64_t add = threadIdx.x >= o ? sh[threadIdx.x - o] : 0;
        __syncthreads();
        sh[threadIdx.x] += add;
        __syncthreads();
      }
      if (i < count) put(i, carry + sh[threadIdx.x] - v);
      carry += sh[1023];
      __syncthreads();
    }
    if (total) *total = carry;
  };
  unsigned mx = 0;
  for (int i = threadIdx.x; i < nb; i += 1024) mx = max(mx, tot[i]);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if ((threadIdx.x & 31) == 0) smax[threadIdx.x >> 5] = mx;
  int64_t nk = 0;
  scan([&](int i) { return (int64_t)tot[i]; }, [&](int i, int64_t v) { bstart[i] = v; }, nb, nullptr);
  scan([&](int i) { return (int64_t)tkept[i]; }, [&](int i, int64_t v) { tkoff[i] = v; }, ntiles,
       &nk);
  if (threadIdx.x == 0) {
    unsigned m = 0;
    for (int w = 0; w < 32; ++w) m = max(m, smax[w]);
    info[0] = nk;
    info[1] = m;
  }
}

// ---------------- K3 -------------------------------------------------------
struct ScatterArgs {
  const int64_t* row1;
  const int64_t* col1;
  const double* val;
  int64_t n;
  KeyMap m;
  int nb, pbits;
  const uint16_t* thist;   // per tile and bucket: count (< 2^16: a tile holds 16K entries)
  const uint16_t* toff;    // per tile and bucket: offset inside the bucket (buckets
                           // above B_CAP < 2^16 entries never reach fast_scatter)
  const int64_t* bstart;
  const int64_t* tkoff;
  bool zeros;          // explicit zeros present: compact, write i1/j1/values
  int* zero_found;     // !zeros: set if a zero value turns up (rerun zero-aware)
  uint64_t* items;
  int64_t* i1;
  int64_t* j1;
  double* values;
};

constexpr size_t K3_SMEM = (size_t)F_TILE * (sizeof(uint64_t) + sizeof(uint16_t)) +
                           2 * (size_t)F_MAXB * sizeof(unsigned);

__global__ void __launch_bounds__(F_CT) fast_scatter(ScatterArgs a) {
  extern __shared__ __align__(16) unsigned char sm[];
  uint64_t* sitem = reinterpret_cast<uint64_t*>(sm);
  unsigned* loff = reinterpret_cast<unsigned*>(sm + (size_t)F_TILE * sizeof(uint64_t));
  unsigned* cur = loff + F_MAXB;
  uint16_t* sb = reinterpret_cast<uint16_t*>(cur + F_MAXB);
  __shared__ unsigned wpart[F_CT / 32];
  __shared__ unsigned s_total;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nb = a.nb;
  const uint16_t* hrow = a.thist + (int64_t)blockIdx.x * nb;
  // tile-local bucket offsets: exclusive scan of this tile's histogram row
  {
    constexpr int PER = F_MAXB / F_CT;   // 8 buckets per thread (nb <= 4096)
    unsigned v[PER], s = 0;
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      const int b = tid * PER + q;
      v[q] = b < nb ? hrow[b] : 0u;
      s += v[q];
    }
    unsigned inc = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned y = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += y;
    }
    if (lane == 31) wpart[warp] = inc;
    __syncthreads();
    unsigned wb = 0, tt = 0;
    for (int w = 0; w < F_CT / 32; ++w) { const unsigned x = wpart[w]; wb += w < warp ? x : 0; tt += x; }
    unsigned run = wb + inc - s;
#pragma unroll
    for (int q = 0; q < PER; ++q) {
      const int b = tid * PER + q;
      if (b < nb) { loff[b] = run; cur[b] = 0; }
      run += v[q];
    }
    if (tid == 0) s_total = tt;
  }
  __syncthreads();
  const int64_t base = blockIdx.x * (int64_t)F_TILE;
  int64_t kbase = a.zeros ? a.tkoff[blockIdx.x] : base;
  const uint64_t lowmask = a.m.s >= 64 ? ~0ull : ((1ull << a.m.s) - 1);
  constexpr int U = 8;   // rounds of loads in flight
  bool saw_zero = false;
#pragma unroll 1
  for (int it0 = 0; it0 < F_IT; it0 += U) {
    int64_t rr[U], cc[U];
    double vv[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = base + (it0 + u) * F_CT + tid;
      const bool ok = i < a.n;
      rr[u] = ok ? a.row1[i] : 1;
      cc[u] = ok ? a.col1[i] : 1;
      vv[u] = ok ? a.val[i] : 0.0;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = base + (it0 + u) * F_CT + tid;
      const bool ok = i < a.n;
      bool keep = ok && vv[u] != 0.0;
      int64_t pos = i;
      if (a.zeros) {
        // kept index in input order: ballot + warp prefix for this round
        const unsigned ball = __ballot_sync(0xffffffffu, keep);
        if (lane == 0) wpart[warp] = __popc(ball);
        __syncthreads();
        unsigned before = 0, tot = 0;
        for (int w = 0; w < F_CT / 32; ++w) { const unsigned x = wpart[w]; before += w < warp ? x : 0; tot += x; }
        pos = kbase + before + __popc(ball & lanemask_lt());
        kbase += tot;
        __syncthreads();
      } else if (ok && !keep) {
        saw_zero = true;   // counted as kept by fast_hist: the result is discarded
        keep = true;
      }
      if (keep) {
        const uint64_t r0 = (uint64_t)(rr[u] - 1), c0 = (uint64_t)(cc[u] - 1);
        const uint64_t br = fdiv(a.m.I1, r0), bc = fdiv(a.m.J1, c0);
        const uint64_t key = br + (uint64_t)a.m.nrb * bc;
        const unsigned b = (unsigned)(key >> a.m.s);
        const unsigned slot = atomicAdd(&cur[b], 1u);   // in-tile slot: order irrelevant
        const unsigned j = loff[b] + slot;
        MPO_DCHECK(b < (unsigned)a.nb && slot < a.thist[(int64_t)blockIdx.x * a.nb + b] &&
                   j < (unsigned)F_TILE);
        sitem[j] = ((key & lowmask) << a.pbits) | (uint64_t)pos;
        sb[j] = (uint16_t)b;
        if (a.zeros) {
          a.i1[pos] = (int64_t)(r0 - br * a.m.I1.d);
          a.j1[pos] = (int64_t)(c0 - bc * a.m.J1.d);
          a.values[pos] = vv[u];
        }
      }
    }
  }
  if (saw_zero) atomicOr(a.zero_found, 1);
  __syncthreads();
  // global start of this tile's run in each bucket (n < 2^31: fits 32 bits)
  const uint16_t* trow = a.toff + (int64_t)blockIdx.x * nb;
  for (int b = tid; b < nb; b += F_CT) cur[b] = (unsigned)(a.bstart[b] + trow[b]) - loff[b];
  __syncthreads();
  const unsigned cnt = s_total;
  for (unsigned j = tid; j < cnt; j += F_CT) {
    MPO_DCHECK(sb[j] < (unsigned)nb);
    a.items[cur[sb[j]] + j] = sitem[j];
  }
}

// ---------------- K4 -------------------------------------------------------
#ifdef MPO_CONV_PROF
// clock64 per phase of fast_bucket, summed over buckets (variant builds only:
// tools/build_variant.sh k4prof convert_fast.cu -DMPO_CONV_PROF)
__device__ unsigned long long g_k4prof[10];
#define K4MARK(i)                                                   \
  do {                                                              \
    __syncthreads();                                                \
    if (threadIdx.x == 0) {                                         \
      const long long t_ = clock64();                               \
      atomicAdd(&g_k4prof[i], (unsigned long long)(t_ - t_prev));   \
      t_prev = t_;                                                  \
    }                                                               \
  } while (0)
#else
#define K4MARK(i) do {} while (0)
#endif
struct BucketArgs {
  const uint64_t* items;
  const unsigned* tot;
  const int64_t* bstart;
  int nb, s, pbits;
  int gbits;   // > 0: group sort (the low key's top gbits select a group --
               // for the square 2^k plans the block column inside the bucket);
               // 0: LSD passes over all s bits
  unsigned* ticket;
  unsigned long long* status;
  int64_t* uniq;
  int64_t* ti;
  int64_t* rank_out;
};

constexpr size_t K4_SMEM = (size_t)B_CAP * sizeof(uint64_t) +
                           (size_t)B_W * B_R * sizeof(uint16_t) +
                           (size_t)(B_R + 1) * sizeof(unsigned) + (size_t)B_R;

// Stable counting pass over the bucket's items x (warp-contiguous: item
// j = warp * wlen + it * 32 + lane for it < reff; slots j >= cnt hold ~0 and
// so sort last) on the digit (x >> shift) & (2^nbits - 1), nbits <= B_RB:
// ranks from warp-private digit counters and a ballot multisplit (lanes with
// equal digits: AND of one ballot per digit bit), A receives the items in
// digit order with ties in their incoming order, x is reloaded from A, and
// dst0[0 .. 2^nbits] holds the digit starts (dst0[2^nbits] = total).
__device__ void stable_pass(uint64_t (&x)[B_IT], int reff, int shift, int nbits, uint64_t* A,
                            uint16_t* wh, unsigned* dst0, unsigned* wtot) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nbin = 1 << nbits;
  const unsigned dmask = (unsigned)nbin - 1u;
  const int wlen = reff * 32;
  for (int i = tid; i < B_W * nbin; i += B_CT) wh[i] = 0;
  __syncthreads();
  unsigned rk[B_IT / 2];
#pragma unroll
  for (int it = 0; it < B_IT; ++it) {
    if (it < reff) {
      const unsigned d = (unsigned)(x[it] >> shift) & dmask;
#ifdef K4_MATCH
      const unsigned peers = __match_any_sync(0xffffffffu, d);
#else
      unsigned peers = 0xffffffffu;
      for (int k = 0; k < nbits; ++k) {
        const bool bit = (d >> k) & 1u;
        const unsigned bt = __ballot_sync(0xffffffffu, bit);
        peers &= bit ? bt : ~bt;
      }
#endif
      const unsigned run = wh[warp * nbin + d];
      const unsigned r = run + __popc(peers & lanemask_lt());
      if (it & 1) rk[it >> 1] |= r << 16; else rk[it >> 1] = r;
      __syncwarp();
      if ((__ffs(peers) - 1) == lane) wh[warp * nbin + d] = (uint16_t)(run + __popc(peers));
      __syncwarp();
    }
  }
  __syncthreads();
  // per digit: exclusive prefix over the warps (in place) and the digit total
  for (int d = tid; d < nbin; d += B_CT) {
    unsigned acc = 0;
    for (int w = 0; w < B_W; ++w) {
      const unsigned v = wh[w * nbin + d];
      wh[w * nbin + d] = (uint16_t)acc;
      acc += v;
    }
    dst0[d] = acc;
  }
  __syncthreads();
  // exclusive scan of the nbin <= B_R digit totals, PD consecutive per thread
  {
    constexpr int PD = (B_R + B_CT - 1) / B_CT;
    unsigned v[PD], sum = 0;
#pragma unroll
    for (int q = 0; q < PD; ++q) {
      const int d = tid * PD + q;
      v[q] = d < nbin ? dst0[d] : 0u;
      sum += v[q];
    }
    unsigned inc = sum;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const unsigned y = __shfl_up_sync(0xffffffffu, inc, o);
      if (lane >= o) inc += y;
    }
    if (lane == 31) wtot[warp] = inc;
    __syncthreads();
    unsigned run = inc - sum;
    for (int w = 0; w < warp; ++w) run += wtot[w];
#pragma unroll
    for (int q = 0; q < PD; ++q) {
      const int d = tid * PD + q;
      if (d < nbin) dst0[d] = run;
      run += v[q];
    }
    if (tid == B_CT - 1) dst0[nbin] = run;
  }
  __syncthreads();
#pragma unroll
  for (int it = 0; it < B_IT; ++it) {
    if (it < reff) {
      const unsigned d = (unsigned)(x[it] >> shift) & dmask;
      const unsigned r = (it & 1) ? (rk[it >> 1] >> 16) : (rk[it >> 1] & 0xffffu);
      MPO_DCHECK(dst0[d] + wh[warp * nbin + d] + r < (unsigned)B_CAP);
      A[dst0[d] + wh[warp * nbin + d] + r] = x[it];
    }
  }
  __syncthreads();
#pragma unroll
  for (int it = 0; it < B_IT; ++it)
    if (it < reff) x[it] = A[warp * wlen + it * 32 + lane];
}

__global__ void __launch_bounds__(B_CT, B_MINB) fast_bucket(BucketArgs a) {
  extern __shared__ __align__(16) unsigned char sm[];
  uint64_t* A = reinterpret_cast<uint64_t*>(sm);
  uint16_t* wh = reinterpret_cast<uint16_t*>(sm + (size_t)B_CAP * sizeof(uint64_t));
  unsigned* dst0 = reinterpret_cast<unsigned*>(wh + B_W * B_R);
  unsigned char* gflag = reinterpret_cast<unsigned char*>(dst0 + B_R + 1);
  __shared__ unsigned s_b, wtot[B_W];
  __shared__ int s_big, s_fpw[B_W];
  __shared__ int64_t s_partw[B_W];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // buckets are taken in ticket order: every predecessor a look-back waits
  // for is resident or done
  if (tid == 0) s_b = atomicAdd(a.ticket, 1u);
  __syncthreads();
  const int b = (int)s_b;
  const int cnt = (int)a.tot[b];
  const int64_t start = a.bstart[b];
#ifdef MPO_CONV_PROF
  long long t_prev = clock64();
#endif
  // warp-contiguous layout over the rounds actually needed
  const int reff = (cnt + B_CT - 1) / B_CT;          // rounds per warp
  const int wlen = reff * 32;                        // items per warp
  // x = ~0: padding (no valid item is ~0: the host keeps s + pbits < 64)
  uint64_t x[B_IT];
#pragma unroll
  for (int it = 0; it < B_IT; ++it) {
    const int j = warp * wlen + it * 32 + lane;
    x[it] = (it < reff && j < cnt) ? a.items[start + j] : ~0ull;
  }
  const uint64_t* Aw = A + warp * wlen + lane;   // item it of this lane at Aw[it * 32]
  const bool lead = warp == 0 && lane == 0;      // item 0 of the bucket
  K4MARK(0);
  // Group sort: a stable counting pass on the low key's top gbits (for the
  // square 2^k plans: the block column inside the bucket) puts every block
  // column's items together in their fast_scatter order -- tile order, so
  // for row-sorted input already ordered by block row except for entries
  // of one column that met in the same tile.  Groups with a key inversion
  // are re-sorted by one warp each (rank sort on the whole item, items are
  // distinct: they carry their position); a flagged group above GMAX items
  // sends the bucket to the LSD passes.
  constexpr int GMAX = 64;
  bool sorted = false;
  if (a.gbits > 0) {
    const int G = 1 << a.gbits;
    const int gshift = a.pbits + a.s - a.gbits;
    stable_pass(x, reff, gshift, a.gbits, A, wh, dst0, wtot);
    K4MARK(1);
    for (int g = tid; g < G; g += B_CT) gflag[g] = 0;
    if (tid == 0) s_big = 0;
    __syncthreads();
    bool inv = false;
#pragma unroll
    for (int it = 0; it < B_IT; ++it) {
      if (it < reff && x[it] != ~0ull && !(it == 0 && lead)) {
        const uint64_t p = Aw[it * 32 - 1];
        if ((p >> gshift) == (x[it] >> gshift) && (p >> a.pbits) > (x[it] >> a.pbits)) {
          gflag[(unsigned)(x[it] >> gshift)] = 1;
          inv = true;
        }
      }
    }
    const int any_inv = __syncthreads_or(inv);
    K4MARK(2);
    if (any_inv) {
      for (int g = warp; g < G; g += B_W) {
        if (!gflag[g]) continue;
        const unsigned lo = dst0[g], n_g = min(dst0[g + 1], (unsigned)cnt) - lo;
        if (n_g > GMAX) {
          if (lane == 0) s_big = 1;
          continue;
        }
        if (n_g <= 32) {
          const uint64_t v = lane < (int)n_g ? A[lo + lane] : ~0ull;
          unsigned r = 0;
          for (int i = 0; i < (int)n_g; ++i) r += __shfl_sync(0xffffffffu, v, i) < v;
          __syncwarp();
          if (lane < (int)n_g) A[lo + r] = v;
        } else {
          const uint64_t v0 = A[lo + lane];
          const uint64_t v1 = lane + 32 < (int)n_g ? A[lo + lane + 32] : ~0ull;
          unsigned r0 = 0, r1 = 0;
          for (int i = 0; i < (int)n_g; ++i) {
            const uint64_t o = i < 32 ? __shfl_sync(0xffffffffu, v0, i & 31)
                                      : __shfl_sync(0xffffffffu, v1, i & 31);
            r0 += o < v0;
            r1 += o < v1;
          }
          __syncwarp();
          A[lo + r0] = v0;
          if (lane + 32 < (int)n_g) A[lo + r1] = v1;
        }
      }
      __syncthreads();
      if (!s_big) {
#pragma unroll
        for (int it = 0; it < B_IT; ++it)
          if (it < reff) x[it] = A[warp * wlen + it * 32 + lane];
      }
    }
    sorted = !s_big;
    __syncthreads();
    K4MARK(3);
  }
  const int npass = sorted ? 0 : (a.s + B_RB - 1) / B_RB;
  for (int pass = 0; pass < npass; ++pass)
    stable_pass(x, reff, a.pbits + pass * B_RB, min(B_RB, a.s - pass * B_RB), A, wh, dst0, wtot);
  if (!sorted && npass == 0) {   // one key per bucket: publish for the neighbour reads
#pragma unroll
    for (int it = 0; it < B_IT; ++it)
      if (it < reff) A[warp * wlen + it * 32 + lane] = x[it];
  }
  __syncthreads();
  K4MARK(4);
  // head flags in sorted order -> local ids (flags kept as a bit mask)
  unsigned mine = 0, hbits = 0;
#pragma unroll
  for (int it = 0; it < B_IT; ++it) {
    if (it < reff) {
      const bool head = x[it] != ~0ull &&
                        ((it == 0 && lead) || (Aw[it * 32 - 1] >> a.pbits) != (x[it] >> a.pbits));
      hbits |= (unsigned)head << it;
      mine += __popc(__ballot_sync(0xffffffffu, head));
    }
  }
  if (lane == 0) wtot[warp] = mine;
  __syncthreads();
  unsigned wbase = 0, U = 0;
  for (int w = 0; w < B_W; ++w) { const unsigned v = wtot[w]; wbase += w < warp ? v : 0; U += v; }
  K4MARK(5);
  // decoupled look-back over the preceding buckets (ticket order): the whole
  // CTA reads B_CT predecessors' status words per step -- the nearest
  // inclusive prefix is usually among the ~2 x 148 buckets in flight
  if (tid == 0) st_release(a.status + b, (b == 0 ? ST_PRE : ST_AGG) | (unsigned long long)U);
  int64_t prefix = 0;
  for (int top = b - 1; top >= 0;) {
    const int idx = top - tid;
    const unsigned long long v = idx >= 0 ? ld_relaxed(a.status + idx) : ST_PRE;
    const unsigned pre = __ballot_sync(0xffffffffu, (v & ST_PRE) != 0);
    if (lane == 0) s_fpw[warp] = pre ? warp * 32 + __ffs(pre) - 1 : B_CT;
    __syncthreads();
    int fp = B_CT;   // nearest predecessor with an inclusive prefix (B_CT: none in this step)
    for (int w = 0; w < B_W; ++w) fp = min(fp, s_fpw[w]);
    int64_t part = (tid <= fp && idx >= 0) ? (int64_t)(v & ST_VAL) : 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
    if (lane == 0) s_partw[warp] = part;
    // a predecessor up to fp has not published yet: read again
    if (__syncthreads_or(tid <= fp && v == 0)) continue;
    for (int w = 0; w < B_W; ++w) prefix += s_partw[w];
    __syncthreads();
    if (fp < B_CT) break;
    top -= B_CT;
  }
  if (tid == 0) {
    if (b > 0) st_release(a.status + b, ST_PRE | (unsigned long long)(prefix + U));
    if (b == a.nb - 1) *a.rank_out = prefix + U;
  }
  K4MARK(6);
  const int64_t P = prefix;
  const uint64_t pmask = (1ull << a.pbits) - 1;
  unsigned run = wbase;
#pragma unroll
  for (int it = 0; it < B_IT; ++it) {
    if (it < reff) {
      const bool head = (hbits >> it) & 1u;
      const unsigned ball = __ballot_sync(0xffffffffu, head);
      if (x[it] != ~0ull) {
        const int64_t id = P + run + __popc(ball & lanemask_lt()) + (head ? 1 : 0) - 1;
        MPO_DCHECK(id >= 0 && id < a.bstart[a.nb - 1] + a.tot[a.nb - 1]);
        MPO_DCHECK((int64_t)(x[it] & pmask) < a.bstart[a.nb - 1] + a.tot[a.nb - 1]);
        if (head) a.uniq[id] = (int64_t)(((uint64_t)b << a.s) | (x[it] >> a.pbits));
        a.ti[(int64_t)(x[it] & pmask)] = id;
      }
      run += __popc(ball);
    }
  }
  K4MARK(7);
}

__global__ void derive_entries(const int64_t* __restrict__ row1, const int64_t* __restrict__ col1,
                               int64_t n, FastDiv I1, FastDiv J1, int64_t* __restrict__ i1,
                               int64_t* __restrict__ j1) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t r0 = (uint64_t)(row1[e] - 1), c0 = (uint64_t)(col1[e] - 1);
    i1[e] = (int64_t)(r0 - fdiv(I1, r0) * I1.d);
    j1[e] = (int64_t)(c0 - fdiv(J1, c0) * J1.d);
  }
}

}  // namespace

bool convert_fast(cudaStream_t st, const int64_t* row1, const int64_t* col1, const double* val,
                  int64_t n, int64_t I1, int64_t J1, int64_t nrb, int64_t ncb, ConvLocal& c) {
  static const int off = std::getenv("MPO_B200_CONV_FAST")
                             ? std::atoi(std::getenv("MPO_B200_CONV_FAST")) == 0 : 0;
  if (off || n <= 0 || n > (int64_t)0x7fffffff) return false;
  const int kb = key_bits((uint64_t)(nrb * ncb - 1));
  // buckets: ~8K entries each on average (room for 2x skew below the
  // 16K on-chip capacity of a K4 CTA), a power of two no larger than the
  // key space
  int lgb = 0;
  while ((1 << lgb) < F_MAXB && ((int64_t)1 << lgb) * (B_CAP / 2) < n) ++lgb;
  lgb = std::min(lgb, kb);
  const int nb = 1 << lgb;
  const int s = kb - lgb;
  const int pbits = std::max(1, key_bits((uint64_t)(n - 1)));
  if (s + pbits >= 64) return false;   // ~0 is fast_bucket's padding sentinel
  KeyMap m{make_div(I1), make_div(J1), nrb, s, -1};
  const int lgr = key_bits((uint64_t)(nrb - 1));
  if ((nrb & (nrb - 1)) == 0 && s >= lgr) m.bc_shift = s - lgr;
  const int ntiles = (int)cdiv(n, F_TILE);
  static std::once_flag once[kMaxDevices];
  once_per_device(once, [] {
    CK(cudaFuncSetAttribute(fast_scatter, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)K3_SMEM));
    CK(cudaFuncSetAttribute(fast_bucket, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)K4_SMEM));
  });
  DBuf<uint16_t> thist((size_t)ntiles * nb, st), toff((size_t)ntiles * nb, st);
  DBuf<unsigned> tot(nb, st),
      tkept(ntiles, st);
  DBuf<int64_t> bstart(nb, st), tkoff(ntiles, st), info(2, st);
  DBuf<int> zflag(1, st);
  // first attempt assumes no explicit zeros (the common case: one read of
  // the values fewer); fast_scatter verifies and a zero triggers one rerun
  for (int zero_aware = 0; zero_aware < 2; ++zero_aware) {
    fast_hist<<<ntiles, F_CT, 0, st>>>(row1, col1, val, n, m, nb, zero_aware != 0, thist.get(),
                                       tkept.get());
    CK_LAUNCH();
    fast_scan_tiles<<<(nb + 31) / 32, 1024, 0, st>>>(thist.get(), ntiles, nb, toff.get(),
                                                     tot.get());
    CK_LAUNCH();
    fast_scan_buckets<<<1, 1024, 0, st>>>(tot.get(), nb, tkept.get(), ntiles, bstart.get(),
                                          tkoff.get(), info.get());
    CK_LAUNCH();
    note_launch(3);
    int64_t h[2] = {0, 0};
    CK(cudaMemcpyAsync(h, info.get(), sizeof(h), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    const int64_t nk = h[0];
    if (h[1] > B_CAP) return false;   // a bucket too large for one CTA: general path
    c.nkept = nk;
    c.ti.alloc(nk, st);
    if (nk == 0) { c.rank = 0; return true; }
    const bool zeros = nk < n;
    c.lazy = false;
    c.i1.reset();
    c.j1.reset();
    c.values.reset();
    if (zeros) {
      c.i1.alloc(nk, st);
      c.j1.alloc(nk, st);
      c.values.alloc(nk, st);
    } else {
      c.lazy = true;   // entries derivable from the input: materialised on demand
      c.src_row = row1;
      c.src_col = col1;
      c.src_val = val;
      c.I1 = I1;
      c.J1 = J1;
    }
    DBuf<uint64_t> items(nk, st);
    CK(cudaMemsetAsync(zflag.get(), 0, sizeof(int), st));
    ScatterArgs sa{row1, col1, val, n, m, nb, pbits, thist.get(), toff.get(), bstart.get(),
                   tkoff.get(), zeros, zflag.get(), items.get(), c.i1.get(), c.j1.get(),
                   c.values.get()};
    fast_scatter<<<ntiles, F_CT, K3_SMEM, st>>>(sa);
    CK_LAUNCH();
    c.uniq.alloc(nk, st);   // capacity: the block count is known after K4
    DBuf<unsigned> ticket(1, st);
    DBuf<unsigned long long> status(nb, st);
    DBuf<int64_t> rank(1, st);
    CK(cudaMemsetAsync(ticket.get(), 0, sizeof(unsigned), st));
    CK(cudaMemsetAsync(status.get(), 0, sizeof(unsigned long long) * nb, st));
    // group sort when the low key splits into a block-column part of at
    // most B_RB bits above the block-row bits (nrb a power of two)
    int gbits = 0;
    if ((nrb & (nrb - 1)) == 0 && s > lgr && s - lgr <= B_RB) gbits = s - lgr;
    BucketArgs ba{items.get(), tot.get(), bstart.get(), nb, s, pbits, gbits, ticket.get(),
                  status.get(), c.uniq.get(), c.ti.get(), rank.get()};
    fast_bucket<<<nb, B_CT, K4_SMEM, st>>>(ba);
    CK_LAUNCH();
    note_launch(1);
#ifdef MPO_CONV_PROF
    {
      unsigned long long hp[10];
      CK(cudaStreamSynchronize(st));
      CK(cudaMemcpyFromSymbol(hp, g_k4prof, sizeof(hp)));
      std::fprintf(stderr, "[k4prof] cycles/bucket: load %.0f group_pass %.0f check %.0f fixup %.0f "
                   "lsd %.0f heads %.0f lookback %.0f write %.0f\n", hp[0] / (double)nb,
                   hp[1] / (double)nb, hp[2] / (double)nb, hp[3] / (double)nb, hp[4] / (double)nb,
                   hp[5] / (double)nb, hp[6] / (double)nb, hp[7] / (double)nb);
      std::memset(hp, 0, sizeof(hp));
      CK(cudaMemcpyToSymbol(g_k4prof, hp, sizeof(hp)));
    }
#endif
    int zf = 0;
    CK(cudaMemcpyAsync(&c.rank, rank.get(), sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(&zf, zflag.get(), sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    if (!zf) return true;
  }
  throw std::runtime_error("convert_fast: zero-aware pass still saw unaccounted zeros");
}

void ensure_entries(cudaStream_t st, ConvLocal& c) {
  if (!c.lazy) return;
  const int64_t n = c.nkept;
  c.i1.alloc(n, st);
  c.j1.alloc(n, st);
  c.values.alloc(n, st);
  if (n > 0) {
    const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(n, 256), 148 * 16));
    derive_entries<<<grid, 256, 0, st>>>(c.src_row, c.src_col, n, make_div(c.I1),
                                         make_div(c.J1), c.i1.get(), c.j1.get());
    CK_LAUNCH();
    note_launch();
    CK(cudaMemcpyAsync(c.values.get(), c.src_val, sizeof(double) * n, cudaMemcpyDeviceToDevice,
                       st));
  }
  c.lazy = false;
}

}  // namespace mpob

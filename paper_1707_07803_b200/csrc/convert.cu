// Sparse -> MPO conversion structure on sm_100a (Algorithm 1,
// sparse.py:234-250 + _build_cores sparse.py:183-204).
//
//   1. compact: drop explicit zeros keeping input order (sparse.py:234),
//      split each 1-based coordinate into in-block offset and block
//      coordinate (i1 = r % I1, br = r / I1; same for columns,
//      sparse.py:240-242) and key the block column-block-major
//      (key = br + nrb * bc, sparse.py:245-246);
//   2. stable onesweep LSD radix sort of (key, position), 8-bit digits,
//      only the bits the key space needs (only the block-column bits when
//      the rows arrive non-decreasing);
//   3. segment: head flags -> block ids (np.unique's return_inverse,
//      sparse.py:247), sorted unique keys, ti scattered back to input order.
//
// HBM-bound integer work: no tensor cores, coalesced tile loads, grids in
// multiples of the SM count.  Ranks come from per-warp private shared-memory
// counters driven by __match_any_sync + popc and prefix sums in a fixed
// order; the few atomics (histogram counts, tile-id dispenser, decoupled
// look-back flags, the sortedness flag) compute order-independent values,
// so the output is bit-deterministic.
#include "common.cuh"
#include "convert.cuh"
#include "kernels.cuh"

namespace mpob {

namespace {

constexpr int CT = 256;              // threads per tile CTA
constexpr int ITEMS = 16;            // keys per thread
constexpr int TILE = CT * ITEMS;     // 4096 keys per tile
constexpr int WARPS = CT / 32;
constexpr int RADIX = 256;

__device__ __forceinline__ unsigned lanemask_lt() {
  unsigned m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// ---------------- exclusive scan of uint32 counts -> int64 offsets ----------
__global__ void scan_block_sums(const unsigned* in, int64_t n, int64_t per, int64_t* bsum) {
  __shared__ int64_t sh[CT];
  const int64_t b0 = blockIdx.x * per, b1 = min(n, b0 + per);
  int64_t s = 0;
  for (int64_t i = b0 + threadIdx.x; i < b1; i += CT) s += in[i];
  sh[threadIdx.x] = s;
  __syncthreads();
  for (int w = CT / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) sh[threadIdx.x] += sh[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) bsum[blockIdx.x] = sh[0];
}

__global__ void scan_top(int64_t* bsum, int nb, int64_t* total) {
  if (threadIdx.x == 0 && blockIdx.x == 0) {
    int64_t acc = 0;
    for (int i = 0; i < nb; ++i) { int64_t v = bsum[i]; bsum[i] = acc; acc += v; }
    *total = acc;
  }
}

__global__ void scan_down(const unsigned* in, int64_t n, int64_t per, const int64_t* bsum,
                          int64_t* out) {
  __shared__ int64_t sh[CT];
  const int64_t b0 = blockIdx.x * per, b1 = min(n, b0 + per);
  int64_t carry = bsum[blockIdx.x];
  for (int64_t base = b0; base < b1; base += CT) {
    int64_t i = base + threadIdx.x;
    int64_t v = i < b1 ? in[i] : 0;
    sh[threadIdx.x] = v;
    __syncthreads();
    for (int o = 1; o < CT; o <<= 1) {
      int64_t add = threadIdx.x >= o ? sh[threadIdx.x - o] : 0;
      __syncthreads();
      sh[threadIdx.x] += add;
      __syncthreads();
    }
    if (i < b1) out[i] = carry + sh[threadIdx.x] - v;
    carry += sh[CT - 1];
    __syncthreads();
  }
}

// ---------------- compaction + split + key ---------------------------------
__global__ void count_nonzero_tiles(const double* __restrict__ val,
                                    const int64_t* __restrict__ row1, int64_t n, unsigned* cnt,
                                    int* unsorted) {
  // kept-entry counts per tile, and whether the rows arrive non-decreasing
  // (then so do the block rows of the kept entries: the sort can skip them)
  __shared__ unsigned sh[WARPS];
  __shared__ int s_uns;
  if (threadIdx.x == 0) s_uns = 0;
  const int64_t base = blockIdx.x * (int64_t)TILE;
  unsigned c = 0;
  bool uns = false;
#pragma unroll
  for (int it = 0; it < ITEMS; ++it) {
    int64_t i = base + it * CT + threadIdx.x;
    if (i < n) {
      if (val[i] != 0.0) ++c;
      if (i > 0 && row1[i - 1] > row1[i]) uns = true;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = c;
  __syncthreads();
  if (uns) s_uns = 1;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned t = 0;
    for (int w = 0; w < WARPS; ++w) t += sh[w];
    cnt[blockIdx.x] = t;
    if (s_uns) atomicOr(unsorted, 1);
  }
}

struct SplitArgs {
  const int64_t* row1;
  const int64_t* col1;
  const double* val;
  int64_t n;
  const int64_t* tile_off;
  int64_t I1, J1, nrb;
  int64_t* i1;
  int64_t* j1;
  double* values;
  uint64_t* key;
  unsigned* pos;
  int64_t pos_base;   // global position of this shard's first kept entry
};

__global__ void split_keys(SplitArgs a) {
  __shared__ unsigned wsum[WARPS];
  const int64_t base = blockIdx.x * (int64_t)TILE;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int64_t out = a.tile_off[blockIdx.x];
  // items in order: round it covers [base + it*CT, base + (it+1)*CT)
  for (int it = 0; it < ITEMS; ++it) {
    int64_t i = base + it * CT + threadIdx.x;
    bool keep = i < a.n && a.val[i] != 0.0;
    unsigned ball = __ballot_sync(0xffffffffu, keep);
    if (lane == 0) wsum[warp] = __popc(ball);
    __syncthreads();
    unsigned before = 0, total = 0;
    for (int w = 0; w < WARPS; ++w) { if (w < warp) before += wsum[w]; total += wsum[w]; }
    if (keep) {
      int64_t o = out + before + __popc(ball & lanemask_lt());
      int64_t r0 = a.row1[i] - 1, c0 = a.col1[i] - 1;
      int64_t br = r0 / a.I1, bc = c0 / a.J1;
      a.i1[o] = r0 - br * a.I1;
      a.j1[o] = c0 - bc * a.J1;
      a.values[o] = a.val[i];
      a.key[o] = (uint64_t)(br + a.nrb * bc);
      a.pos[o] = (unsigned)o;
    }
    out += total;
    __syncthreads();
  }
}

// ---------------- radix sort ------------------------------------------------
// ---------------- onesweep LSD passes (decoupled look-back) ----------------
// One read of the keys computes the digit histograms of every pass; each
// pass is then ONE kernel: tiles take ids from an atomic counter (launch
// order, so a tile only ever waits on tiles already running), rank their
// keys exactly as radix_scatter does, publish per-digit tile counts and
// find their global per-digit offsets by looking back over the preceding
// tiles' published counts/prefixes.  The atomics only schedule and signal:
// ranks and offsets are the same as the two-kernel pass, so the sort stays
// stable and the output bit-deterministic.
constexpr int MAXPASS = 8;
// smaller tiles than the two-kernel passes: 8 keys per thread keep the
// kernel at <= 64 registers, 4 CTAs (32 warps) per SM to hide the loads
constexpr int OS_ITEMS = 8, OS_TILE = CT * OS_ITEMS, OS_WITEMS = 32 * OS_ITEMS;
constexpr size_t OS_SMEM = (size_t)OS_TILE * (sizeof(uint64_t) + sizeof(unsigned));
constexpr unsigned long long OS_AGG = 1ull << 62, OS_PRE = 2ull << 62,
                             OS_VAL = (1ull << 62) - 1;

__global__ void __launch_bounds__(CT) onesweep_hist(const uint64_t* __restrict__ key, int64_t n,
                                                    int npass, int shift0,
                                                    unsigned* __restrict__ part) {
  // histograms of the passes at shift0 + 8p, one read of the keys
  __shared__ unsigned h[MAXPASS][RADIX];
  for (int i = threadIdx.x; i < MAXPASS * RADIX; i += CT) (&h[0][0])[i] = 0;
  __syncthreads();
  // 8 keys per thread in flight per step (a one-load loop is latency-bound)
  constexpr int U = 8;
  const int64_t stride = (int64_t)gridDim.x * CT;
  for (int64_t i0 = blockIdx.x * (int64_t)CT + threadIdx.x; i0 < n; i0 += U * stride) {
    uint64_t k[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = i0 + u * stride;
      k[u] = i < n ? key[i] >> shift0 : ~0ull;
    }
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (k[u] != ~0ull)
        for (int p = 0; p < npass; ++p) atomicAdd(&h[p][(k[u] >> (8 * p)) & (RADIX - 1)], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < npass * RADIX; i += CT)
    part[(int64_t)blockIdx.x * npass * RADIX + i] = (&h[0][0])[i];
}

// per pass: digit totals summed over the histogram CTAs in a fixed order,
// then the exclusive scan over digits -> global digit offsets
__global__ void onesweep_offsets(const unsigned* __restrict__ part, int nblk, int npass,
                                 int64_t* __restrict__ doff) {
  __shared__ int64_t tot[RADIX];
  const int p = blockIdx.x, d = threadIdx.x;
  int64_t s = 0;
#pragma unroll 8
  for (int b = 0; b < nblk; ++b) s += part[((int64_t)b * npass + p) * RADIX + d];
  tot[d] = s;
  __syncthreads();
  // exclusive scan over the 256 digits (Hillis-Steele)
  for (int o = 1; o < RADIX; o <<= 1) {
    const int64_t add = d >= o ? tot[d - o] : 0;
    __syncthreads();
    tot[d] += add;
    __syncthreads();
  }
  doff[p * RADIX + d] = tot[d] - s;
}

__device__ __forceinline__ unsigned long long ld_volatile_u64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.volatile.global.u64 %0, [%1];" : "=l"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ void st_volatile_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.volatile.global.u64 [%0], %1;" ::"l"(p), "l"(v));
}

__global__ void __launch_bounds__(CT, 4) onesweep_scatter(
    const uint64_t* __restrict__ key, const unsigned* __restrict__ pay, int64_t n, int shift,
    const int64_t* __restrict__ doff, unsigned long long* status, unsigned* tile_ctr,
    uint64_t* __restrict__ key_out, unsigned* __restrict__ pay_out) {
  extern __shared__ __align__(16) unsigned char ssm[];
  uint64_t* skey = reinterpret_cast<uint64_t*>(ssm);
  unsigned* spay = reinterpret_cast<unsigned*>(ssm + (size_t)OS_TILE * sizeof(uint64_t));
  __shared__ unsigned wh[WARPS][RADIX];
  __shared__ unsigned dstart[RADIX];
  __shared__ int64_t tbase[RADIX];
  __shared__ unsigned s_tile;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) s_tile = atomicAdd(tile_ctr, 1u);
  for (int d = threadIdx.x; d < WARPS * RADIX; d += CT) (&wh[0][0])[d] = 0;
  __syncthreads();
  const int64_t tile = s_tile;
  const int64_t tstart = tile * OS_TILE;
  const int tcount = (int)((n - tstart) < OS_TILE ? (n - tstart) : OS_TILE);
  const int64_t wbase = tstart + warp * OS_WITEMS;
  uint64_t k[OS_ITEMS];
  unsigned pv[OS_ITEMS], rank[OS_ITEMS];
#pragma unroll
  for (int it = 0; it < OS_ITEMS; ++it) {
    const int64_t i = wbase + it * 32 + lane;
    const bool valid = i < n;
    k[it] = valid ? key[i] : 0;
    pv[it] = valid ? pay[i] : 0;
  }
#pragma unroll
  for (int it = 0; it < OS_ITEMS; ++it) {
    const bool valid = wbase + it * 32 + lane < n;
    unsigned dig = valid ? (unsigned)((k[it] >> shift) & (RADIX - 1)) : RADIX;
    unsigned peers = __match_any_sync(0xffffffffu, dig);
    int leader = __ffs(peers) - 1;
    unsigned run = valid ? wh[warp][dig] : 0;
    rank[it] = run + __popc(peers & lanemask_lt());
    __syncwarp();
    if (valid && lane == leader) wh[warp][dig] = run + __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  if (threadIdx.x < RADIX) {
    const int d = threadIdx.x;
    unsigned acc = 0;
    for (int w = 0; w < WARPS; ++w) { unsigned v = wh[w][d]; wh[w][d] = acc; acc += v; }
    dstart[d] = acc;
    // publish this tile's count, look back for the prefix, publish the prefix
    unsigned long long* st = status + tile * RADIX + d;
    int64_t prefix = 0;
    if (tile == 0) {
      st_volatile_u64(st, OS_PRE | (unsigned long long)acc);
    } else {
      st_volatile_u64(st, OS_AGG | (unsigned long long)acc);
      int64_t j = tile - 1;
      while (true) {
        const unsigned long long v = ld_volatile_u64(status + j * RADIX + d);
        if (v & OS_PRE) { prefix += (int64_t)(v & OS_VAL); break; }
        if (v & OS_AGG) { prefix += (int64_t)(v & OS_VAL); --j; }
      }
      st_volatile_u64(st, OS_PRE | (unsigned long long)(prefix + acc));
    }
    tbase[d] = doff[d] + prefix;
  }
  __syncthreads();
  {
    unsigned v = threadIdx.x < RADIX ? dstart[threadIdx.x] : 0;
    const unsigned orig = v;
    for (int o = 1; o < RADIX; o <<= 1) {
      unsigned add = (threadIdx.x >= o && threadIdx.x < RADIX) ? dstart[threadIdx.x - o] : 0;
      __syncthreads();
      if (threadIdx.x < RADIX) { v += add; dstart[threadIdx.x] = v; }
      __syncthreads();
    }
    if (threadIdx.x < RADIX) dstart[threadIdx.x] = v - orig;
  }
  __syncthreads();
#pragma unroll
  for (int it = 0; it < OS_ITEMS; ++it) {
    int64_t i = wbase + it * 32 + lane;
    if (i < n) {
      unsigned dig = (unsigned)((k[it] >> shift) & (RADIX - 1));
      unsigned lp = dstart[dig] + wh[warp][dig] + rank[it];
      skey[lp] = k[it];
      spay[lp] = pv[it];
    }
  }
  __syncthreads();
  for (int j = threadIdx.x; j < tcount; j += CT) {
    const uint64_t kk = skey[j];
    const unsigned dig = (unsigned)((kk >> shift) & (RADIX - 1));
    const int64_t o = tbase[dig] + (j - (int64_t)dstart[dig]);
    key_out[o] = kk;
    pay_out[o] = spay[j];
  }
}

// ---------------- segment / unique / inverse --------------------------------
__global__ void head_counts(const uint64_t* __restrict__ key, int64_t n, unsigned* cnt) {
  __shared__ unsigned sh[WARPS];
  const int64_t base = blockIdx.x * (int64_t)TILE;
  unsigned c = 0;
#pragma unroll
  for (int it = 0; it < ITEMS; ++it) {
    int64_t i = base + it * CT + threadIdx.x;
    if (i < n && (i == 0 || key[i] != key[i - 1])) ++c;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0) sh[threadIdx.x >> 5] = c;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned t = 0;
    for (int w = 0; w < WARPS; ++w) t += sh[w];
    cnt[blockIdx.x] = t;
  }
}

__global__ void __launch_bounds__(CT) assign_ids(const uint64_t* __restrict__ key,
                                                 const unsigned* __restrict__ pos, int64_t n,
                                                 const int64_t* __restrict__ tile_off,
                                                 int64_t* uniq, int64_t* ti, int64_t pos_base) {
  // items i = base + it*CT + t; every load is issued before any rank is
  // formed, and one barrier publishes the per-(item row, warp) head counts
  __shared__ unsigned wcnt[ITEMS][WARPS];
  const int64_t base = blockIdx.x * (int64_t)TILE;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint64_t k[ITEMS], kp[ITEMS];
  unsigned pv[ITEMS];
#pragma unroll
  for (int it = 0; it < ITEMS; ++it) {
    const int64_t i = base + it * CT + threadIdx.x;
    const bool valid = i < n;
    k[it] = valid ? key[i] : 0;
    kp[it] = (valid && i > 0) ? key[i - 1] : ~k[it];
    pv[it] = valid ? pos[i] : 0;
  }
  unsigned ball[ITEMS];
#pragma unroll
  for (int it = 0; it < ITEMS; ++it) {
    const int64_t i = base + it * CT + threadIdx.x;
    const bool head = i < n && k[it] != kp[it];
    ball[it] = __ballot_sync(0xffffffffu, head);
    if (lane == 0) wcnt[it][warp] = __popc(ball[it]);
  }
  __syncthreads();
  int64_t run = tile_off[blockIdx.x];  // heads strictly before this tile
#pragma unroll
  for (int it = 0; it < ITEMS; ++it) {
    unsigned before = 0, total = 0;
#pragma unroll
    for (int w = 0; w < WARPS; ++w) {
      const unsigned c = wcnt[it][w];
      before += (w < warp) ? c : 0;
      total += c;
    }
    const int64_t i = base + it * CT + threadIdx.x;
    if (i < n) {
      const bool head = (ball[it] >> lane) & 1u;
      // id = (#heads at or before i) - 1
      const int64_t id = run + before + __popc(ball[it] & lanemask_lt()) + (head ? 1 : 0) - 1;
      if (head) uniq[id] = (int64_t)k[it];
      ti[(int64_t)pv[it] - pos_base] = id;
    }
    run += total;
  }
}

__global__ void level_digits_kernel(const int64_t* __restrict__ uniq, int64_t rank, int64_t nrb,
                                    int64_t rdiv, int64_t rmod, int64_t cdiv_, int64_t cmod,
                                    int64_t* rowd, int64_t* cold) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < rank;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t u = uniq[t];
    int64_t br = u % nrb, bc = u / nrb;
    rowd[t] = (br / rdiv) % rmod;
    cold[t] = (bc / cdiv_) % cmod;
  }
}

int grid_tiles(int64_t n) { return (int)std::max<int64_t>(1, cdiv(n, TILE)); }

}  // namespace

void exclusive_scan_u32(cudaStream_t st, const unsigned* in, int64_t n, int64_t* out,
                        int64_t* total_dev) {
  const int64_t per = std::max<int64_t>(CT * 8, cdiv(n, 592));
  const int nb = (int)std::max<int64_t>(1, cdiv(n, per));
  DBuf<int64_t> bsum(nb, st);
  scan_block_sums<<<nb, CT, 0, st>>>(in, n, per, bsum.get());
  CK_LAUNCH();
  scan_top<<<1, 32, 0, st>>>(bsum.get(), nb, total_dev);
  CK_LAUNCH();
  scan_down<<<nb, CT, 0, st>>>(in, n, per, bsum.get(), out);
  CK_LAUNCH();
  note_launch(3);
}

int key_bits(uint64_t max_key) {
  int b = 0;
  while (b < 64 && (max_key >> b) != 0) ++b;
  return b;
}

void radix_sort_pairs(cudaStream_t st, uint64_t* key, unsigned* pay, int64_t n, int bits,
                      uint64_t* key_tmp, unsigned* pay_tmp, bool& result_in_tmp, int low_bits) {
  result_in_tmp = false;
  if (n <= 1 || bits == 0) return;
  // presorted low bits (the caller knows the keys are non-decreasing in
  // their low `low_bits` bits): a stable sort on the high bits alone yields
  // the full key order
  const int shift0 = (low_bits > 0 && low_bits < bits) ? low_bits : 0;
  const int npass = (bits - shift0 + 7) / 8;
  if (npass > MAXPASS) throw ValueError("sort key wider than 64 bits");
  const int64_t ntiles = cdiv(n, OS_TILE);
  static std::once_flag once[kMaxDevices];   // per device, thread-safe
  once_per_device(once, [] {
    CK(cudaFuncSetAttribute(onesweep_scatter, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)OS_SMEM));
  });
  const int hblk = (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(n, CT * 16), 148 * 4));
  DBuf<unsigned> part((size_t)hblk * npass * RADIX, st), ctr(npass, st);
  DBuf<int64_t> doff((size_t)npass * RADIX, st);
  CK(cudaMemsetAsync(ctr.get(), 0, sizeof(unsigned) * npass, st));
  onesweep_hist<<<hblk, CT, 0, st>>>(key, n, npass, shift0, part.get());
  CK_LAUNCH();
  onesweep_offsets<<<npass, RADIX, 0, st>>>(part.get(), hblk, npass, doff.get());
  CK_LAUNCH();
  note_launch(2);
  DBuf<unsigned long long> status((size_t)ntiles * RADIX, st);
  uint64_t *ks = key, *kd = key_tmp;
  unsigned *ps = pay, *pd = pay_tmp;
  for (int p = 0; p < npass; ++p) {
    CK(cudaMemsetAsync(status.get(), 0, sizeof(unsigned long long) * ntiles * RADIX, st));
    onesweep_scatter<<<(int)ntiles, CT, OS_SMEM, st>>>(ks, ps, n, shift0 + 8 * p,
                                                       doff.get() + p * RADIX, status.get(),
                                                       ctr.get() + p, kd, pd);
    CK_LAUNCH();
    note_launch();
    std::swap(ks, kd);
    std::swap(ps, pd);
    result_in_tmp = !result_in_tmp;
  }
}

ConvLocal convert_local(cudaStream_t st, const int64_t* row1, const int64_t* col1,
                        const double* val, int64_t n, int64_t I1, int64_t J1, int64_t nrb,
                        int64_t ncb) {
  ConvLocal c;
  if (n < 0) throw ValueError("negative nonzero count");
  if (convert_fast(st, row1, col1, val, n, I1, J1, nrb, ncb, c)) return c;
  const int64_t tiles = grid_tiles(n);
  DBuf<unsigned> cnt(tiles, st);
  DBuf<int64_t> toff(tiles, st), tot(1, st);
  DBuf<int> uns(1, st);
  int h_uns = 1;
  if (n > 0) {
    CK(cudaMemsetAsync(uns.get(), 0, sizeof(int), st));
    count_nonzero_tiles<<<(int)tiles, CT, 0, st>>>(val, row1, n, cnt.get(), uns.get());
    CK_LAUNCH();
    note_launch();
    exclusive_scan_u32(st, cnt.get(), tiles, toff.get(), tot.get());
    CK(cudaMemcpyAsync(&c.nkept, tot.get(), sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(&h_uns, uns.get(), sizeof(int), cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
  }
  const int64_t nk = c.nkept;
  c.i1.alloc(nk, st);
  c.j1.alloc(nk, st);
  c.values.alloc(nk, st);
  c.ti.alloc(nk, st);
  if (nk == 0) { c.rank = 0; return c; }
  DBuf<uint64_t> key(nk, st), key2(nk, st);
  DBuf<unsigned> pos(nk, st), pos2(nk, st);
  SplitArgs sa{row1, col1, val, n, toff.get(), I1, J1, nrb, c.i1.get(), c.j1.get(),
               c.values.get(), key.get(), pos.get(), 0};
  split_keys<<<(int)tiles, CT, 0, st>>>(sa);
  CK_LAUNCH();
  note_launch();
  const uint64_t max_key = (uint64_t)(nrb * ncb - 1);
  bool in_tmp = false;
  // rows non-decreasing and nrb a power of two: the keys (br + nrb bc) are
  // then non-decreasing in their low log2(nrb) bits, only the block-column
  // bits need sorting
  const int low = (!h_uns && (nrb & (nrb - 1)) == 0) ? key_bits((uint64_t)(nrb - 1)) : 0;
  radix_sort_pairs(st, key.get(), pos.get(), nk, key_bits(max_key), key2.get(), pos2.get(), in_tmp,
                   low);
  const uint64_t* sk = in_tmp ? key2.get() : key.get();
  const unsigned* sp = in_tmp ? pos2.get() : pos.get();
  const int64_t t2 = grid_tiles(nk);
  DBuf<unsigned> hc(t2, st);
  DBuf<int64_t> hoff(t2, st), htot(1, st);
  head_counts<<<(int)t2, CT, 0, st>>>(sk, nk, hc.get());
  CK_LAUNCH();
  note_launch();
  exclusive_scan_u32(st, hc.get(), t2, hoff.get(), htot.get());
  CK(cudaMemcpyAsync(&c.rank, htot.get(), sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  c.uniq.alloc(c.rank, st);
  assign_ids<<<(int)t2, CT, 0, st>>>(sk, sp, nk, hoff.get(), c.uniq.get(), c.ti.get(), 0);
  CK_LAUNCH();
  note_launch();
  return c;
}

void level_digits(cudaStream_t st, const int64_t* uniq, int64_t rank, int64_t nrb,
                  const std::vector<int64_t>& rf, const std::vector<int64_t>& cf, int level,
                  int64_t* rowd, int64_t* cold) {
  // digits of level k (1-based core index k >= 1), level-2 fastest (sparse.py:173-180)
  int64_t rdiv = 1, cdv = 1;
  for (int q = 1; q < level; ++q) { rdiv *= rf[q]; cdv *= cf[q]; }
  if (rank <= 0) return;
  int blocks = (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(rank, 256), 148 * 8));
  level_digits_kernel<<<blocks, 256, 0, st>>>(uniq, rank, nrb, rdiv, rf[level], cdv, cf[level],
                                               rowd, cold);
  CK_LAUNCH();
  note_launch();
}

}  // namespace mpob

// Sparse -> MPO conversion structure on sm_100a (Algorithm 1,
// sparse.py:234-250 + _build_cores sparse.py:183-204).
//
//   1. compact: drop explicit zeros keeping input order (sparse.py:234),
//      split each 1-based coordinate into in-block offset and block
//      coordinate (i1 = r % I1, br = r / I1; same for columns,
//      sparse.py:240-242) and key the block column-block-major
//      (key = br + nrb * bc, sparse.py:245-246);
//   2. stable LSD radix sort of (key, position), 8-bit digits, only the
//      bits the key space needs;
//   3. segment: head flags -> block ids (np.unique's return_inverse,
//      sparse.py:247), sorted unique keys, ti scattered back to input order.
//
// HBM-bound integer work: no tensor cores, coalesced tile loads, grids in
// multiples of the SM count, and no atomics anywhere (per-warp private
// shared-memory counters driven by __match_any_sync + popc, prefix sums
// over tiles in a fixed order), so the output is bit-deterministic.
#include "common.cuh"
#include "convert.cuh"
#include "kernels.cuh"

namespace mpob {

namespace {

constexpr int CT = 256;              // threads per tile CTA
constexpr int ITEMS = 16;            // keys per thread
constexpr int TILE = CT * ITEMS;     // 4096 keys per tile
constexpr int WARPS = CT / 32;
constexpr int WITEMS = 32 * ITEMS;   // keys per warp (512)
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
__global__ void count_nonzero_tiles(const double* __restrict__ val, int64_t n, unsigned* cnt) {
  __shared__ unsigned sh[WARPS];
  const int64_t base = blockIdx.x * (int64_t)TILE;
  unsigned c = 0;
#pragma unroll
  for (int it = 0; it < ITEMS; ++it) {
    int64_t i = base + it * CT + threadIdx.x;
    if (i < n && val[i] != 0.0) ++c;
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

// ---------------- radix sort passes ----------------------------------------
// warp-private digit counters, walked in item order (stable, atomics-free)
__global__ void radix_hist(const uint64_t* __restrict__ key, int64_t n, int shift,
                           unsigned* hist, int64_t ntiles) {
  __shared__ unsigned wh[WARPS][RADIX];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int d = threadIdx.x; d < WARPS * RADIX; d += CT) (&wh[0][0])[d] = 0;
  __syncthreads();
  const int64_t wbase = blockIdx.x * (int64_t)TILE + warp * WITEMS;
  // all loads in flight before the ranking loop (its __syncwarp()s are
  // memory fences that would otherwise expose one load latency per item)
  unsigned digs[ITEMS];
#pragma unroll
  for (int it = 0; it < ITEMS; ++it) {
    const int64_t i = wbase + it * 32 + lane;
    digs[it] = i < n ? (unsigned)((key[i] >> shift) & (RADIX - 1)) : RADIX;  // RADIX = invalid
  }
#pragma unroll
  for (int it = 0; it < ITEMS; ++it) {
    const unsigned dig = digs[it];
    const bool valid = dig < RADIX;
    unsigned peers = __match_any_sync(0xffffffffu, dig);
    int leader = __ffs(peers) - 1;
    if (valid && lane == leader) wh[warp][dig] += __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  for (int d = threadIdx.x; d < RADIX; d += CT) {
    unsigned s = 0;
    for (int w = 0; w < WARPS; ++w) s += wh[w][d];
    hist[(int64_t)d * ntiles + blockIdx.x] = s;   // digit-major for the scan
  }
}

// Stable scatter of one 8-bit digit pass.  Keys are ranked inside the tile
// (warp-private counters, then a digit-major prefix), staged in shared
// memory in digit order, and written out as contiguous per-digit runs so
// the global stores coalesce (a direct scatter would touch one 32-byte
// sector per 8-byte key).
constexpr size_t SCATTER_SMEM = (size_t)TILE * (sizeof(uint64_t) + sizeof(unsigned));

__global__ void __launch_bounds__(CT) radix_scatter(const uint64_t* __restrict__ key,
                                                    const unsigned* __restrict__ pay, int64_t n,
                                                    int shift, const int64_t* __restrict__ offs,
                                                    int64_t ntiles, uint64_t* __restrict__ key_out,
                                                    unsigned* __restrict__ pay_out) {
  extern __shared__ __align__(16) unsigned char ssm[];
  uint64_t* skey = reinterpret_cast<uint64_t*>(ssm);
  unsigned* spay = reinterpret_cast<unsigned*>(ssm + (size_t)TILE * sizeof(uint64_t));
  __shared__ unsigned wh[WARPS][RADIX];
  __shared__ unsigned dstart[RADIX];
  __shared__ int64_t tbase[RADIX];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int d = threadIdx.x; d < WARPS * RADIX; d += CT) (&wh[0][0])[d] = 0;
  for (int d = threadIdx.x; d < RADIX; d += CT) tbase[d] = offs[(int64_t)d * ntiles + blockIdx.x];
  __syncthreads();
  const int64_t tstart = blockIdx.x * (int64_t)TILE;
  const int tcount = (int)((n - tstart) < TILE ? (n - tstart) : TILE);
  const int64_t wbase = tstart + warp * WITEMS;
  uint64_t k[ITEMS];
  unsigned pv[ITEMS], rank[ITEMS];
#pragma unroll
  for (int it = 0; it < ITEMS; ++it) {   // all loads first (see radix_hist)
    const int64_t i = wbase + it * 32 + lane;
    const bool valid = i < n;
    k[it] = valid ? key[i] : 0;
    pv[it] = valid ? pay[i] : 0;
  }
#pragma unroll
  for (int it = 0; it < ITEMS; ++it) {
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
  // per digit: exclusive prefix over warps, and the digit's tile total
  if (threadIdx.x < RADIX) {
    const int d = threadIdx.x;
    unsigned acc = 0;
    for (int w = 0; w < WARPS; ++w) { unsigned v = wh[w][d]; wh[w][d] = acc; acc += v; }
    dstart[d] = acc;
  }
  __syncthreads();
  // exclusive scan of the 256 digit totals (Hillis-Steele, one value/thread)
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
  for (int it = 0; it < ITEMS; ++it) {
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

__global__ void assign_ids(const uint64_t* __restrict__ key, const unsigned* __restrict__ pos,
                           int64_t n, const int64_t* __restrict__ tile_off, int64_t* uniq,
                           int64_t* ti, int64_t pos_base) {
  __shared__ unsigned wsum[WARPS];
  const int64_t base = blockIdx.x * (int64_t)TILE;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int64_t run = tile_off[blockIdx.x];  // heads strictly before this tile
  for (int it = 0; it < ITEMS; ++it) {
    int64_t i = base + it * CT + threadIdx.x;
    bool valid = i < n;
    bool head = valid && (i == 0 || key[i] != key[i - 1]);
    unsigned ball = __ballot_sync(0xffffffffu, head);
    if (lane == 0) wsum[warp] = __popc(ball);
    __syncthreads();
    unsigned before = 0, total = 0;
    for (int w = 0; w < WARPS; ++w) { if (w < warp) before += wsum[w]; total += wsum[w]; }
    if (valid) {
      // id = (#heads at or before i) - 1
      int64_t id = run + before + __popc(ball & lanemask_lt()) + (head ? 1 : 0) - 1;
      if (head) uniq[id] = (int64_t)key[i];
      ti[(int64_t)pos[i] - pos_base] = id;
    }
    run += total;
    __syncthreads();
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
                      uint64_t* key_tmp, unsigned* pay_tmp, bool& result_in_tmp) {
  result_in_tmp = false;
  if (n <= 1 || bits == 0) return;
  const int64_t ntiles = cdiv(n, TILE);
  static const bool attr = [] {   // thread-safe one-time setup
    CK(cudaFuncSetAttribute(radix_scatter, cudaFuncAttributeMaxDynamicSharedMemorySize,
                            (int)SCATTER_SMEM));
    return true;
  }();
  (void)attr;
  DBuf<unsigned> hist((size_t)RADIX * ntiles, st);
  DBuf<int64_t> offs((size_t)RADIX * ntiles, st), total(1, st);
  uint64_t *ks = key, *kd = key_tmp;
  unsigned *ps = pay, *pd = pay_tmp;
  for (int shift = 0; shift < bits; shift += 8) {
    radix_hist<<<(int)ntiles, CT, 0, st>>>(ks, n, shift, hist.get(), ntiles);
    CK_LAUNCH();
    exclusive_scan_u32(st, hist.get(), RADIX * ntiles, offs.get(), total.get());
    radix_scatter<<<(int)ntiles, CT, SCATTER_SMEM, st>>>(ks, ps, n, shift, offs.get(), ntiles, kd,
                                                          pd);
    CK_LAUNCH();
    note_launch(2);
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
  const int64_t tiles = grid_tiles(n);
  DBuf<unsigned> cnt(tiles, st);
  DBuf<int64_t> toff(tiles, st), tot(1, st);
  if (n > 0) {
    count_nonzero_tiles<<<(int)tiles, CT, 0, st>>>(val, n, cnt.get());
    CK_LAUNCH();
    note_launch();
    exclusive_scan_u32(st, cnt.get(), tiles, toff.get(), tot.get());
    CK(cudaMemcpyAsync(&c.nkept, tot.get(), sizeof(int64_t), cudaMemcpyDeviceToHost, st));
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
  radix_sort_pairs(st, key.get(), pos.get(), nk, key_bits(max_key), key2.get(), pos2.get(), in_tmp);
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

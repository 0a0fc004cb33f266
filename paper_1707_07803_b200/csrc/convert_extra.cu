// Conversion helpers: densified cores (Mpo.densify of the SparseCore chain,
// mpo.py:184-197 over sparse.py:183-204) and the multi-GPU merge primitives
// (global sorted-unique of gathered block keys, binary-search lookup,
// id remap) used by the nnz-sharded conversion.
#include "common.cuh"
#include "convert.cuh"
#include "kernels.cuh"

namespace mpob {

namespace {

inline int gridn(int64_t n) {
  return (int)std::max<int64_t>(1, std::min<int64_t>(cdiv(n, 256), 148 * 16));
}

__global__ void scatter_core0(const int64_t* i1, const int64_t* j1, const int64_t* ti,
                              const double* v, int64_t n, int64_t I1, int64_t J1, double* out) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x)
    out[i1[e] + I1 * (j1[e] + J1 * ti[e])] = v[e];   // coordinates are unique: no accumulation
}

__global__ void scatter_core0_range(const int64_t* i1, const int64_t* j1, const int64_t* ti,
                                    const double* v, int64_t n, int64_t I1, int64_t J1,
                                    int64_t start, int64_t stop, double* out) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n;
       e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t t = ti[e];
    if (t >= start && t < stop) out[i1[e] + I1 * (j1[e] + J1 * (t - start))] = v[e];
  }
}

__global__ void scatter_selector(const int64_t* rowd, const int64_t* cold, int64_t rank,
                                 int64_t Ik, int64_t Jk, bool last, double* out) {
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < rank;
       t += (int64_t)gridDim.x * blockDim.x) {
    int64_t right = last ? 0 : t;
    out[t + rank * (rowd[t] + Ik * (cold[t] + Jk * right))] = 1.0;
  }
}

__global__ void i64_to_u64(const int64_t* in, int64_t n, uint64_t* out, unsigned* pos) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    out[i] = (uint64_t)in[i];
    pos[i] = (unsigned)i;
  }
}

__global__ void heads_flags(const uint64_t* key, int64_t n, unsigned* flag) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    flag[i] = (i == 0 || key[i] != key[i - 1]) ? 1u : 0u;
}

__global__ void write_heads(const uint64_t* key, const unsigned* flag, const int64_t* off,
                            int64_t n, int64_t* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    if (flag[i]) out[off[i]] = (int64_t)key[i];
}

__global__ void lookup_kernel(const int64_t* table, int64_t ntab, const int64_t* q, int64_t nq,
                              int64_t* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nq;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t x = q[i], lo = 0, hi = ntab;
    while (lo < hi) {
      int64_t mid = (lo + hi) >> 1;
      if (table[mid] < x) lo = mid + 1; else hi = mid;
    }
    out[i] = (lo < ntab && table[lo] == x) ? lo : -1;
  }
}

__global__ void search_kernel(const int64_t* table, int64_t ntab, const int64_t* q, int64_t nq,
                              int64_t offset, bool exact, int64_t* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nq;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t x = q[i], lo = 0, hi = ntab;
    while (lo < hi) {
      int64_t mid = (lo + hi) >> 1;
      if (table[mid] < x) lo = mid + 1; else hi = mid;
    }
    out[i] = (exact && !(lo < ntab && table[lo] == x)) ? -1 : lo + offset;
  }
}

__global__ void remap_kernel(const int64_t* map, int64_t* ti, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    ti[i] = map[ti[i]];
}

}  // namespace

void conv_dense_core(cudaStream_t st, const ConvLocal& c, const std::vector<int64_t>& rf,
                     const std::vector<int64_t>& cf, int level, double* out) {
  const int d = (int)rf.size();
  const int64_t rank = c.rank;
  int64_t nrb = 1;
  for (int q = 1; q < d; ++q) nrb *= rf[q];
  if (level == 0) {
    const int64_t sz = rf[0] * cf[0] * rank;
    fill_zero(st, out, sz);
    if (c.nkept) {
      scatter_core0<<<gridn(c.nkept), 256, 0, st>>>(c.i1.get(), c.j1.get(), c.ti.get(),
                                                   c.values.get(), c.nkept, rf[0], cf[0], out);
      CK_LAUNCH();
      note_launch();
    }
    return;
  }
  const bool last = level == d - 1;
  const int64_t sz = rank * rf[level] * cf[level] * (last ? 1 : rank);
  fill_zero(st, out, sz);
  DBuf<int64_t> rd(rank, st), cd(rank, st);
  level_digits(st, c.uniq.get(), rank, nrb, rf, cf, level, rd.get(), cd.get());
  scatter_selector<<<gridn(rank), 256, 0, st>>>(rd.get(), cd.get(), rank, rf[level], cf[level],
                                               last, out);
  CK_LAUNCH();
  note_launch();
}

void conv_chunk_core(cudaStream_t st, const ConvLocal& c, const std::vector<int64_t>& rf,
                     const std::vector<int64_t>& cf, int level, int64_t start, int64_t stop,
                     double* out) {
  const int d = (int)rf.size();
  const int64_t sub = stop - start;
  int64_t nrb = 1;
  for (int q = 1; q < d; ++q) nrb *= rf[q];
  if (level == 0) {
    fill_zero(st, out, rf[0] * cf[0] * sub);
    if (c.nkept) {
      scatter_core0_range<<<gridn(c.nkept), 256, 0, st>>>(c.i1.get(), c.j1.get(), c.ti.get(),
                                                         c.values.get(), c.nkept, rf[0], cf[0],
                                                         start, stop, out);
      CK_LAUNCH();
      note_launch();
    }
    return;
  }
  const bool last = level == d - 1;
  fill_zero(st, out, sub * rf[level] * cf[level] * (last ? 1 : sub));
  DBuf<int64_t> rd(sub, st), cd(sub, st);
  level_digits(st, c.uniq.get() + start, sub, nrb, rf, cf, level, rd.get(), cd.get());
  scatter_selector<<<gridn(sub), 256, 0, st>>>(rd.get(), cd.get(), sub, rf[level], cf[level],
                                              last, out);
  CK_LAUNCH();
  note_launch();
}

int64_t keys_unique(cudaStream_t st, const int64_t* keys, int64_t n, int64_t max_key,
                    int64_t* out) {
  if (n <= 0) return 0;
  DBuf<uint64_t> k1(n, st), k2(n, st);
  DBuf<unsigned> p1(n, st), p2(n, st), flag(n, st);
  i64_to_u64<<<gridn(n), 256, 0, st>>>(keys, n, k1.get(), p1.get());
  CK_LAUNCH();
  bool in_tmp = false;
  radix_sort_pairs(st, k1.get(), p1.get(), n, key_bits((uint64_t)max_key), k2.get(), p2.get(),
                   in_tmp);
  const uint64_t* sk = in_tmp ? k2.get() : k1.get();
  heads_flags<<<gridn(n), 256, 0, st>>>(sk, n, flag.get());
  CK_LAUNCH();
  DBuf<int64_t> off(n, st), tot(1, st);
  exclusive_scan_u32(st, flag.get(), n, off.get(), tot.get());
  write_heads<<<gridn(n), 256, 0, st>>>(sk, flag.get(), off.get(), n, out);
  CK_LAUNCH();
  note_launch(3);
  int64_t h = 0;
  CK(cudaMemcpyAsync(&h, tot.get(), sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return h;
}

void keys_lookup(cudaStream_t st, const int64_t* table, int64_t ntab, const int64_t* q, int64_t nq,
                 int64_t* out) {
  if (nq <= 0) return;
  lookup_kernel<<<gridn(nq), 256, 0, st>>>(table, ntab, q, nq, out);
  CK_LAUNCH();
  note_launch();
}

void keys_search(cudaStream_t st, const int64_t* table, int64_t ntab, const int64_t* q,
                 int64_t nq, int64_t offset, bool exact, int64_t* out) {
  if (nq <= 0) return;
  search_kernel<<<gridn(nq), 256, 0, st>>>(table, ntab, q, nq, offset, exact, out);
  CK_LAUNCH();
  note_launch();
}

void remap_ids(cudaStream_t st, const int64_t* map, int64_t* ti, int64_t n) {
  if (n <= 0) return;
  remap_kernel<<<gridn(n), 256, 0, st>>>(map, ti, n);
  CK_LAUNCH();
  note_launch();
}

}  // namespace mpob

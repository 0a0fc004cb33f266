// extern "C" boundary (include/mpo_b200.h): handles, argument validation,
// exception -> status-code mapping.  See the header for the reference
// functions each entry point replaces.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <mutex>
#include <cstring>
#include <string>

#include "convert.cuh"
#include "kernels.cuh"
#include "mpo_b200.h"
#include "tnrsvd.cuh"

#define MPO_API extern "C" __attribute__((visibility("default")))

namespace mpob {
unsigned long long g_launches = 0;
unsigned long long g_round_paths[5] = {0, 0, 0, 0, 0};
}

struct mpo_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
};

struct mpo_dev {
  mpob::Cores cores;
};

struct mpo_conv {
  mpob::ConvLocal c;
  std::vector<int64_t> rf, cf;
  int64_t nrb = 1;
};

namespace {

thread_local std::string g_err;

template <typename F>
int guarded(mpo_ctx* ctx, F&& f) {
  try {
    if (ctx) CK(cudaSetDevice(ctx->device));
    f();
    return MPO_OK;
  } catch (const mpob::ValueError& e) {
    g_err = e.what();
    return MPO_EVALUE;
  } catch (const mpob::OutOfMemory& e) {
    g_err = e.what();
    return MPO_ENOMEM;
  } catch (const mpob::CudaError& e) {
    g_err = e.what();
    return MPO_ECUDA;
  } catch (const std::bad_alloc& e) {
    g_err = "host allocation failed";
    return MPO_ENOMEM;
  } catch (const std::exception& e) {
    g_err = e.what();
    return MPO_EINTERNAL;
  }
}

void need(bool ok, const char* msg) {
  if (!ok) throw mpob::ValueError(msg);
}

cudaMemcpyKind kind_in(int from_host) {
  return from_host ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
}
cudaMemcpyKind kind_out(int to_host) {
  return to_host ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice;
}

mpo_dev* wrap(mpob::Cores&& c) {
  auto* m = new mpo_dev;
  m->cores = std::move(c);
  return m;
}

}  // namespace

MPO_API const char* mpo_b200_last_error(void) { return g_err.c_str(); }
MPO_API int mpo_b200_abi_version(void) { return 1; }
MPO_API unsigned long long mpo_b200_launch_count(void) { return mpob::g_launches; }
MPO_API int mpo_b200_round_paths(unsigned long long* out) {
  for (int i = 0; i < 5; ++i) out[i] = mpob::g_round_paths[i];
  return MPO_OK;
}

MPO_API int mpo_b200_profile_enable(int on) {
  mpob::g_prof.on = on != 0;
  mpob::g_prof.reset();
  return MPO_OK;
}

MPO_API int mpo_b200_profile_read(int which, double* ms, double* flops,
                                  unsigned long long* launches) {
  if (which < 0 || which >= mpob::KernelProfile::N) { g_err = "profile index out of range"; return MPO_EVALUE; }
  *ms = mpob::g_prof.ms[which];
  *flops = mpob::g_prof.flops[which];
  *launches = mpob::g_prof.launches[which];
  return MPO_OK;
}

MPO_API int mpo_ctx_create(int device, void* stream, mpo_ctx** out) {
  return guarded(nullptr, [&] {
    need(out != nullptr, "null output pointer");
    int n = 0;
    CK(cudaGetDeviceCount(&n));
    need(device >= 0 && device < n, "invalid CUDA device");
    CK(cudaSetDevice(device));
    // keep freed pool blocks cached: the sweeps allocate/free per bond
    cudaMemPool_t pool;
    CK(cudaDeviceGetDefaultMemPool(&pool, device));
    uint64_t thr = ~0ull;
    CK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
    // grow the pool once up front (MPO_B200_POOL_RESERVE_GB, default 8):
    // growing it mid-sweep maps new physical memory inside the timed path
    static std::once_flag reserved[64];
    std::call_once(reserved[device & 63], [&] {
      const char* e = std::getenv("MPO_B200_POOL_RESERVE_GB");
      const double gb = e ? std::atof(e) : 8.0;
      size_t fr = 0, tot = 0;
      CK(cudaMemGetInfo(&fr, &tot));
      const size_t want = std::min((size_t)(gb * (1ull << 30)), fr / 2);
      if (want > 0) {
        void* p = nullptr;
        CK(cudaMallocAsync(&p, want, nullptr));
        CK(cudaFreeAsync(p, nullptr));
        CK(cudaStreamSynchronize(nullptr));
      }
    });
    auto* c = new mpo_ctx;
    c->device = device;
    c->stream = static_cast<cudaStream_t>(stream);
    *out = c;
  });
}

MPO_API int mpo_ctx_set_stream(mpo_ctx* ctx, void* stream) {
  return guarded(ctx, [&] { ctx->stream = static_cast<cudaStream_t>(stream); });
}

MPO_API int mpo_ctx_synchronize(mpo_ctx* ctx) {
  return guarded(ctx, [&] { CK(cudaStreamSynchronize(ctx->stream)); });
}

MPO_API int mpo_ctx_destroy(mpo_ctx* ctx) {
  delete ctx;
  return MPO_OK;
}

// ---- MPO handles -------------------------------------------------------------
MPO_API int mpo_dev_create(mpo_ctx* ctx, int d, const int64_t* shapes, const double* const* cores,
                           int from_host, mpo_dev** out) {
  return guarded(ctx, [&] {
    need(d >= 1, "an MPO needs at least one core");
    mpob::Cores cs;
    for (int k = 0; k < d; ++k) {
      const int64_t* s = shapes + 4 * k;
      for (int q = 0; q < 4; ++q)
        if (s[q] < 1) throw mpob::ValueError("core " + std::to_string(k) + " has empty extent");
      mpob::Core c = mpob::make_core(ctx->stream, s[0], s[1], s[2], s[3]);
      CK(cudaMemcpyAsync(c.p(), cores[k], sizeof(double) * c.size(), kind_in(from_host),
                         ctx->stream));
      cs.push_back(std::move(c));
    }
    mpob::validate_chain(cs);
    *out = wrap(std::move(cs));
  });
}

// all cores from ONE packed buffer (F-ordered cores back to back): one H2D
// transfer and per-core device copies instead of one blocking pageable copy
// per core
MPO_API int mpo_dev_create_packed(mpo_ctx* ctx, int d, const int64_t* shapes, const double* packed,
                                  int from_host, mpo_dev** out) {
  return guarded(ctx, [&] {
    need(d >= 1, "an MPO needs at least one core");
    int64_t total = 0;
    for (int k = 0; k < d; ++k) {
      const int64_t* s = shapes + 4 * k;
      for (int q = 0; q < 4; ++q)
        if (s[q] < 1) throw mpob::ValueError("core " + std::to_string(k) + " has empty extent");
      total += s[0] * s[1] * s[2] * s[3];
    }
    cudaStream_t st = ctx->stream;
    mpob::DBuf<double> stage;
    const double* src = packed;
    if (from_host) {
      stage.alloc((size_t)total, st);
      CK(cudaMemcpyAsync(stage.get(), packed, sizeof(double) * total, cudaMemcpyHostToDevice, st));
      src = stage.get();
    }
    mpob::Cores cs;
    int64_t off = 0;
    for (int k = 0; k < d; ++k) {
      const int64_t* s = shapes + 4 * k;
      mpob::Core c = mpob::make_core(st, s[0], s[1], s[2], s[3]);
      CK(cudaMemcpyAsync(c.p(), src + off, sizeof(double) * c.size(), cudaMemcpyDeviceToDevice, st));
      off += c.size();
      cs.push_back(std::move(c));
    }
    mpob::validate_chain(cs);
    *out = wrap(std::move(cs));
  });
}

// every core into ONE packed buffer (F-ordered cores back to back): device
// copies into a staging buffer and a single D2H transfer
MPO_API int mpo_dev_copy_all(mpo_ctx* ctx, const mpo_dev* m, double* dst, int to_host) {
  return guarded(ctx, [&] {
    cudaStream_t st = ctx->stream;
    int64_t total = 0;
    for (const auto& c : m->cores) total += c.size();
    mpob::DBuf<double> stage;
    double* dev_dst = dst;
    if (to_host) {
      stage.alloc((size_t)total, st);
      dev_dst = stage.get();
    }
    int64_t off = 0;
    for (const auto& c : m->cores) {
      CK(cudaMemcpyAsync(dev_dst + off, c.p(), sizeof(double) * c.size(), cudaMemcpyDeviceToDevice,
                         st));
      off += c.size();
    }
    if (to_host) {
      CK(cudaMemcpyAsync(dst, stage.get(), sizeof(double) * total, cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
    }
  });
}

MPO_API int mpo_dev_num_cores(const mpo_dev* m, int* d) {
  *d = (int)m->cores.size();
  return MPO_OK;
}

MPO_API int mpo_dev_shapes(const mpo_dev* m, int64_t* shapes) {
  for (size_t k = 0; k < m->cores.size(); ++k) {
    const auto& c = m->cores[k];
    shapes[4 * k] = c.R; shapes[4 * k + 1] = c.I; shapes[4 * k + 2] = c.J; shapes[4 * k + 3] = c.S;
  }
  return MPO_OK;
}

MPO_API int mpo_dev_core_ptr(const mpo_dev* m, int k, const double** p) {
  if (k < 0 || k >= (int)m->cores.size()) { g_err = "core index out of range"; return MPO_EVALUE; }
  *p = m->cores[k].p();
  return MPO_OK;
}

MPO_API int mpo_dev_copy_core(mpo_ctx* ctx, const mpo_dev* m, int k, double* dst, int to_host) {
  return guarded(ctx, [&] {
    need(k >= 0 && k < (int)m->cores.size(), "core index out of range");
    const auto& c = m->cores[k];
    CK(cudaMemcpyAsync(dst, c.p(), sizeof(double) * c.size(), kind_out(to_host), ctx->stream));
    if (to_host) CK(cudaStreamSynchronize(ctx->stream));
  });
}

MPO_API int mpo_dev_free(mpo_dev* m) {
  delete m;
  return MPO_OK;
}

// ---- TNrSVD stages -----------------------------------------------------------
MPO_API int mpo_matmul(mpo_ctx* ctx, const mpo_dev* a, int ta, const mpo_dev* b, int tb,
                       mpo_dev** out) {
  return guarded(ctx, [&] { *out = wrap(mpob::matmul(ctx->stream, a->cores, ta, b->cores, tb)); });
}

MPO_API int mpo_transpose(mpo_ctx* ctx, const mpo_dev* a, mpo_dev** out) {
  return guarded(ctx, [&] { *out = wrap(mpob::transpose(ctx->stream, a->cores)); });
}

MPO_API int mpo_merge_leading_cores(mpo_ctx* ctx, const mpo_dev* m, int count, mpo_dev** out) {
  return guarded(ctx, [&] { *out = wrap(mpob::merge_leading(ctx->stream, m->cores, count)); });
}

MPO_API int mpo_qr(mpo_ctx* ctx, const mpo_dev* y, double tol, int has_tol, mpo_dev** q,
                   double* r_host) {
  return guarded(ctx, [&] {
    mpob::DBuf<double> r;
    mpob::Cores qc = mpob::qr(ctx->stream, y->cores, has_tol != 0, tol, &r);
    if (r_host && r.size())
      CK(cudaMemcpyAsync(r_host, r.get(), sizeof(double) * r.size(), cudaMemcpyDeviceToHost,
                         ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    *q = wrap(std::move(qc));
  });
}

MPO_API int mpo_svd(mpo_ctx* ctx, const mpo_dev* b, double tol, int has_tol, double* w_host,
                    double* s_host, mpo_dev** v) {
  return guarded(ctx, [&] {
    mpob::DBuf<double> w, s;
    mpob::Cores vc = mpob::svd(ctx->stream, b->cores, has_tol != 0, tol, w, s);
    if (w_host)
      CK(cudaMemcpyAsync(w_host, w.get(), sizeof(double) * w.size(), cudaMemcpyDeviceToHost,
                         ctx->stream));
    if (s_host)
      CK(cudaMemcpyAsync(s_host, s.get(), sizeof(double) * s.size(), cudaMemcpyDeviceToHost,
                         ctx->stream));
    CK(cudaStreamSynchronize(ctx->stream));
    *v = wrap(std::move(vc));
  });
}

MPO_API int mpo_subspace_iteration(mpo_ctx* ctx, const mpo_dev* a, const mpo_dev* o, int q,
                                   double tol, int has_tol, mpo_dev** out) {
  return guarded(ctx, [&] {
    *out = wrap(mpob::subspace_iteration(ctx->stream, a->cores, o->cores, q, has_tol != 0, tol));
  });
}

MPO_API int mpo_tnrsvd(mpo_ctx* ctx, const mpo_dev* am, const mpo_dev* o, int k_target, int q,
                       double tol, int has_tol, mpo_dev** u, double* s_host, mpo_dev** v) {
  return guarded(ctx, [&] {
    mpob::Cores uc, vc;
    std::vector<double> s;
    mpob::tnrsvd(ctx->stream, am->cores, o->cores, k_target, q, has_tol != 0, tol, uc, s, vc);
    std::memcpy(s_host, s.data(), sizeof(double) * s.size());
    *u = wrap(std::move(uc));
    *v = wrap(std::move(vc));
  });
}

MPO_API int mpo_round(mpo_ctx* ctx, const mpo_dev* m, double rel_tol, mpo_dev** out) {
  return guarded(ctx, [&] { *out = wrap(mpob::round_cores(ctx->stream, m->cores, rel_tol)); });
}

MPO_API int mpo_add(mpo_ctx* ctx, const mpo_dev* a, const mpo_dev* b, mpo_dev** out) {
  return guarded(ctx, [&] { *out = wrap(mpob::add(ctx->stream, a->cores, b->cores)); });
}

// ---- conversion --------------------------------------------------------------
MPO_API int mpo_sparse_convert(mpo_ctx* ctx, const int64_t* row1, const int64_t* col1,
                               const double* val, int64_t n, int from_host, int d,
                               const int64_t* rf, const int64_t* cf, mpo_conv** out) {
  return guarded(ctx, [&] {
    need(d >= 1, "factor lists must be non-empty and equal length");
    need(n >= 0, "negative entry count");
    auto* c = new mpo_conv;
    try {
      c->rf.assign(rf, rf + d);
      c->cf.assign(cf, cf + d);
      int64_t ncb = 1;
      for (int q = 1; q < d; ++q) { c->nrb *= rf[q]; ncb *= cf[q]; }
      const cudaStream_t st = ctx->stream;
      const int64_t* r = row1;
      const int64_t* cc = col1;
      const double* v = val;
      mpob::DBuf<int64_t> hr, hc;
      mpob::DBuf<double> hv;
      if (from_host && n > 0) {
        hr.alloc(n, st); hc.alloc(n, st); hv.alloc(n, st);
        CK(cudaMemcpyAsync(hr.get(), row1, sizeof(int64_t) * n, cudaMemcpyHostToDevice, st));
        CK(cudaMemcpyAsync(hc.get(), col1, sizeof(int64_t) * n, cudaMemcpyHostToDevice, st));
        CK(cudaMemcpyAsync(hv.get(), val, sizeof(double) * n, cudaMemcpyHostToDevice, st));
        r = hr.get(); cc = hc.get(); v = hv.get();
      }
      c->c = mpob::convert_local(st, r, cc, v, n, rf[0], cf[0], c->nrb, ncb);
      // lazily derived entries read the uploads: the handle keeps them
      c->c.own_row = std::move(hr);
      c->c.own_col = std::move(hc);
      c->c.own_val = std::move(hv);
    } catch (...) {
      delete c;
      throw;
    }
    *out = c;
  });
}

MPO_API int mpo_conv_info(const mpo_conv* c, int64_t* nkept, int64_t* rank) {
  if (nkept) *nkept = c->c.nkept;
  if (rank) *rank = c->c.rank;
  return MPO_OK;
}

MPO_API int mpo_conv_copy(mpo_ctx* ctx, const mpo_conv* c, int64_t* i1, int64_t* j1, int64_t* ti,
                          double* values, int64_t* uniq, int to_host) {
  return guarded(ctx, [&] {
    const cudaStream_t st = ctx->stream;
    const int64_t n = c->c.nkept, r = c->c.rank;
    if (i1 || j1 || values) mpob::ensure_entries(st, const_cast<mpo_conv*>(c)->c);
    auto cp = [&](void* dst, const void* src, size_t bytes) {
      if (dst && bytes) CK(cudaMemcpyAsync(dst, src, bytes, kind_out(to_host), st));
    };
    cp(i1, c->c.i1.get(), sizeof(int64_t) * n);
    cp(j1, c->c.j1.get(), sizeof(int64_t) * n);
    cp(ti, c->c.ti.get(), sizeof(int64_t) * n);
    cp(values, c->c.values.get(), sizeof(double) * n);
    cp(uniq, c->c.uniq.get(), sizeof(int64_t) * r);
    if (to_host) CK(cudaStreamSynchronize(st));
  });
}

MPO_API int mpo_conv_ptrs(mpo_ctx* ctx, const mpo_conv* c, int64_t** i1, int64_t** j1,
                          int64_t** ti, double** values, int64_t** uniq) {
  return guarded(ctx, [&] {
    auto& cl = const_cast<mpo_conv*>(c)->c;
    if (i1 || j1 || values) mpob::ensure_entries(ctx->stream, cl);
    if (i1) *i1 = cl.i1.get();
    if (j1) *j1 = cl.j1.get();
    if (ti) *ti = cl.ti.get();
    if (values) *values = cl.values.get();
    if (uniq) *uniq = cl.uniq.get();
  });
}

MPO_API int mpo_conv_level(mpo_ctx* ctx, const mpo_conv* c, int level, int64_t* rowd,
                           int64_t* cold, int to_host) {
  return guarded(ctx, [&] {
    need(level >= 1 && level < (int)c->rf.size(), "level out of range");
    const cudaStream_t st = ctx->stream;
    const int64_t r = c->c.rank;
    if (!to_host) {
      mpob::level_digits(st, c->c.uniq.get(), r, c->nrb, c->rf, c->cf, level, rowd, cold);
      return;
    }
    mpob::DBuf<int64_t> a(r, st), b(r, st);
    mpob::level_digits(st, c->c.uniq.get(), r, c->nrb, c->rf, c->cf, level, a.get(), b.get());
    if (r) {
      CK(cudaMemcpyAsync(rowd, a.get(), sizeof(int64_t) * r, cudaMemcpyDeviceToHost, st));
      CK(cudaMemcpyAsync(cold, b.get(), sizeof(int64_t) * r, cudaMemcpyDeviceToHost, st));
    }
    CK(cudaStreamSynchronize(st));
  });
}

MPO_API int mpo_conv_chunk(mpo_ctx* ctx, const mpo_conv* c, int64_t start, int64_t stop,
                           mpo_dev** out) {
  return guarded(ctx, [&] {
    need(start >= 0 && stop > start && stop <= c->c.rank, "chunk out of range");
    const int d = (int)c->rf.size();
    const int64_t sub = stop - start;
    mpob::ensure_entries(ctx->stream, const_cast<mpo_conv*>(c)->c);
    mpob::Cores cs;
    for (int k = 0; k < d; ++k) {
      mpob::Core core = k == 0 ? mpob::make_core(ctx->stream, 1, c->rf[0], c->cf[0], sub)
                               : mpob::make_core(ctx->stream, sub, c->rf[k], c->cf[k],
                                                 k == d - 1 ? 1 : sub);
      mpob::conv_chunk_core(ctx->stream, c->c, c->rf, c->cf, k, start, stop, core.p());
      cs.push_back(std::move(core));
    }
    *out = wrap(std::move(cs));
  });
}

MPO_API int mpo_conv_dense_core(mpo_ctx* ctx, const mpo_conv* c, int level, double* dst,
                                int to_host) {
  return guarded(ctx, [&] {
    const int d = (int)c->rf.size();
    need(level >= 0 && level < d, "level out of range");
    need(c->c.rank >= 1, "no blocks");
    const cudaStream_t st = ctx->stream;
    if (level == 0) mpob::ensure_entries(st, const_cast<mpo_conv*>(c)->c);
    const int64_t r = c->c.rank;
    int64_t sz = (level == 0) ? c->rf[0] * c->cf[0] * r
                              : r * c->rf[level] * c->cf[level] * (level == d - 1 ? 1 : r);
    if (!to_host) {
      mpob::conv_dense_core(st, c->c, c->rf, c->cf, level, dst);
      return;
    }
    mpob::DBuf<double> tmp(sz, st);
    mpob::conv_dense_core(st, c->c, c->rf, c->cf, level, tmp.get());
    CK(cudaMemcpyAsync(dst, tmp.get(), sizeof(double) * sz, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
  });
}

MPO_API int mpo_conv_free(mpo_conv* c) {
  delete c;
  return MPO_OK;
}

MPO_API int mpo_keys_unique(mpo_ctx* ctx, const int64_t* keys, int64_t n, int64_t max_key,
                            int64_t* out, int64_t* nuniq) {
  return guarded(ctx, [&] { *nuniq = mpob::keys_unique(ctx->stream, keys, n, max_key, out); });
}

MPO_API int mpo_keys_lookup(mpo_ctx* ctx, const int64_t* table, int64_t ntab, const int64_t* q,
                            int64_t nq, int64_t* out) {
  return guarded(ctx, [&] { mpob::keys_lookup(ctx->stream, table, ntab, q, nq, out); });
}

MPO_API int mpo_keys_search(mpo_ctx* ctx, const int64_t* table, int64_t ntab, const int64_t* q,
                            int64_t nq, int64_t offset, int exact, int64_t* out) {
  return guarded(ctx, [&] { mpob::keys_search(ctx->stream, table, ntab, q, nq, offset, exact != 0, out); });
}

MPO_API int mpo_remap_ids(mpo_ctx* ctx, const int64_t* map, int64_t* ti, int64_t n) {
  return guarded(ctx, [&] { mpob::remap_ids(ctx->stream, map, ti, n); });
}

// ---- dense factorisations of device matrices (column-major) -------------
// rsvd.py:106 / :128 on one shard of a row-distributed unfolding (the local
// step of distributed.tsqr / tsqr_svd)
MPO_API int mpo_dense_qr(mpo_ctx* ctx, int64_t m, int64_t n, const double* a, int64_t lda,
                         double* q, int64_t ldq, double* r, int64_t ldr) {
  return guarded(ctx, [&] {
    need(m >= n && n >= 1, "mpo_dense_qr: need m >= n >= 1");
    need(lda >= m && ldq >= m && ldr >= n, "mpo_dense_qr: leading dimension too small");
    cudaStream_t st = ctx->stream;
    mpob::DBuf<double> w((size_t)m * n, st);
    mpob::copy_matrix(st, m, n, a, lda, w.get(), m);
    if (!mpob::small_qr(st, m, n, w.get(), m, q, ldq, r, ldr))
      mpob::householder_qr(st, m, n, w.get(), m, q, ldq, r, ldr);
  });
}

// thin SVD M = U diag(s) Vt of an m x n device matrix (m >= n): s descending
// (n), U (m x n) orthonormal columns, Vt (n x n)
MPO_API int mpo_dense_svd(mpo_ctx* ctx, int64_t m, int64_t n, const double* a, int64_t lda,
                          double* s, double* u, int64_t ldu, double* vt, int64_t ldvt) {
  return guarded(ctx, [&] {
    need(m >= n && n >= 1, "mpo_dense_svd: need m >= n >= 1");
    need(lda >= m && ldu >= m && ldvt >= n, "mpo_dense_svd: leading dimension too small");
    cudaStream_t st = ctx->stream;
    mpob::SvdOut o;
    if (!mpob::small_svd(st, m, n, a, lda, o, 0.0)) mpob::svd_thin(st, m, n, a, lda, o, 0.0);
    CK(cudaMemcpyAsync(s, o.s.get(), sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
    // U = Ucarry diag(1/s), completed to orthonormal where s == 0
    mpob::DBuf<double> w((size_t)n * n, st);
    if (m == n) {
      mpob::svd_left_vectors(st, n, o.ucarry.get(), m, o.s.get(), w.get());
      mpob::copy_matrix(st, m, n, w.get(), n, u, ldu);
    } else {
      // tall: U = M Vt^T diag(1/s) would lose orthogonality for tiny s; QR of
      // M first (M = Qm Rm), then U = Qm U_R from the square factor's SVD
      mpob::DBuf<double> qm((size_t)m * n, st), rm((size_t)n * n, st), mc((size_t)m * n, st);
      mpob::copy_matrix(st, m, n, a, lda, mc.get(), m);
      mpob::householder_qr(st, m, n, mc.get(), m, qm.get(), m, rm.get(), n);
      mpob::SvdOut o2;
      if (!mpob::small_svd(st, n, n, rm.get(), n, o2, 0.0)) mpob::svd_thin(st, n, n, rm.get(), n, o2, 0.0);
      CK(cudaMemcpyAsync(s, o2.s.get(), sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
      mpob::svd_left_vectors(st, n, o2.ucarry.get(), n, o2.s.get(), w.get());
      mpob::dgemm(st, false, false, m, n, n, 1.0, qm.get(), m, w.get(), n, 0.0, u, ldu);
      o = std::move(o2);
    }
    mpob::copy_matrix(st, n, n, o.vh.get(), n, vt, ldvt);
  });
}

// C = alpha op(A) op(B) + beta C on device matrices (the DMMA GEMM)
MPO_API int mpo_dense_gemm(mpo_ctx* ctx, int ta, int tb, int64_t m, int64_t n, int64_t k,
                           double alpha, const double* a, int64_t lda, const double* b,
                           int64_t ldb, double beta, double* c, int64_t ldc) {
  return guarded(ctx, [&] {
    need(m >= 0 && n >= 0 && k >= 0, "mpo_dense_gemm: negative extent");
    mpob::dgemm(ctx->stream, ta != 0, tb != 0, m, n, k, alpha, a, lda, b, ldb, beta, c, ldc);
  });
}

// Device-resident MPO and the TNrSVD pipeline (rsvd.py), orchestrated in C++
// on the host; every FLOP runs in the sm_100a kernels of gemm/qr/svd/core_ops.
#pragma once

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "common.cuh"

namespace mpob {

struct Core {
  int64_t R = 1, I = 1, J = 1, S = 1;
  DBuf<double> buf;
  int64_t size() const { return R * I * J * S; }
  double* p() const { return buf.get(); }
};

using Cores = std::vector<Core>;

// MPO_B200_TRACE=1: per-call device timing of the dense factorizations
// (synchronises around each call; diagnostics only)
struct Trace {
  bool on;
  cudaStream_t st;
  const char* what;
  int64_t m, n;
  std::chrono::steady_clock::time_point t0;
  Trace(cudaStream_t s, const char* w, int64_t mm, int64_t nn) : st(s), what(w), m(mm), n(nn) {
    static const bool env = std::getenv("MPO_B200_TRACE") != nullptr;
    on = env;
    if (on) { cudaStreamSynchronize(st); t0 = std::chrono::steady_clock::now(); }
  }
  ~Trace() {
    if (!on) return;
    cudaStreamSynchronize(st);
    double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    fprintf(stderr, "[mpo_b200] %s %lldx%lld %.3f ms\n", what, (long long)m, (long long)n, ms);
  }
};

Core make_core(cudaStream_t st, int64_t R, int64_t I, int64_t J, int64_t S);
Cores clone(cudaStream_t st, const Cores& c);
void validate_chain(const Cores& c);  // Mpo.__init__ checks (mpo.py:124-145)

Cores matmul(cudaStream_t st, const Cores& a, bool ta, const Cores& b, bool tb);
Cores transpose(cudaStream_t st, const Cores& a);
Cores merge_leading(cudaStream_t st, const Cores& m, int count);
// mpo_qr: returns Q cores; R (K x K, column-major) into r_dev (device, K*K)
Cores qr(cudaStream_t st, const Cores& y, bool has_tol, double tol, DBuf<double>* r_out);
// mpo_svd: W (K x K device), s (K device), V cores (tall)
Cores svd(cudaStream_t st, const Cores& b, bool has_tol, double tol, DBuf<double>& w,
          DBuf<double>& s);
// mpo_qr(mpo_matmul(op(a), op(b))) with the product never materialised when
// round_tol > 0 (sweep.cu)
Cores qr_of_product(cudaStream_t st, const Cores& a, bool ta, const Cores& b, bool tb,
                    bool has_tol, double tol);
// Left-orthonormal chain of op(a)·op(b) (b != nullptr) or of *consume
// (moved from), bond ranks bounded by min(left, right extent) (sweep.cu)
Cores orthogonalize_product(cudaStream_t st, const Cores* a, bool ta, const Cores* b, bool tb,
                            Cores* consume);
bool fused_sweeps_enabled();   // MPO_B200_FUSED=0 restores the materialised sweeps
Cores subspace_iteration(cudaStream_t st, const Cores& a, const Cores& o, int q, bool has_tol,
                         double tol);
Cores round_cores(cudaStream_t st, const Cores& m, double rel_tol);
Cores add(cudaStream_t st, const Cores& a, const Cores& b);
void tnrsvd(cudaStream_t st, const Cores& am, const Cores& o, int k_target, int q, bool has_tol,
            double tol, Cores& u, std::vector<double>& s, Cores& v);

}  // namespace mpob

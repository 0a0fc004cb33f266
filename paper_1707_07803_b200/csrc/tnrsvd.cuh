// Device-resident MPO and the TNrSVD pipeline (rsvd.py), orchestrated in C++
// on the host; every FLOP runs in the sm_100a kernels of gemm/qr/svd/core_ops.
#pragma once

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
Cores subspace_iteration(cudaStream_t st, const Cores& a, const Cores& o, int q, bool has_tol,
                         double tol);
Cores round_cores(cudaStream_t st, const Cores& m, double rel_tol);
Cores add(cudaStream_t st, const Cores& a, const Cores& b);
void tnrsvd(cudaStream_t st, const Cores& am, const Cores& o, int k_target, int q, bool has_tol,
            double tol, Cores& u, std::vector<double>& s, Cores& v);

}  // namespace mpob

// Rank-bounded left-to-right orthogonalisation of an MPO that may be the
// unmaterialised per-core product op(A)·op(B) (rsvd.py:62-79 followed by
// rsvd.py:102-108 inside the rounding of rsvd.py:111-136).
//
// The reference materialises every product core (Ra·Rb, I, K, Sa·Sb) and
// QR-factors its unfoldings left to right, so its bond ranks after the L2R
// sweep are min(left extent, Ra·Rb) -- at config 5 (q = 1) the B = Q^T A
// cores reach (65536, 1, 2, 65536) = 34 GB each and the reference dies with
// a MemoryError.  Here:
//
//  1. an R2L pre-pass runs over the right end of the chain while it lowers
//     a bond rank below both the product rank and the left extent: each
//     step contracts the product core with the carried factor without
//     forming the core (two DMMA GEMMs); the transposed unfolding is wide
//     there, so the core becomes the identity and the unfolding itself is
//     carried on (no factorisation: a reduced QR would only add an
//     orthogonal gauge on the new bond), then
//  2. the L2R sweep contracts the carried factor into each product core
//     the same way (two GEMMs instead of materialise + GEMM) and
//     Householder-factors the tall unfoldings; wide ones again keep the
//     identity core and carry the unfolding.
//
// Every bond rank is then <= min(left extent, right extent, Ra·Rb), the
// exact rank bound; the chain is left-orthonormal exactly as after the
// reference's L2R sweep and represents the same tensor, so the truncating
// R2L SVD sweep that follows sees matrices with the same nonzero singular
// values (the reference's extra rank is numerically zero: singular values
// at O(eps·||B||), far below delta = tol·||B||/sqrt(d-1), and truncated by
// _truncation_rank, mpo.py:297-304).  Used only for round_tol > 0, where
// the output ranks are decided by truncation; round_tol None/0 keeps the
// reference's materialised sweep (its ranks then are the raw QR ranks).
#include <cstdlib>

#include "kernels.cuh"
#include "tnrsvd.cuh"

namespace mpob {

namespace {

// Logical view of one factor core: op(X) with extents (R, I, J, S); the
// physical storage is (R, I, J, S), or (R, J, I, S) when transposed.
struct Fac {
  const Core* c;
  bool t;
  int64_t R() const { return c->R; }
  int64_t I() const { return t ? c->J : c->I; }
  int64_t J() const { return t ? c->I : c->J; }
  int64_t S() const { return c->S; }
};

// Data of op(X) laid out as (R, p0, p1, S) where (p0, p1) = (I, J) if
// !swap else (J, I); copies only when both middle extents exceed 1.
const double* layout(cudaStream_t st, const Fac& f, bool swap, DBuf<double>& tmp) {
  // physical middle order is (I, J) if !f.t; we want logical (I, J) if !swap
  const bool phys_matches = (f.t == swap);
  if (phys_matches || f.c->I == 1 || f.c->J == 1) return f.c->p();
  tmp.alloc((size_t)f.c->size(), st);
  int64_t dims[4] = {f.c->R, f.c->I, f.c->J, f.c->S};
  int perm[4] = {0, 2, 1, 3};
  permute(st, f.c->p(), tmp.get(), 4, dims, perm);
  return tmp.get();
}

}  // namespace

// One entry of the chain: an explicit core, or the pair (op(a), op(b)).
struct PEntry {
  Core own;
  bool expl = true;
  Fac a{nullptr, false}, b{nullptr, false};
  int64_t R() const { return expl ? own.R : a.R() * b.R(); }
  int64_t I() const { return expl ? own.I : a.I(); }
  int64_t K() const { return expl ? own.J : b.J(); }
  int64_t S() const { return expl ? own.S : a.S() * b.S(); }
};

namespace {

// N (m, I, K, S) = C (m x R) x_1 P
Core left_absorb(cudaStream_t st, const double* C, int64_t m, const PEntry& e) {
  Core n = make_core(st, m, e.I(), e.K(), e.S());
  if (e.expl) {
    dgemm(st, false, false, m, e.I() * e.K() * e.S(), e.R(), 1.0, C, m, e.own.p(), e.R(), 0.0,
          n.p(), m);
    return n;
  }
  const int64_t Ra = e.a.R(), I = e.a.I(), Jc = e.a.J(), Sa = e.a.S();
  const int64_t Rb = e.b.R(), K = e.b.J(), Sb = e.b.S();
  DBuf<double> tb, ta;
  // B as (b, jc, k, b'), A as (a, jc, i, a')
  const double* Bu = layout(st, e.b, false, tb);
  const double* A2 = layout(st, e.a, true, ta);
  // T[x, a, jc, k, b'] = sum_b C[x, a, b] B[b, jc, k, b']
  DBuf<double> T((size_t)(m * Ra * Jc * K * Sb), st);
  dgemm(st, false, false, m * Ra, Jc * K * Sb, Rb, 1.0, C, m * Ra, Bu, Rb, 0.0, T.get(), m * Ra);
  // N[x, i, k, a', b'] = sum_{a, jc} T[x, a, jc, k, b'] A2[a, jc, i, a']
  const int64_t kc = Ra * Jc;
  if (K == 1) {
    dgemm(st, false, false, m, I * Sa, kc, 1.0, T.get(), m, A2, kc, 0.0, n.p(), m, Sb, m * kc, 0,
          m * I * Sa);
  } else {
    for (int64_t k = 0; k < K; ++k)
      for (int64_t i = 0; i < I; ++i)
        dgemm(st, false, false, m, Sa, kc, 1.0, T.get() + m * kc * k, m, A2 + kc * i, kc * I, 0.0,
              n.p() + m * (i + I * k), m * I * K, Sb, m * kc * K, 0, m * I * K * Sa);
  }
  return n;
}

double left_absorb_flops(const PEntry& e, int64_t m) {
  if (e.expl) return 2.0 * m * e.R() * e.I() * e.K() * e.S();
  const double Ra = e.a.R(), I = e.a.I(), Jc = e.a.J(), Sa = e.a.S();
  const double Rb = e.b.R(), K = e.b.J(), Sb = e.b.S();
  return 2.0 * m * Ra * Rb * Jc * K * Sb + 2.0 * m * Ra * Jc * I * Sa * K * Sb;
}

// contraction-order costs of right_absorb_t: B·L first or A·L first
void right_absorb_orders(const PEntry& e, int64_t r, double& f_bl, double& f_al) {
  const double Ra = e.a.R(), I = e.a.I(), Jc = e.a.J(), Sa = e.a.S();
  const double Rb = e.b.R(), K = e.b.J(), Sb = e.b.S();
  f_bl = 2.0 * (Rb * Jc * K * Sb * Sa * r + Ra * I * Jc * Sa * Rb * K * r);
  f_al = 2.0 * (Ra * I * Jc * Sa * Sb * r + Ra * I * Jc * Sb * r * Rb * K);
}

double right_absorb_flops(const PEntry& e, int64_t r) {
  if (e.expl) return 2.0 * e.R() * e.I() * e.K() * e.S() * r;
  double f_bl, f_al;
  right_absorb_orders(e, r, f_bl, f_al);
  return std::min(f_bl, f_al);
}

// Mt (I·K·r x R) = (P x_4 Lt^T)^T with Lt (r x S, ld r), i.e. the transposed
// unfolding of the core P·Lt^T that the pre-pass factors.
void right_absorb_t(cudaStream_t st, const PEntry& e, const double* Lt, int64_t r, double* Mt) {
  const int64_t R = e.R(), IK = e.I() * e.K(), S = e.S();
  if (e.expl) {
    // M (R·IK x r) = P (R·IK x S) · Lt^T, then transpose to (IK·r x R)
    DBuf<double> M((size_t)(R * IK * r), st);
    dgemm(st, false, true, R * IK, r, S, 1.0, e.own.p(), R * IK, Lt, r, 0.0, M.get(), R * IK);
    int64_t dims[3] = {R, IK, r};
    int perm[3] = {1, 2, 0};
    permute(st, M.get(), Mt, 3, dims, perm);
    return;
  }
  const int64_t Ra = e.a.R(), I = e.a.I(), Jc = e.a.J(), Sa = e.a.S();
  const int64_t Rb = e.b.R(), K = e.b.J(), Sb = e.b.S();
  DBuf<double> tb, ta;
  const double* Bu = layout(st, e.b, false, tb);   // (b, jc, k, b')
  const double* Au = layout(st, e.a, false, ta);   // (a, i, jc, a')
  // contraction order: B·L first (cost ~ Ra·I·Jc·Sa·Rb·K·r) or A·L first
  // (~ Ra·I·Jc·Sa·Sb·r); the latter wins when op(A) carries the large ranks
  // (B = Q^T A at config 5: Ra = Sa = 4096, Rb = Sb = 16)
  double f_bl, f_al;
  right_absorb_orders(e, r, f_bl, f_al);
  if (f_al < f_bl) {
    // V[a, i, jc, s, b'] = sum_a' A[a, i, jc, a'] Lt[s, a' + Sa·b']  (batched over b')
    DBuf<double> V((size_t)(Ra * I * Jc * r * Sb), st);
    dgemm(st, false, true, Ra * I * Jc, r, Sa, 1.0, Au, Ra * I * Jc, Lt, r, 0.0, V.get(),
          Ra * I * Jc, Sb, 0, r * Sa, Ra * I * Jc * r);
    // V'[a, i, s, jc, b']
    DBuf<double> Vp((size_t)(Ra * I * Jc * r * Sb), st);
    {
      int64_t dims[5] = {Ra, I, Jc, r, Sb};
      int perm[5] = {0, 1, 3, 2, 4};
      permute(st, V.get(), Vp.get(), 5, dims, perm);
    }
    V.reset();
    // Bv[jc, b', b, k] = B[b, jc, k, b']
    DBuf<double> Bv((size_t)(Rb * Jc * K * Sb), st);
    {
      int64_t dims[4] = {Rb, Jc, K, Sb};
      int perm[4] = {1, 3, 0, 2};
      permute(st, Bu, Bv.get(), 4, dims, perm);
    }
    // M''[a, i, s, b, k] = sum_{jc, b'} V'[a, i, s, jc, b'] Bv[jc, b', b, k]
    DBuf<double> Mpp((size_t)(Ra * I * r * Rb * K), st);
    dgemm(st, false, false, Ra * I * r, Rb * K, Jc * Sb, 1.0, Vp.get(), Ra * I * r, Bv.get(),
          Jc * Sb, 0.0, Mpp.get(), Ra * I * r);
    Vp.reset();
    // Mt[i, k, s, a, b]
    int64_t dims[5] = {Ra, I, r, Rb, K};
    int perm[5] = {1, 4, 2, 0, 3};
    permute(st, Mpp.get(), Mt, 5, dims, perm);
    return;
  }
  // L'[b', a', s] = Lt[s, a' + Sa·b']
  DBuf<double> Lp((size_t)(Sb * Sa * r), st);
  {
    int64_t dims[3] = {r, Sa, Sb};
    int perm[3] = {2, 1, 0};
    permute(st, Lt, Lp.get(), 3, dims, perm);
  }
  // U[b, jc, k, a', s] = sum_b' B[b, jc, k, b'] L'[b', a', s]
  DBuf<double> U((size_t)(Rb * Jc * K * Sa * r), st);
  dgemm(st, false, false, Rb * Jc * K, Sa * r, Sb, 1.0, Bu, Rb * Jc * K, Lp.get(), Sb, 0.0, U.get(),
        Rb * Jc * K);
  Lp.reset();
  // U'[jc, a', b, k, s]
  DBuf<double> Up((size_t)(Rb * Jc * K * Sa * r), st);
  {
    int64_t dims[5] = {Rb, Jc, K, Sa, r};
    int perm[5] = {1, 3, 0, 2, 4};
    permute(st, U.get(), Up.get(), 5, dims, perm);
  }
  U.reset();
  // M'[a, i, b, k, s] = sum_{jc, a'} A[a, i, jc, a'] U'[jc, a', b, k, s]
  DBuf<double> Mp((size_t)(Ra * I * Rb * K * r), st);
  dgemm(st, false, false, Ra * I, Rb * K * r, Jc * Sa, 1.0, Au, Ra * I, Up.get(), Jc * Sa, 0.0,
        Mp.get(), Ra * I);
  Up.reset();
  // Mt[i, k, s, a, b]
  int64_t dims[5] = {Ra, I, Rb, K, r};
  int perm[5] = {1, 3, 4, 0, 2};
  permute(st, Mp.get(), Mt, 5, dims, perm);
}

// Explicit (R, I, K, S) core of an entry (materialises a product core).
Core materialise(cudaStream_t st, const PEntry& e) {
  if (e.expl) {
    Core n = make_core(st, e.own.R, e.own.I, e.own.J, e.own.S);
    CK(cudaMemcpyAsync(n.p(), e.own.p(), sizeof(double) * e.own.size(), cudaMemcpyDeviceToDevice,
                       st));
    return n;
  }
  Core n = make_core(st, e.R(), e.I(), e.K(), e.S());
  CoreView va{e.a.c->p(), e.a.R(), e.a.I(), e.a.J(), e.a.S(), e.a.t};
  CoreView vb{e.b.c->p(), e.b.R(), e.b.I(), e.b.J(), e.b.S(), e.b.t};
  core_product(st, va, vb, n.p());
  return n;
}

int64_t sat_mul(int64_t x, int64_t y) {
  const int64_t cap = (int64_t)1 << 60;
  if (x >= cap || y >= cap || (double)x * (double)y >= (double)cap) return cap;
  return x * y;
}

}  // namespace

bool fused_sweeps_enabled() {
  static const bool on = std::getenv("MPO_B200_FUSED") ? std::atoi(std::getenv("MPO_B200_FUSED")) != 0
                                                       : true;
  return on;
}

Cores orthogonalize_product(cudaStream_t st, const Cores* a, bool ta, const Cores* b, bool tb,
                            Cores* consume) {
  std::vector<PEntry> P;
  size_t d;
  if (b) {
    if (a->size() != b->size()) throw ValueError("operands must have the same number of cores");
    d = a->size();
    P.resize(d);
    for (size_t k = 0; k < d; ++k) {
      P[k].expl = false;
      P[k].a = Fac{&(*a)[k], ta};
      P[k].b = Fac{&(*b)[k], tb};
      if (P[k].a.J() != P[k].b.I()) throw ValueError("inner dims differ per core");
    }
  } else {
    d = consume->size();
    P.resize(d);
    for (size_t k = 0; k < d; ++k) P[k].own = std::move((*consume)[k]);
  }
  Cores out(d);
  if (d == 1) {
    out[0] = materialise(st, P[0]);
    return out;
  }
  // left extents at each bond: left[j] = prod_{i <= j} I_i K_i
  std::vector<int64_t> left(d);
  for (size_t k = 0; k < d; ++k)
    left[k] = sat_mul(k ? left[k - 1] : 1, P[k].I() * P[k].K());

  // 1. R2L pre-pass while it lowers the bond rank below min(R, left extent)
  DBuf<double> Lt;          // carried factor (rr x S_meet), rows = reduced rank
  int64_t rr = 1;           // reduced rank of the bond right of the meeting core
  size_t meet = d - 1;      // cores > meet are explicit and right-reduced
  for (size_t j = d - 1; j >= 1; --j) {
    const int64_t IK = P[j].I() * P[j].K(), R = P[j].R();
    const int64_t nr = IK * rr;
    if (std::getenv("MPO_B200_TRACE"))
      fprintf(stderr, "[mpo_b200]   pre-pass core %zu: R %lld IK %lld rr %lld left %lld -> %s\n", j,
              (long long)R, (long long)IK, (long long)rr, (long long)left[j - 1],
              (nr < R && nr < left[j - 1]) ? "reduce" : "stop");
    if (!(nr < R && nr < left[j - 1])) break;
    DBuf<double> Mt((size_t)(nr * R), st);
    if (j == d - 1) {
      Core m = materialise(st, P[j]);   // (R, IK, 1) -> transpose
      int64_t dims[2] = {R, IK};
      int perm[2] = {1, 0};
      permute(st, m.p(), Mt.get(), 2, dims, perm);
    } else {
      Trace tr(st, "pre_absorb", R, nr);
      right_absorb_t(st, P[j], Lt.get(), rr, Mt.get());
    }
    // Mt (nr x R) is wide (nr < R): its row space already has an orthonormal
    // basis of size nr -- the identity -- so the rank reduction needs no
    // factorisation: core j <- I_nr as (nr, I, K, rr) (right-orthonormal),
    // Lt <- Mt.  The reference's reduced QR (Q^T, R) of the same wide
    // unfolding differs only by an orthogonal nr x nr gauge on the new bond.
    Core c = make_core(st, nr, P[j].I(), P[j].K(), rr);
    set_identity(st, nr, nr, c.p(), nr);
    P[j].expl = true;
    P[j].own = std::move(c);
    Lt = std::move(Mt);
    rr = nr;
    meet = j - 1;
  }

  // 2. L2R QR sweep; the meeting core absorbs Lt on its right.  The explicit
  // Q of each step is only read after the sweep: it is formed on the Q stream
  // while the next step's absorb and latency-bound panels run (joined on exit).
  DeferredQScope qscope(st);
  DBuf<double> C;   // carried R (m x R_k)
  int64_t m = 1;
  for (size_t k = 0; k < d; ++k) {
    const bool is_meet = (k == meet) && (meet < d - 1);
    Core n;
    if (k == 0 && !is_meet) {
      n = materialise(st, P[0]);
    } else if (!is_meet) {
      Trace tr(st, "l2r_absorb", m, P[k].S());
      n = left_absorb(st, C.get(), m, P[k]);
    } else {
      Trace tr(st, "meet_absorb", m, rr);
      // pick the smaller intermediate: P x_4 Lt^T (R·IK·rr) or C x_1 P (m·IK·S)
      const int64_t IK = P[k].I() * P[k].K();
      const int64_t R = P[k].R(), S = P[k].S();
      const double f_right = right_absorb_flops(P[k], rr) + 2.0 * m * IK * rr * R;
      const double f_left = left_absorb_flops(P[k], m) + 2.0 * m * IK * S * rr;
      const bool right_first = (k == 0) || f_right <= f_left;
      if (tr.on)
        fprintf(stderr, "[mpo_b200]   meet core %zu of %zu: m %lld R %lld IK %lld S %lld rr %lld, "
                "right-first %.3g flops, left-first %.3g flops\n", k, d, (long long)m, (long long)R,
                (long long)IK, (long long)S, (long long)rr, f_right, f_left);
      if (right_first) {
        DBuf<double> Mt((size_t)(IK * rr * R), st);
        right_absorb_t(st, P[k], Lt.get(), rr, Mt.get());
        if (k == 0) {
          // R = 1: Mt (IK·rr x 1) is the core (1, I, K, rr) itself
          n = make_core(st, 1, P[k].I(), P[k].K(), rr);
          CK(cudaMemcpyAsync(n.p(), Mt.get(), sizeof(double) * IK * rr, cudaMemcpyDeviceToDevice,
                             st));
        } else {
          // N (m x IK·rr) = C (m x R) · Mt^T
          n = make_core(st, m, P[k].I(), P[k].K(), rr);
          dgemm(st, false, true, m, IK * rr, R, 1.0, C.get(), m, Mt.get(), IK * rr, 0.0, n.p(), m);
        }
      } else {
        Core t = left_absorb(st, C.get(), m, P[k]);   // (m, I, K, S)
        n = make_core(st, m, P[k].I(), P[k].K(), rr);
        dgemm(st, false, true, m * IK, rr, S, 1.0, t.p(), m * IK, Lt.get(), rr, 0.0, n.p(), m * IK);
      }
      Lt.reset();
    }
    C.reset();
    if (P[k].expl) P[k].own = Core();   // release the consumed input
    if (k == d - 1) {
      out[k] = std::move(n);
      break;
    }
    const int64_t rows = n.R * n.I * n.J, cols = n.S, kk = std::min(rows, cols);
    Core q = make_core(st, n.R, n.I, n.J, kk);
    if (rows <= cols) {
      // wide unfolding: the identity is an orthonormal basis of its column
      // space -- core k <- I, the unfolding itself is the carried factor
      // (the reduced QR would only add an orthogonal gauge on the bond)
      set_identity(st, rows, rows, q.p(), rows);
      out[k] = std::move(q);
      C = std::move(n.buf);
      m = rows;
      continue;
    }
    DBuf<double> rm((size_t)(kk * cols), st);
    {
      Trace tr(st, "l2r_qr", rows, cols);
      householder_qr(st, rows, cols, n.p(), rows, q.p(), rows, rm.get(), kk, /*defer_q=*/true);
    }
    out[k] = std::move(q);
    C = std::move(rm);
    m = kk;
  }
  return out;
}

}  // namespace mpob

"""Generate the golden fixtures by running the UNMODIFIED reference package.

Run in the build container only (the reference does not travel to the GPU
box):  PYTHONPATH=/root/reference/pkg/src python tests/golden/make_golden.py

Every fixture stores the inputs (or the seeds + generator recipe) and the
reference's outputs, so the oracle restatement (oracle/mposvd_oracle.py)
and the CUDA path can both be checked against them without the reference.
"""

from __future__ import annotations

import math
import os
import sys

import numpy as np

sys.path.insert(0, os.environ.get("MPOSVD_REF", "/root/reference/pkg/src"))
import mposvd  # noqa: E402  (the reference, imported read-only)
from mposvd import mpo as rmpo  # noqa: E402
from mposvd import rsvd as rrsvd  # noqa: E402
from mposvd import sparse as rsparse  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def pack_cores(prefix, cores, out):
    out[f"{prefix}_n"] = np.array(len(cores))
    for k, c in enumerate(cores):
        out[f"{prefix}_{k}"] = np.asarray(c, dtype=np.float64)


def conv_case(name, coo, plan):
    m = rsparse.matrix_to_mpo(coo, plan, densify_limit=0)
    out = {
        "rows": np.array(coo.rows), "cols": np.array(coo.cols),
        "row": coo.row, "col": coo.col, "val": coo.val,
        "row_factors": np.array(plan.row_factors),
        "col_factors": np.array(plan.col_factors),
        "ranks": np.array(m.ranks),
    }
    c0 = m.cores[0]
    if isinstance(c0, rmpo.SparseCore):
        out["i1"], out["j1"], out["ti"] = c0.row, c0.col, c0.right
        out["values"] = c0.values
        for k, c in enumerate(m.cores[1:], start=1):
            out[f"lvl{k}_row"], out[f"lvl{k}_col"] = c.row, c.col
    dense = rsparse.matrix_to_mpo(coo, plan)
    if not dense.is_sparse:
        pack_cores("dense", dense.cores, out)
    np.savez_compressed(os.path.join(HERE, f"conv_{name}.npz"), **out)


def band_scatter(n, extra, seed):
    """Tridiagonal band + uniform scatter, duplicates merged by summation
    (config 4's recipe at a desk-scale size)."""
    rng = np.random.default_rng(seed)
    main = np.arange(n)
    r = np.concatenate([main, main[:-1], main[1:]])
    c = np.concatenate([main, main[1:], main[:-1]])
    v = rng.standard_normal(r.size)
    rr = rng.integers(0, n, extra)
    cc = rng.integers(0, n, extra)
    vv = rng.standard_normal(extra)
    r = np.concatenate([r, rr]); c = np.concatenate([c, cc]); v = np.concatenate([v, vv])
    key = r * n + c
    uk, inv = np.unique(key, return_inverse=True)
    vs = np.zeros(uk.size)
    np.add.at(vs, inv, v)
    return rsparse.SparseMatrixCoo(n, n, uk // n + 1, uk % n + 1, vs)


def svd_case(name, a_cores, k, q, tol, os_, seed):
    a = rmpo.Mpo(a_cores)
    lr = rrsvd.tnrsvd(a, k, q=q, round_tol=tol, oversample=os_, seed=seed)
    out = {"k": np.array(k), "q": np.array(q),
           "tol": np.array(np.nan if tol is None else tol),
           "oversample": np.array(os_), "seed": np.array(seed),
           "s": lr.s, "u_ranks": np.array(lr.u.ranks),
           "v_ranks": np.array(lr.v.ranks), "K": np.array(lr.k_oversampled)}
    pack_cores("a", a.cores, out)
    pack_cores("u", lr.u.cores, out)
    pack_cores("v", lr.v.cores, out)
    np.savez_compressed(os.path.join(HERE, f"svd_{name}.npz"), **out)


def main():
    # -- conversion -----------------------------------------------------
    coo = rsparse.SparseMatrixCoo(2, 6, [1, 2], [1, 4], [2.0, -5.0])
    conv_case("worked_2x6", coo,
              mposvd.plan_partition(2, 6, ((1, 1, 2), (1, 3, 2))))
    rng = np.random.default_rng(7)
    f = [rng.standard_normal((2, 2)) for _ in range(3)]
    conv_case("kron8", rsparse.SparseMatrixCoo.from_dense(
        np.kron(f[2], np.kron(f[1], f[0]))),
        mposvd.plan_partition(8, 8, ([2] * 3, [2] * 3)))
    coo = rsparse.random_sparse_coo(6, 6, 0.3, seed=4)
    conv_case("pad6in8", coo, mposvd.plan_partition(8, 8, "descending"))
    coo = rsparse.random_sparse_coo(35, 12, 0.2, seed=420)
    conv_case("rect35x12", coo, mposvd.plan_partition(35, 12, "descending"))
    coo = rsparse.random_sparse_coo(64, 64, 0.05, seed=4096)
    conv_case("blk4x4_64", coo, mposvd.plan_partition(64, 64, "4x4"))
    # explicit zeros must be dropped
    coo = rsparse.SparseMatrixCoo(4, 4, [1, 2, 3, 4], [1, 2, 3, 1],
                                  [1.0, 0.0, 3.0, -2.0])
    conv_case("stored_zero", coo, mposvd.plan_partition(4, 4, ([2, 2], [2, 2])))
    coo = band_scatter(1 << 12, 20000, seed=4)
    conv_case("band_scatter_4096", coo,
              mposvd.plan_partition(1 << 12, 1 << 12, ([2] * 12, [2] * 12)))
    coo = band_scatter(1 << 10, 3000, seed=5)
    conv_case("band_scatter_1024_blk8", coo,
              mposvd.plan_partition(1 << 10, 1 << 10, ([8, 4, 4, 2, 2, 2], [4, 8, 2, 2, 2, 4])))

    # -- TNrSVD ---------------------------------------------------------
    # config 1 exactly (BASELINE.json configs[0]; SURVEY.md 8(d) seeds A:1, O:2)
    svd_case("c1", rmpo.random_mpo([2] * 10, [2] * 10, [3] * 9, seed=1).cores,
             10, 0, 1e-9, 2.0, 2)
    svd_case("small_q1", rmpo.random_mpo([4, 2, 2, 2], [4, 2, 2, 2], [3, 3, 3],
                                         seed=27).cores, 5, 1, 1e-12, 2.0, 28)
    svd_case("small_q2", rmpo.random_mpo([2] * 8, [2] * 8, [3] * 7,
                                         seed=11).cores, 4, 2, 1e-9, 2.0, 12)
    svd_case("noround_q1", rmpo.random_mpo([4, 2, 2, 2], [4, 2, 2, 2], [2, 3, 2],
                                           seed=13).cores, 3, 1, None, 2.0, 14)
    # config-5 instance shape at reduced d (q=1 compounds ranks 16 -> 256 -> 4096)
    c5 = rmpo.random_mpo([2] * 12, [2] * 12, [4] * 11, seed=50).cores
    svd_case("c5mini_q1", c5, 16, 1, 1e-9, 1.5, 51)
    # config-2 recipe at reduced d: N(0,1)/sqrt(8) cores, rank 8
    c2 = [c / math.sqrt(8.0) for c in
          rmpo.random_mpo([2] * 12, [2] * 12, [8] * 11, seed=1).cores]
    svd_case("c2mini_q1", c2, 20, 1, 1e-9, 1.5, 2)
    # config-3 recipe at reduced size: n=4, rank 16, decaying middle bond
    c3 = [c / 8.0 for c in rmpo.random_mpo([4] * 6, [4] * 6, [16] * 5, seed=3).cores]
    c3[2] = c3[2] * (0.5 ** np.arange(16))[None, None, None, :]
    svd_case("c3mini_q0", c3, 16, 0, 1e-9, 1.5, 4)

    # prescribed spectrum 0.5^k built in MPO form by the reference's own
    # bench generator (bench.py:107-139): truncation is active in every sweep
    from mposvd import bench as rbench
    for n in (12, 14):
        a, _, _ = rbench.gen_prescribed_spectrum_mpo(
            n, 0.5 ** np.arange(20), seed=np.random.default_rng([0, n, 0]))
        svd_case(f"spectrum_n{n}", a.cores, 20, 1, 1e-9, 1.5, 5)
    # exact low-rank matrix (rsvd test :272-280 recipe): zero singular values
    u = rmpo.random_unit_rank_mpo([8, 2, 2], 3, seed=34)
    vt = rmpo.random_unit_rank_mpo([8, 2, 2], 3, seed=35)
    a = rrsvd.mpo_matmul(u, rmpo.mpo_transpose(vt))
    svd_case("lowrank3", a.cores, 3, 2, 1e-13, 2.0, 36)

    # -- sub-stages -----------------------------------------------------
    y = rmpo.random_unit_rank_mpo([16, 2, 2], 8, seed=10)
    q, r = rrsvd.mpo_qr(y)
    out = {"r": r}
    pack_cores("y", y.cores, out)
    pack_cores("q", q.cores, out)
    np.savez_compressed(os.path.join(HERE, "stage_qr_exact.npz"), **out)
    y = rmpo.random_mpo([8, 2, 2, 2], [8, 1, 1, 1], [6, 6, 4], seed=12)
    q, r = rrsvd.mpo_qr(y, round_tol=1e-10)
    out = {"r": r, "q_ranks": np.array(q.ranks)}
    pack_cores("y", y.cores, out)
    pack_cores("q", q.cores, out)
    np.savez_compressed(os.path.join(HERE, "stage_qr_round.npz"), **out)
    b = rmpo.random_mpo([3, 1, 1], [4, 2, 2], [3, 2], seed=16)
    w, s, v = rrsvd.mpo_svd(b)
    out = {"w": w, "s": s}
    pack_cores("b", b.cores, out)
    pack_cores("v", v.cores, out)
    np.savez_compressed(os.path.join(HERE, "stage_svd.npz"), **out)
    a = rmpo.random_mpo([2, 3, 2], [3, 2, 2], [3, 2], seed=3)
    bb = rmpo.random_mpo([3, 2, 2], [2, 2, 3], [2, 3], seed=4)
    p = rrsvd.mpo_matmul(a, bb)
    out = {}
    pack_cores("a", a.cores, out)
    pack_cores("b", bb.cores, out)
    pack_cores("p", p.cores, out)
    np.savez_compressed(os.path.join(HERE, "stage_matmul.npz"), **out)
    m = rmpo.random_mpo([2] * 10, [2] * 10, [3] * 9, seed=19)
    mm = rrsvd.merge_leading_cores(m, 5)
    out = {}
    pack_cores("m", m.cores, out)
    pack_cores("mm", mm.cores, out)
    np.savez_compressed(os.path.join(HERE, "stage_merge.npz"), **out)
    print("golden fixtures written to", HERE)


def big():
    """BASELINE-size reference runs (minutes each): only the small outputs
    (singular values, ranks, flop-relevant shapes) are kept."""
    import time
    cases = {}
    # config 2: A seed 1, O seed 2, cores / sqrt(8)
    a = rmpo.random_mpo([2] * 20, [2] * 20, [8] * 19, seed=1)
    a = rmpo.Mpo([c / math.sqrt(8.0) for c in a.cores])
    cases["c2"] = (a, dict(k_target=20, q=1, round_tol=1e-9, oversample=1.5, seed=2))
    # config-5 TNrSVD instance, oracle-feasible q=0 variant (instance seed 50)
    a = rmpo.random_mpo([2] * 20, [2] * 20, [16] * 19, seed=50)
    cases["c5inst_q0"] = (a, dict(k_target=16, q=0, round_tol=1e-9, oversample=1.5, seed=51))
    # config-5 recipe (rank 16, q=1) at d=16: the largest d at which the
    # reference's materialised B = Q^T A cores (12288 x 2 x 16384) still fit
    # in host memory; exercises the device's fused, rank-bounded sweeps where
    # the product ranks exceed the bond extents 16-fold
    a = rmpo.random_mpo([2] * 16, [2] * 16, [16] * 15, seed=50)
    cases["c5d16_q1"] = (a, dict(k_target=16, q=1, round_tol=1e-9, oversample=1.5, seed=51))
    # config 3 at the oracle-feasible q=0 (q=2 dies with a 1.5 TiB core):
    # cores N(0,1)/8, middle bond (core 5's right rank index k) scaled by 0.5^k
    a = rmpo.random_mpo([4] * 12, [4] * 12, [64] * 11, seed=3)
    cores = [c / 8.0 for c in a.cores]
    cores[5] = cores[5] * (0.5 ** np.arange(64))[None, None, None, :]
    cases["c3q0"] = (rmpo.Mpo(cores), dict(k_target=32, q=0, round_tol=1e-9, oversample=1.5, seed=4))
    only = sys.argv[2:] or list(cases)
    for name in only:
        a, kw = cases[name]
        t0 = time.perf_counter()
        lr = rrsvd.tnrsvd(a, **kw)
        secs = time.perf_counter() - t0
        np.savez_compressed(os.path.join(HERE, f"big_{name}.npz"), s=lr.s,
                            u_ranks=np.array(lr.u.ranks), v_ranks=np.array(lr.v.ranks),
                            K=np.array(lr.k_oversampled), seconds=np.array(secs))
        print(name, secs, lr.u.ranks, lr.v.ranks)
    # config 4 conversion (2^16 square band + 1e6 scatter, seed 4)
    coo = band_scatter(1 << 16, 1_000_000, seed=4)
    plan = mposvd.plan_partition(1 << 16, 1 << 16, ([2] * 16, [2] * 16))
    m = rsparse.matrix_to_mpo(coo, plan, densify_limit=0)
    c0 = m.cores[0]
    np.savez_compressed(os.path.join(HERE, "big_c4conv.npz"),
                        nnz=np.array(coo.val.size), rank=np.array(m.ranks[1]),
                        ti_sum=np.array(int(c0.right.sum())),
                        ti_hash=np.array(int((c0.right * np.arange(c0.right.size, dtype=np.int64)).sum())),
                        lvl_hash=np.array([int((c.row * 3 + c.col).sum()) for c in m.cores[1:]]))
    print("c4", coo.val.size, m.ranks[1])


def io_fixtures():
    """Reference-written .mpo and Matrix Market files (byte-compatibility
    fixtures for paper_1707_07803_b200.io)."""
    m = rmpo.random_mpo([2, 3, 2], [2, 2, 3], [3, 4], seed=18)
    rmpo.save_mpo(m, os.path.join(HERE, "io_ref.mpo"))
    rng = np.random.default_rng(7)
    dense = np.where(rng.random((9, 13)) < 0.2, rng.standard_normal((9, 13)), 0.0)
    coo = rsparse.SparseMatrixCoo.from_dense(dense)
    rsparse.write_matrix_market(os.path.join(HERE, "io_ref.mtx"), coo)
    np.savez_compressed(os.path.join(HERE, "io_ref_mtx.npz"), rows=np.array(coo.rows),
                        cols=np.array(coo.cols), row=coo.row, col=coo.col, val=coo.val)
    print("io fixtures written")


if __name__ == "__main__":
    if len(sys.argv) > 1 and sys.argv[1] == "--big":
        big()
    elif len(sys.argv) > 1 and sys.argv[1] == "--io":
        io_fixtures()
    else:
        main()

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
    sel = sys.argv[2:]
    only = [x for x in sel if x in cases] if sel else list(cases)
    sys.path.insert(0, os.path.dirname(HERE))
    import mpo_checks as mc   # tests/mpo_checks.py: the same formulas the GPU tests use
    for name in only:
        a, kw = cases[name]
        t0 = time.perf_counter()
        lr = rrsvd.tnrsvd(a, **kw)
        secs = time.perf_counter() - t0
        # MPO-form accuracy of the reference's own result (BASELINE config 2:
        # "residual ||A V - U S|| contracted in TT format"), on the merged
        # operator the factors live on; the 4-layer V^T A^T A V environment
        # is 4096^2 x 64^2 doubles at config 3, so only U^T A A^T U there
        am = rrsvd.merge_leading_cores(a, a.num_cores - lr.u.num_cores + 1)
        t1 = time.perf_counter()
        chk = mc.summary(lr.u.cores, lr.s, lr.v.cores, am.cores, av=(name != "c3q0"))
        extra = {f"chk_{k}": np.asarray(v) for k, v in chk.items()}
        np.savez_compressed(os.path.join(HERE, f"big_{name}.npz"), s=lr.s,
                            u_ranks=np.array(lr.u.ranks), v_ranks=np.array(lr.v.ranks),
                            K=np.array(lr.k_oversampled), seconds=np.array(secs), **extra)
        print(name, secs, time.perf_counter() - t1, lr.u.ranks, lr.v.ranks,
              chk.get("res_av"), chk.get("res_atu"), flush=True)
        del lr, am, chk
    if "conv5" not in sys.argv[2:] and sys.argv[2:]:
        return
    conv5()
    # config 4 conversion (2^16 square band + 1e6 scatter, seed 4)
    conv4()


def _sha(x):
    import hashlib
    return hashlib.sha256(np.ascontiguousarray(x).tobytes()).hexdigest()


def conv5():
    """Config 5's conversion at full size (2^22 square, power-law rows,
    seed 55; paper_1707_07803_b200.workloads.powerlaw_coo): the reference's
    matrix_to_mpo output is kept as sha256 digests of its index arrays (the
    arrays are ~1 GB), plus the COO constructor and conversion times."""
    import time
    sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
    from paper_1707_07803_b200.workloads import powerlaw_coo
    n = 1 << 22
    r, c, v = powerlaw_coo(n, seed=55)
    t0 = time.perf_counter()
    coo = rsparse.SparseMatrixCoo(n, n, r, c, v)
    t_ctor = time.perf_counter() - t0
    plan = mposvd.plan_partition(n, n, ([2] * 22, [2] * 22))
    t0 = time.perf_counter()
    m = rsparse.matrix_to_mpo(coo, plan, densify_limit=0)
    t_conv = time.perf_counter() - t0
    c0 = m.cores[0]
    lv = [1, 11, 21]
    out = dict(nnz=np.array(c0.values.size), rank=np.array(m.ranks[1]),
               ti_sha=np.array(_sha(c0.right)), i1_sha=np.array(_sha(c0.row)),
               j1_sha=np.array(_sha(c0.col)), values_sha=np.array(_sha(c0.values)),
               levels=np.array(lv),
               lvl_row_sha=np.array([_sha(m.cores[k].row) for k in lv]),
               lvl_col_sha=np.array([_sha(m.cores[k].col) for k in lv]),
               seconds_ctor=np.array(t_ctor), seconds_convert=np.array(t_conv))
    np.savez_compressed(os.path.join(HERE, "big_c5conv.npz"), **out)
    print("c5conv", out["nnz"], out["rank"], t_ctor, t_conv, flush=True)


def conv4():
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


def round_fixtures():
    """mpo_add (mpo.py:264-294), mpo_round (mpo.py:323-354) and the capped
    matrix_to_mpo (sparse.py:260-275) run by the reference: output ranks
    and the dense matrices (desk scale)."""
    out = {}
    # a redundant sum: exact rank 6 (5 + 1 shared directions) per bond,
    # represented at rank 10 + noise at 1e-12 (kept at 1e-14, cut at 1e-10)
    a = rmpo.random_mpo([2] * 7, [2] * 7, [5] * 6, seed=61)
    b = rmpo.random_mpo([2] * 7, [2] * 7, [1] * 6, seed=62)
    ab = rmpo.mpo_add(a, b)
    noise = rmpo.random_mpo([2] * 7, [2] * 7, [2] * 6, seed=63)
    noise = rmpo.Mpo([noise.cores[0] * 1e-12] + noise.cores[1:])
    m = rmpo.mpo_add(rmpo.mpo_add(ab, a), noise)
    pack_cores("add_a", a.cores, out)
    pack_cores("add_b", b.cores, out)
    pack_cores("add_ab", ab.cores, out)
    pack_cores("round_in", m.cores, out)
    for tag, tol in (("t10", 1e-10), ("t14", 1e-14), ("t6", 1e-6)):
        r = rmpo.mpo_round(m, tol)
        out[f"round_{tag}_ranks"] = np.array(r.ranks)
        out[f"round_{tag}_dense"] = rmpo.contract_to_matrix(r)
    out["round_in_dense"] = rmpo.contract_to_matrix(m)
    # capped conversions
    cases = [("rand64", rsparse.random_sparse_coo(64, 64, 0.2, seed=64), ([2] * 6, [2] * 6), 8, None),
             ("band256", band_scatter(256, 600, seed=65), ([2] * 8, [2] * 8), 32, None),
             ("rand64_t8", rsparse.random_sparse_coo(64, 64, 0.2, seed=66), ([2] * 6, [2] * 6), 8, 1e-8)]
    for tag, coo, fac, cap, tol in cases:
        plan = mposvd.plan_partition(coo.rows, coo.cols, fac)
        mm = rsparse.matrix_to_mpo(coo, plan, rank_cap=cap, round_tol=tol)
        out[f"cap_{tag}_rows"], out[f"cap_{tag}_cols"] = np.array(coo.rows), np.array(coo.cols)
        out[f"cap_{tag}_row"], out[f"cap_{tag}_col"], out[f"cap_{tag}_val"] = coo.row, coo.col, coo.val
        out[f"cap_{tag}_fac"] = np.array(fac)
        out[f"cap_{tag}_cap"] = np.array(cap)
        out[f"cap_{tag}_tol"] = np.array(np.nan if tol is None else tol)
        out[f"cap_{tag}_ranks"] = np.array(mm.ranks)
        out[f"cap_{tag}_dense"] = rmpo.contract_to_matrix(mm)
        print(tag, mm.ranks)
    np.savez_compressed(os.path.join(HERE, "round_add_cap.npz"), **out)
    print("round fixtures written", {k: v for k, v in out.items() if k.endswith("_ranks")})


def tail_fixtures():
    """mpo_round (mpo.py:323-354) by the reference on MPOs whose bond
    spectrum has a dense tail straddling delta at ranks >= 256 -- the
    regime of the device's rank certificate / tail truncation
    (csrc/rankcert.cu): output ranks and dense matrices."""
    out = {}
    rng = np.random.default_rng(71)

    def orth(m, n):
        q, _ = np.linalg.qr(rng.standard_normal((m, n)))
        return q

    # two cores, bond 256 = min(left, right extent): A = U diag(s) V^T,
    # s geometric from 1 to 1e-12 (about 43 values below delta at 1e-10)
    s = 10.0 ** (-12.0 * np.arange(256) / 255)
    u, v = orth(256, 256), orth(256, 256)
    c0 = (u * s).reshape(1, 16, 16, 256, order="F")
    c1 = v.T.reshape(256, 16, 16, 1, order="F")
    # three cores: the same left factor at bond 0, a graded second bond
    d0 = (u * s).reshape(1, 16, 16, 256, order="F")
    d1 = rng.standard_normal((256, 2, 2, 64)) * (10.0 ** (-np.arange(64) / 8.0))
    d2 = rng.standard_normal((64, 8, 8, 1))
    for tag, cores in (("two", [c0, c1]), ("three", [d0, d1, d2])):
        m = rmpo.Mpo(cores)
        pack_cores(f"tail_{tag}_in", m.cores, out)
        for ttag, tol in (("t10", 1e-10), ("t8", 1e-8)):
            r = rmpo.mpo_round(m, tol)
            out[f"tail_{tag}_{ttag}_ranks"] = np.array(r.ranks)
            out[f"tail_{tag}_{ttag}_dense"] = rmpo.contract_to_matrix(r)
            print(tag, ttag, r.ranks)
        out[f"tail_{tag}_dense"] = rmpo.contract_to_matrix(m)
    np.savez_compressed(os.path.join(HERE, "round_tail.npz"), **out)
    print("tail fixtures written")


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
    elif len(sys.argv) > 1 and sys.argv[1] == "--round":
        round_fixtures()
    elif len(sys.argv) > 1 and sys.argv[1] == "--tail":
        tail_fixtures()
    elif len(sys.argv) > 1 and sys.argv[1] == "--io":
        io_fixtures()
    else:
        main()

"""Pin the CPU oracle (oracle/mposvd_oracle.py) against fixtures produced by
the unmodified reference (tests/golden/make_golden.py)."""

import glob
import os

import numpy as np
import pytest

from conftest import GOLDEN, load_golden, unpack_cores
from oracle import mposvd_oracle as orc

CONV = sorted(os.path.basename(p) for p in glob.glob(os.path.join(GOLDEN, "conv_*.npz")))
SVD = sorted(os.path.basename(p) for p in glob.glob(os.path.join(GOLDEN, "svd_*.npz")))


@pytest.mark.parametrize("name", CONV)
def test_conversion_structure_bit_exact(name):
    z = load_golden(name)
    rf, cf = list(z["row_factors"]), list(z["col_factors"])
    st = orc.conversion_structure(z["row"], z["col"], z["val"], rf, cf)
    assert (1,) + (st.rank,) * (len(rf) - 1) + (1,) == tuple(z["ranks"]) or st.rank == 0
    if "ti" in z:
        assert np.array_equal(st.i1, z["i1"])
        assert np.array_equal(st.j1, z["j1"])
        assert np.array_equal(st.ti, z["ti"])
        assert np.array_equal(st.values, z["values"])
        ur, uc = orc.block_digits(st.uniq, rf, cf)
        for k in range(1, len(rf)):
            assert np.array_equal(ur[k - 1], z[f"lvl{k}_row"])
            assert np.array_equal(uc[k - 1], z[f"lvl{k}_col"])
    if "dense_n" in z:
        want = unpack_cores(z, "dense")
        got = orc.conversion_dense_cores(st, rf, cf)
        for g, w in zip(got, want):
            assert np.array_equal(g, w)


def _tol(z):
    t = float(z["tol"])
    return None if np.isnan(t) else t


@pytest.mark.parametrize("name", SVD)
def test_tnrsvd_oracle_matches_reference(name):
    z = load_golden(name)
    a = unpack_cores(z, "a")
    res = orc.tnrsvd(a, int(z["k"]), q=int(z["q"]), round_tol=_tol(z),
                     oversample=float(z["oversample"]), seed=int(z["seed"]))
    assert orc.ranks_of(res.u) == tuple(z["u_ranks"])
    assert orc.ranks_of(res.v) == tuple(z["v_ranks"])
    assert res.k_oversampled == int(z["K"])
    np.testing.assert_allclose(res.s, z["s"], rtol=1e-12, atol=0)
    # same LAPACK calls in the same order: the factors agree core by core
    for got, want in ((res.u, unpack_cores(z, "u")), (res.v, unpack_cores(z, "v"))):
        for g, w in zip(got, want):
            np.testing.assert_allclose(g, w, rtol=0, atol=1e-10 * max(1.0, np.abs(w).max()))


def test_stage_matmul_and_merge():
    z = load_golden("stage_matmul.npz")
    got = orc.mpo_matmul(unpack_cores(z, "a"), unpack_cores(z, "b"))
    for g, w in zip(got, unpack_cores(z, "p")):
        assert np.array_equal(g, w)
    z = load_golden("stage_merge.npz")
    got = orc.merge_leading(unpack_cores(z, "m"), 5)
    for g, w in zip(got, unpack_cores(z, "mm")):
        np.testing.assert_allclose(g, w, rtol=0, atol=1e-12)


def test_stage_qr_svd():
    z = load_golden("stage_qr_exact.npz")
    q, r = orc.mpo_qr(unpack_cores(z, "y"))
    np.testing.assert_allclose(r, z["r"], atol=1e-12)
    z = load_golden("stage_qr_round.npz")
    q, r = orc.mpo_qr(unpack_cores(z, "y"), 1e-10)
    assert orc.ranks_of(q) == tuple(z["q_ranks"])
    np.testing.assert_allclose(np.abs(r), np.abs(z["r"]), atol=1e-10)
    z = load_golden("stage_svd.npz")
    w, s, v = orc.mpo_svd(unpack_cores(z, "b"))
    np.testing.assert_allclose(s, z["s"], rtol=1e-13)


def test_oracle_ledger_counts_c1():
    z = load_golden("svd_c1.npz")
    led = orc.Ledger()
    orc.tnrsvd(unpack_cores(z, "a"), 10, q=0, round_tol=1e-9, oversample=2.0,
               seed=2, ledger=led)
    # SURVEY.md 6.2 / BASELINE.md 2: c1 = 2.01e6 model flops
    assert 1.8e6 < led.total < 2.2e6


def test_truncation_rank_rules():
    s = np.array([3.0, 2.0, 1.0, 0.5])
    assert orc.truncation_rank(s, 0.5, 1e-3) == 3
    assert orc.truncation_rank(s, 10.0, 1e-3) == 1
    assert orc.truncation_rank(np.array([1.0, 0.0, 0.0]), 0.0, 0.0) == 1
    assert orc.truncation_rank(np.zeros(3), 0.0, 0.0) == 1

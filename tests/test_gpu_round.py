"""Parity of the device mpo_add / mpo_round and the capped sparse->MPO
conversion against the reference's own runs
(tests/golden/round_add_cap.npz, make_golden.py --round):

* mpo_add (mpo.py:264-294): cores identical (block-diagonal stacking);
* mpo_round (mpo.py:323-354) at rel_tol 1e-6, 1e-10 and 1e-14 (the capped
  conversion's default; below the Jacobi noise floor of 64 eps, which must
  then shrink with delta): equal ranks, matrix within 1e-12 relative;
* capped matrix_to_mpo (sparse.py:260-275), chunks built on the device
  from the conversion handle: equal ranks, matrix within 1e-12 relative."""

import numpy as np
import pytest

from conftest import load_golden, unpack_cores
from oracle import mposvd_oracle as orc

pytestmark = pytest.mark.gpu


def _api():
    import paper_1707_07803_b200 as m
    return m


def test_mpo_add_matches_reference():
    m = _api()
    z = load_golden("round_add_cap.npz")
    got = m.mpo_add(m.Mpo(unpack_cores(z, "add_a")), m.Mpo(unpack_cores(z, "add_b")))
    for g, w in zip(got.cores, unpack_cores(z, "add_ab")):
        assert np.array_equal(np.asarray(g), w)


@pytest.mark.parametrize("tag,tol", [("t6", 1e-6), ("t10", 1e-10), ("t14", 1e-14)])
def test_mpo_round_matches_reference(tag, tol):
    m = _api()
    z = load_golden("round_add_cap.npz")
    got = m.mpo_round(m.Mpo(unpack_cores(z, "round_in")), tol)
    assert got.ranks == tuple(z[f"round_{tag}_ranks"])
    want = z[f"round_{tag}_dense"]
    dense = orc.contract(got.cores)
    assert np.linalg.norm(dense - want) <= 1e-12 * np.linalg.norm(want)
    # and the rounding budget of mpo.py:328-330 against the unrounded input
    full = z["round_in_dense"]
    assert np.linalg.norm(dense - full) <= max(tol, 1e-13) * np.linalg.norm(full)


@pytest.mark.parametrize("tag", ["rand64", "band256", "rand64_t8"])
def test_capped_conversion_matches_reference(tag):
    m = _api()
    z = load_golden("round_add_cap.npz")
    p = f"cap_{tag}_"
    coo = m.SparseMatrixCoo(int(z[p + "rows"]), int(z[p + "cols"]), z[p + "row"], z[p + "col"],
                            z[p + "val"])
    fac = z[p + "fac"]
    plan = m.plan_partition(coo.rows, coo.cols, (tuple(fac[0]), tuple(fac[1])))
    tol = float(z[p + "tol"])
    got = m.matrix_to_mpo(coo, plan, rank_cap=int(z[p + "cap"]),
                          round_tol=None if np.isnan(tol) else tol)
    assert got.ranks == tuple(z[p + "ranks"])
    want = z[p + "dense"]
    assert np.linalg.norm(orc.contract(got.cores) - want) <= 1e-12 * np.linalg.norm(want)


@pytest.mark.parametrize("tag,ttag,tol", [("two", "t10", 1e-10), ("two", "t8", 1e-8),
                                          ("three", "t10", 1e-10), ("three", "t8", 1e-8)])
def test_mpo_round_dense_tail_matches_reference(tag, ttag, tol):
    """Bond spectra with a dense tail straddling delta at rank 256 (the
    rank certificate / tail truncation regime, rankcert.cu) rounded by the
    reference's mpo_round (tests/golden/round_tail.npz): equal ranks, matrix
    within 1e-12 relative; the two-core case at 1e-10 must take the tail
    truncation (43 values below delta inside the 64-vector block)."""
    m = _api()
    from paper_1707_07803_b200 import _lib
    z = load_golden("round_tail.npz")
    before = _lib.round_paths()
    got = m.mpo_round(m.Mpo(unpack_cores(z, f"tail_{tag}_in")), tol)
    after = _lib.round_paths()
    assert got.ranks == tuple(z[f"tail_{tag}_{ttag}_ranks"])
    want = z[f"tail_{tag}_{ttag}_dense"]
    assert np.linalg.norm(orc.contract(got.cores) - want) <= 1e-12 * np.linalg.norm(want)
    if (tag, ttag) == ("two", "t10"):
        assert after["tail"] > before["tail"], (before, after)

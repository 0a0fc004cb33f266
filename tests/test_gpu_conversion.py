"""Parity of the device sparse->MPO conversion (convert.cu via the C-ABI)
against the reference's golden structures: bit-exact i1, j1, ti, values,
sorted block keys and per-level digits; dense cores bit-exact."""

import glob
import os

import numpy as np
import pytest

from conftest import GOLDEN, load_golden, unpack_cores
from oracle import mposvd_oracle as orc

pytestmark = pytest.mark.gpu

CONV = sorted(os.path.basename(p) for p in glob.glob(os.path.join(GOLDEN, "conv_*.npz")))


def _api():
    import paper_1707_07803_b200 as m
    return m


@pytest.mark.parametrize("name", CONV)
def test_conversion_matches_reference_structure(name):
    m = _api()
    z = load_golden(name)
    plan = m.PartitionPlan(tuple(z["row_factors"]), tuple(z["col_factors"]))
    coo = m.SparseMatrixCoo(int(z["rows"]), int(z["cols"]), z["row"], z["col"], z["val"])
    got = m.matrix_to_mpo(coo, plan, densify_limit=0)
    assert got.ranks == tuple(z["ranks"])
    if "ti" in z:
        c0 = got.cores[0]
        assert np.array_equal(c0.row, z["i1"])
        assert np.array_equal(c0.col, z["j1"])
        assert np.array_equal(c0.right, z["ti"])
        assert np.array_equal(c0.values, z["values"])
        for k in range(1, plan.d):
            assert np.array_equal(got.cores[k].row, z[f"lvl{k}_row"])
            assert np.array_equal(got.cores[k].col, z[f"lvl{k}_col"])
    if "dense_n" in z:
        dense = m.matrix_to_mpo(coo, plan)
        for g, w in zip(dense.cores, unpack_cores(z, "dense")):
            assert np.array_equal(np.asarray(g), w)


def test_conversion_c4_full_size_structure():
    """Config 4 at its full 2^16 size, against the reference run
    (tests/golden/big_c4conv.npz) and the oracle restatement."""
    m = _api()
    from paper_1707_07803_b200.workloads import band_scatter_coo, square_plan
    r, c, v = band_scatter_coo(1 << 16, 1_000_000, 4)
    z = load_golden("big_c4conv.npz")
    assert r.size == int(z["nnz"])
    plan = square_plan(16)
    res = m.convert_structure(r, c, v, plan)
    assert res.rank == int(z["rank"])
    i1, j1, ti, vals, uniq = res.arrays()
    assert int(ti.sum()) == int(z["ti_sum"])
    assert int((ti * np.arange(ti.size, dtype=np.int64)).sum()) == int(z["ti_hash"])
    for k in range(1, 16):
        rd, cd = res.level(k)
        assert int((rd * 3 + cd).sum()) == int(z["lvl_hash"][k - 1])
    st = orc.conversion_structure(r, c, v, plan.row_factors, plan.col_factors)
    assert np.array_equal(st.ti, ti) and np.array_equal(st.uniq, uniq)
    assert np.array_equal(st.i1, i1) and np.array_equal(st.j1, j1)
    assert np.array_equal(st.values, vals)


def test_conversion_properties_large_random():
    """Size-independent properties at ~5M nonzeros: keys strictly sorted,
    ti consistent with the keys, rank = distinct blocks."""
    m = _api()
    from paper_1707_07803_b200.workloads import powerlaw_coo, square_plan
    r, c, v = powerlaw_coo(1 << 19, seed=9)
    plan = square_plan(19)
    res = m.convert_structure(r, c, v, plan)
    i1, j1, ti, vals, uniq = res.arrays()
    assert np.all(np.diff(uniq) > 0)
    nrb = 1 << 18
    key = (r - 1) // 2 + nrb * ((c - 1) // 2)
    assert np.array_equal(uniq[ti], key)
    assert np.array_equal(i1, (r - 1) % 2) and np.array_equal(j1, (c - 1) % 2)
    assert res.rank == np.unique(key).size


@pytest.mark.parametrize("order", ["shuffled", "row_sorted", "col_sorted"])
def test_conversion_input_order(order):
    """The sort skips the block-row digit passes when the kept keys already
    arrive sorted by block row (row-sorted COO); any other order takes the
    full-key sort.  Both must match the oracle bit for bit."""
    m = _api()
    from paper_1707_07803_b200.workloads import powerlaw_coo, square_plan
    r, c, v = powerlaw_coo(1 << 17, seed=21)
    rng = np.random.default_rng(5)
    if order == "shuffled":
        p = rng.permutation(r.size)
    elif order == "col_sorted":
        p = np.lexsort((r, c))
    else:
        p = np.arange(r.size)
    r, c, v = r[p], c[p], v[p]
    v[rng.integers(0, v.size, 1000)] = 0.0   # explicit zeros are dropped
    plan = square_plan(17)
    res = m.convert_structure(r, c, v, plan)
    i1, j1, ti, vals, uniq = res.arrays()
    st = orc.conversion_structure(r, c, v, plan.row_factors, plan.col_factors)
    assert np.array_equal(st.uniq, uniq) and np.array_equal(st.ti, ti)
    assert np.array_equal(st.i1, i1) and np.array_equal(st.j1, j1)
    assert np.array_equal(st.values, vals)


def test_conversion_empty_and_zero_values():
    m = _api()
    a = m.SparseMatrixCoo(8, 8, [], [], [])
    got = m.matrix_to_mpo(a, m.plan_partition(8, 8, "descending"))
    assert got.ranks == (1, 1, 1, 1)
    a = m.SparseMatrixCoo(4, 4, [1, 2], [1, 2], [0.0, 0.0])
    got = m.matrix_to_mpo(a, m.plan_partition(4, 4, "descending"))
    assert got.ranks == (1, 1, 1)


def test_conversion_errors():
    m = _api()
    a = m.SparseMatrixCoo(16, 16, [1], [1], [1.0])
    with pytest.raises(ValueError):
        m.matrix_to_mpo(a, m.plan_partition(8, 8, "descending"))
    with pytest.raises(ValueError):
        m.matrix_to_mpo(a, m.plan_partition(16, 16, "descending"), rank_cap=0)


def test_conversion_rank_cap_rounds_on_device():
    m = _api()
    rng = np.random.default_rng(5)
    dense = rng.standard_normal((16, 16)) * (rng.random((16, 16)) < 0.4)
    a = m.SparseMatrixCoo.from_dense(dense)
    plan = m.plan_partition(16, 16, ([2] * 4, [2] * 4))
    uncapped = m.matrix_to_mpo(a, plan)
    capped = m.matrix_to_mpo(a, plan, rank_cap=8, round_tol=1e-14)
    assert uncapped.max_rank > 8
    assert capped.max_rank < uncapped.max_rank
    got = orc.contract(capped.cores)
    assert np.linalg.norm(got - dense) <= 1e-12 * np.linalg.norm(dense)


def test_conversion_deterministic():
    m = _api()
    from paper_1707_07803_b200.workloads import powerlaw_coo, square_plan
    r, c, v = powerlaw_coo(1 << 14, seed=3)
    plan = square_plan(14)
    a1 = m.convert_structure(r, c, v, plan).arrays()
    a2 = m.convert_structure(r, c, v, plan).arrays()
    for x, y in zip(a1, a2):
        assert np.array_equal(x, y)

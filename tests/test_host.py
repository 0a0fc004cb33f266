"""Host-side logic of the drop-in (no device): partition planning, sketch
width / merge count, the sketch RNG stream, Mpo validation, COO
validation.  Mirrors the reference's own test cases."""

import numpy as np
import pytest

from conftest import load_golden, unpack_cores
from oracle import mposvd_oracle as orc
import paper_1707_07803_b200 as m
from paper_1707_07803_b200 import rsvd


def test_prime_factorize_and_plans():
    assert m.prime_factorize(150102) == [2, 3, 3, 31, 269]
    assert m.prime_factorize(1) == []
    p = m.plan_partition(35, 12, "descending")
    assert p.row_factors == (7, 5, 1) and p.col_factors == (3, 2, 2)
    p = m.plan_partition(64, 64, "4x4")
    assert p.block_shape == (4, 4) and p.rows == 64
    p = m.plan_partition(6, 6, "descending", pad=True)
    assert p.rows == 8
    with pytest.raises(ValueError):
        m.plan_partition(8, 8, ([2, 2], [2, 2]))
    with pytest.raises(ValueError):
        m.plan_partition(8, 8, "bogus")
    with pytest.raises(ValueError):
        m.PartitionPlan((2, 2), (2,))


def test_sketch_width_and_merge_count_match_oracle():
    for k, os_ in [(10, 2.0), (20, 1.5), (32, 1.5), (50, 1.2), (16, 1.5)]:
        assert rsvd.sketch_width(k, os_) == orc.sketch_width(k, os_)
    for dims, kk in [([2] * 10, 20), ([2] * 20, 30), ([4] * 12, 48), ([2] * 20, 24)]:
        assert rsvd.merge_count(dims, dims, kk) == orc.merge_count(dims, dims, kk)
    with pytest.raises(ValueError):
        rsvd.merge_count([2, 2], [2, 2], 8)


def test_sketch_stream_bit_identical_to_reference_generator():
    a = m.random_unit_rank_mpo([32, 2, 2, 2], 20, seed=2)
    b = orc.random_unit_rank_mpo([32, 2, 2, 2], 20, seed=2)
    for x, y in zip(a.cores, b):
        assert np.array_equal(x, y)
    z = load_golden("svd_c1.npz")
    for x, y in zip(m.random_mpo([2] * 10, [2] * 10, [3] * 9, seed=1).cores,
                    unpack_cores(z, "a")):
        assert np.array_equal(x, y)


def test_mpo_validation():
    with pytest.raises(ValueError):
        m.Mpo([])
    with pytest.raises(ValueError):
        m.Mpo([np.zeros((2, 2, 2, 1))])
    with pytest.raises(ValueError):
        m.Mpo([np.zeros((1, 2, 2, 2)), np.zeros((3, 2, 2, 1))])
    mp = m.random_mpo([2, 3], [2, 2], [4], seed=0)
    assert mp.ranks == (1, 4, 1) and mp.num_rows == 6 and mp.num_cols == 4


def test_coo_validation():
    with pytest.raises(ValueError):
        m.SparseMatrixCoo(2, 2, [1, 1], [1, 1], [1.0, 2.0])
    with pytest.raises(ValueError):
        m.SparseMatrixCoo(2, 2, [3], [1], [1.0])
    a = m.SparseMatrixCoo(2, 3, [1, 2], [1, 3], [1.5, 0.0])
    assert a.nnz == 1
    assert m.min_rank_lower_bound(726674, 1614, 1614) == 1


def test_workload_generators_match_golden_recipe():
    from paper_1707_07803_b200.workloads import band_scatter_coo
    z = load_golden("conv_band_scatter_4096.npz")
    r, c, v = band_scatter_coo(1 << 12, 20000, 4)
    assert np.array_equal(r, z["row"]) and np.array_equal(c, z["col"])
    assert np.array_equal(v, z["val"])

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


def _sha(x):
    import hashlib
    return hashlib.sha256(np.ascontiguousarray(x).tobytes()).hexdigest()


def test_conversion_c5_full_size_bit_exact():
    """Config 5's conversion at its full size (2^22 square, 32.7M power-law
    nonzeros): every index array bit-identical to the reference's
    matrix_to_mpo run (sha256 digests in tests/golden/big_c5conv.npz,
    sparse.py:207-258): i1, j1, ti, values and the level digits of three
    cores."""
    m = _api()
    from paper_1707_07803_b200.workloads import powerlaw_coo, square_plan
    z = load_golden("big_c5conv.npz")
    r, c, v = powerlaw_coo(1 << 22, seed=55)
    res = m.convert_structure(r, c, v, square_plan(22))
    assert res.rank == int(z["rank"])
    i1, j1, ti, vals, uniq = res.arrays()
    assert ti.size == int(z["nnz"])
    assert _sha(ti) == str(z["ti_sha"])
    assert _sha(i1) == str(z["i1_sha"]) and _sha(j1) == str(z["j1_sha"])
    assert _sha(vals) == str(z["values_sha"])
    for k, lv in enumerate(z["levels"]):
        rd, cd = res.level(int(lv))
        assert _sha(rd) == str(z["lvl_row_sha"][k]) and _sha(cd) == str(z["lvl_col_sha"][k])


@pytest.mark.parametrize("world", [2, 4, 8])
def test_sharded_exchange_on_device(world):
    """The multi-GPU conversion's per-rank kernels (local convert, sample
    splitters, key-range merge, global-id search, remap) on one device, the
    ranks run in lock step with their collectives emulated
    (distributed.convert_sharded_emulated): config 5's recipe at 2^20,
    bit-exact against the oracle's single-pass structure."""
    import torch
    from paper_1707_07803_b200.distributed import (DeviceOps, convert_sharded_emulated,
                                                   shard_range)
    from paper_1707_07803_b200.workloads import powerlaw_coo, square_plan
    r, c, v = powerlaw_coo(1 << 20, seed=55)
    v[::11] = 0.0   # explicit zeros are dropped before keying (sparse.py:234)
    plan = square_plan(20)
    ops = DeviceOps(0)
    shards = []
    for k in range(world):
        lo, hi = shard_range(r.size, world, k)
        shards.append(tuple(torch.from_numpy(x[lo:hi]).cuda() for x in (r, c, v)))
    res = convert_sharded_emulated(shards, plan, ops)
    st = orc.conversion_structure(r, c, v, plan.row_factors, plan.col_factors)
    cat = lambda xs: np.concatenate([x.cpu().numpy() for x in xs])
    assert np.array_equal(cat([x.ti for x in res]), st.ti)
    assert np.array_equal(cat([x.i1 for x in res]), st.i1)
    assert np.array_equal(cat([x.j1 for x in res]), st.j1)
    assert np.array_equal(cat([x.values for x in res]), st.values)
    assert np.array_equal(cat([x.uniq for x in res]), st.uniq)
    assert all(x.rank == st.rank for x in res)
    assert max(x.uniq.numel() for x in res) <= 1.25 * st.rank / world


def test_conversion_skewed_bucket_falls_back():
    """Entries concentrated in one column block overflow the bucketed fast
    path's on-chip capacity (16K entries per bucket): the onesweep path takes
    over, same result as the oracle."""
    m = _api()
    from paper_1707_07803_b200.workloads import square_plan
    rng = np.random.default_rng(8)
    n = 1 << 16
    r = np.sort(rng.choice(n, 60000, replace=False)) + 1
    c = np.full(r.size, 77, dtype=np.int64)
    r = np.concatenate([r, rng.integers(1, n + 1, 20000)])
    c = np.concatenate([c, rng.integers(1, n + 1, 20000)])
    key = np.unique((r - 1) * n + (c - 1))
    r, c = key // n + 1, key % n + 1
    v = rng.standard_normal(r.size)
    plan = square_plan(16)
    i1, j1, ti, vals, uniq = m.convert_structure(r, c, v, plan).arrays()
    st = orc.conversion_structure(r, c, v, plan.row_factors, plan.col_factors)
    assert np.array_equal(st.uniq, uniq) and np.array_equal(st.ti, ti)
    assert np.array_equal(st.i1, i1) and np.array_equal(st.j1, j1)


def test_conversion_fast_and_onesweep_paths_agree():
    """The bucketed fast path (default) and the onesweep path
    (MPO_B200_CONV_FAST=0, a fresh process) give bit-identical structures on
    shuffled input with explicit zeros."""
    import subprocess
    import sys
    code = (
        "import sys, numpy as np; sys.path.insert(0, '.');"
        "import paper_1707_07803_b200 as m;"
        "from paper_1707_07803_b200.workloads import powerlaw_coo, square_plan;"
        "r, c, v = powerlaw_coo(1 << 18, seed=31);"
        "p = np.random.default_rng(2).permutation(r.size); r, c, v = r[p], c[p], v[p].copy();"
        "v[::97] = 0.0;"
        "a = m.convert_structure(r, c, v, square_plan(18)).arrays();"
        "np.savez(sys.argv[1], *a)")
    import os
    import tempfile
    from conftest import ROOT
    outs = []
    for fast in ("1", "0"):
        path = os.path.join(tempfile.mkdtemp(), "o.npz")
        env = dict(os.environ, MPO_B200_CONV_FAST=fast)
        subprocess.run([sys.executable, "-c", code, path], cwd=ROOT, env=env, check=True)
        z = np.load(path)
        outs.append([z[f"arr_{k}"] for k in range(5)])
    for x, y in zip(*outs):
        assert np.array_equal(x, y)


@pytest.mark.parametrize("order", ["shuffled", "row_sorted"])
def test_conversion_dense_block_column(order):
    """A block column with ~3000 entries fits one bucket but exceeds the
    group sort's per-warp fix-up (64 items): shuffled, its group has key
    inversions and the bucket takes the on-chip LSD passes; row-sorted, the
    group arrives in order.  Both bit-exact against the oracle."""
    m = _api()
    from paper_1707_07803_b200.workloads import square_plan
    rng = np.random.default_rng(12)
    n = 1 << 16
    r = np.concatenate([rng.choice(n, 3000, replace=False) + 1, rng.integers(1, n + 1, 40000)])
    c = np.concatenate([np.full(3000, 4097, dtype=np.int64), rng.integers(1, n + 1, 40000)])
    key = np.unique((r - 1) * n + (c - 1))
    r, c = key // n + 1, key % n + 1
    if order == "shuffled":
        p = rng.permutation(r.size)
        r, c = r[p], c[p]
    v = rng.standard_normal(r.size)
    plan = square_plan(16)
    i1, j1, ti, vals, uniq = m.convert_structure(r, c, v, plan).arrays()
    st = orc.conversion_structure(r, c, v, plan.row_factors, plan.col_factors)
    assert np.array_equal(st.uniq, uniq) and np.array_equal(st.ti, ti)
    assert np.array_equal(st.i1, i1) and np.array_equal(st.j1, j1)

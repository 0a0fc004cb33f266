"""Host file formats at the boundary (paper_1707_07803_b200.io) against
reference-written fixtures (tests/golden/make_golden.py --io): the .mpo
container (mpo.py:477-515) byte for byte, Matrix Market ingest/egest
(sparse.py:96-110).  No GPU needed."""

import os

import numpy as np
import pytest

from conftest import GOLDEN
import paper_1707_07803_b200 as m


def test_load_reference_written_mpo():
    back = m.load_mpo(os.path.join(GOLDEN, "io_ref.mpo"))
    want = m.random_mpo([2, 3, 2], [2, 2, 3], [3, 4], seed=18)
    assert back.row_dims == want.row_dims and back.col_dims == want.col_dims
    assert back.ranks == want.ranks
    for c1, c2 in zip(back.cores, want.cores):
        assert np.array_equal(c1, c2)


def test_save_is_byte_identical_to_reference(tmp_path):
    path = tmp_path / "m.mpo"
    m.save_mpo(m.random_mpo([2, 3, 2], [2, 2, 3], [3, 4], seed=18), path)
    assert path.read_bytes() == open(os.path.join(GOLDEN, "io_ref.mpo"), "rb").read()


def test_file_format_layout(tmp_path):
    path = tmp_path / "tiny.mpo"
    m.save_mpo(m.Mpo([np.arange(4.0).reshape(1, 2, 2, 1, order="F")]), path)
    blob = path.read_bytes()
    assert blob[:4] == b"MPO1"
    hlen = int.from_bytes(blob[4:8], "little")
    assert blob[8:8 + hlen].decode() == ('{"format":1,"num_cores":1,"row_dims":[2],'
                                         '"col_dims":[2],"ranks":[1,1]}')
    assert np.array_equal(np.frombuffer(blob[8 + hlen:], dtype="<f8"), [0.0, 1.0, 2.0, 3.0])


@pytest.mark.gpu
def test_sparse_cores_are_expanded(tmp_path):
    """matrix_to_mpo (device conversion) -> sparse cores -> .mpo -> back."""
    coo = m.SparseMatrixCoo(4, 4, [1, 2, 4], [1, 3, 4], [1.0, 2.0, 3.0])
    plan = m.plan_partition(4, 4, "descending")
    mp = m.matrix_to_mpo(coo, plan, densify_limit=0)
    assert mp.is_sparse
    path = tmp_path / "s.mpo"
    m.save_mpo(mp, path)
    back = m.load_mpo(path)
    for c1, c2 in zip(back.cores, mp.densify().cores):
        assert np.array_equal(c1, np.asarray(c2))


@pytest.mark.parametrize("blob", [b"NOPE" + b"\x00" * 16,
                                  b"MPO1" + (5).to_bytes(4, "little") + b"{bad}",
                                  b"MPO1" + (12).to_bytes(4, "little") + b'{"format":2}'])
def test_load_rejects_garbage(tmp_path, blob):
    path = tmp_path / "bad.mpo"
    path.write_bytes(blob)
    with pytest.raises(ValueError):
        m.load_mpo(path)


@pytest.mark.gpu
def test_save_device_mpo(tmp_path):
    """A DeviceMpo (TNrSVD output left in HBM) is written core by core."""
    a = m.random_mpo([2] * 6, [2] * 6, [3] * 5, seed=4)
    da = m.DeviceMpo.from_host(a)
    path = tmp_path / "d.mpo"
    m.save_mpo(da, path)
    back = m.load_mpo(path)
    for c1, c2 in zip(back.cores, a.cores):
        assert np.array_equal(c1, c2)


def test_load_rejects_truncated(tmp_path):
    path = tmp_path / "t.mpo"
    m.save_mpo(m.random_mpo([2, 2], [2, 2], [3], seed=1), path)
    path.write_bytes(path.read_bytes()[:-8])
    with pytest.raises(ValueError):
        m.load_mpo(path)


def test_read_reference_written_mtx():
    z = np.load(os.path.join(GOLDEN, "io_ref_mtx.npz"))
    a = m.read_matrix_market(os.path.join(GOLDEN, "io_ref.mtx"))
    assert (a.rows, a.cols) == (int(z["rows"]), int(z["cols"]))
    want = np.zeros((a.rows, a.cols))
    want[z["row"] - 1, z["col"] - 1] = z["val"]
    assert np.allclose(a.to_dense(), want, atol=1e-14)


def test_mtx_roundtrip_and_header(tmp_path):
    rng = np.random.default_rng(3)
    dense = np.where(rng.random((9, 13)) < 0.2, rng.standard_normal((9, 13)), 0.0)
    a = m.SparseMatrixCoo.from_dense(dense)
    path = tmp_path / "a.mtx"
    m.write_matrix_market(path, a)
    assert path.read_text().splitlines()[0].startswith(
        "%%MatrixMarket matrix coordinate real general")
    b = m.read_matrix_market(path)
    assert (b.rows, b.cols) == (9, 13)
    assert np.allclose(b.to_dense(), dense, atol=1e-14)


def test_mtx_symmetric_expansion_and_complex(tmp_path):
    path = tmp_path / "s.mtx"
    path.write_text("%%MatrixMarket matrix coordinate real symmetric\n3 3 2\n1 1 2.0\n3 1 5.0\n")
    d = m.read_matrix_market(path).to_dense()
    assert d[0, 0] == 2.0 and d[2, 0] == 5.0 and d[0, 2] == 5.0
    path.write_text("%%MatrixMarket matrix coordinate complex general\n2 2 1\n1 1 2.0 1.0\n")
    with pytest.raises(ValueError):
        m.read_matrix_market(path)

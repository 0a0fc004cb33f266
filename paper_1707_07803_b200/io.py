"""Host file formats at the drop-in boundary.

* ``save_mpo`` / ``load_mpo``: the reference's ``.mpo`` container
  (mpo.py:477-515): 4-byte magic ``MPO1``, little-endian uint32 header
  length, a compact JSON header (format, num_cores, row_dims, col_dims,
  ranks -- in that key order), then every core as little-endian FP64 in
  F order (R, I, J, S).  Files are byte-identical to the reference's, so
  either package reads the other's.  Device-resident MPOs are downloaded
  core by core; sparse cores are expanded as the reference does (the format
  has no sparse encoding).
* ``read_matrix_market`` / ``write_matrix_market``: Matrix Market coordinate
  files via scipy.io (sparse.py:96-110), symmetric storage expanded,
  complex rejected with ``ValueError``.
"""

from __future__ import annotations

import json
import struct
from math import prod

import numpy as np

from .mpo import DeviceMpo, Mpo
from .sparse import SparseMatrixCoo

__all__ = ["save_mpo", "load_mpo", "read_matrix_market", "write_matrix_market"]

_MAGIC = b"MPO1"


def save_mpo(m, path) -> None:
    """Write an MPO (host ``Mpo`` or ``DeviceMpo``) in the ``.mpo`` format."""
    if isinstance(m, DeviceMpo):
        m = m.to_host()
    m = m.densify()
    header = {"format": 1, "num_cores": m.num_cores, "row_dims": list(m.row_dims),
              "col_dims": list(m.col_dims), "ranks": list(m.ranks)}
    blob = json.dumps(header, separators=(",", ":")).encode("utf-8")
    with open(path, "wb") as f:
        f.write(_MAGIC)
        f.write(struct.pack("<I", len(blob)))
        f.write(blob)
        for core in m.cores:
            f.write(np.asarray(core, dtype="<f8").reshape(-1, order="F").tobytes())


def load_mpo(path) -> Mpo:
    """Read a ``.mpo`` file (``ValueError`` on a bad magic, an unknown format
    or truncated core data)."""
    with open(path, "rb") as f:
        if f.read(4) != _MAGIC:
            raise ValueError(f"{path}: not an MPO file")
        raw = f.read(4)
        if len(raw) != 4:
            raise ValueError(f"{path}: truncated header")
        (hlen,) = struct.unpack("<I", raw)
        try:
            header = json.loads(f.read(hlen).decode("utf-8"))
        except (UnicodeDecodeError, json.JSONDecodeError) as e:
            raise ValueError(f"{path}: corrupt header ({e})") from None
        if header.get("format") != 1:
            raise ValueError(f"unsupported MPO format {header.get('format')}")
        ranks = header["ranks"]
        cores = []
        for k in range(header["num_cores"]):
            shape = (ranks[k], header["row_dims"][k], header["col_dims"][k], ranks[k + 1])
            nbytes = prod(shape) * 8
            raw = f.read(nbytes)
            if len(raw) != nbytes:
                raise ValueError(f"{path}: truncated core data")
            cores.append(np.frombuffer(raw, dtype="<f8").astype(np.float64)
                         .reshape(shape, order="F"))
    return Mpo(cores)


def read_matrix_market(path) -> SparseMatrixCoo:
    """Matrix Market file -> 1-based ``SparseMatrixCoo``."""
    import scipy.io
    mat = scipy.io.mmread(path)
    if np.iscomplexobj(mat):
        raise ValueError(f"{path}: complex matrices are not supported")
    if isinstance(mat, np.ndarray):
        return SparseMatrixCoo.from_dense(mat)
    coo = mat.tocoo()
    return SparseMatrixCoo(coo.shape[0], coo.shape[1], coo.row + 1, coo.col + 1, coo.data)


def write_matrix_market(path, a: SparseMatrixCoo) -> None:
    """Write ``%%MatrixMarket matrix coordinate real general``."""
    import scipy.io
    import scipy.sparse as sp
    m = sp.coo_matrix((a.val, (a.row - 1, a.col - 1)), shape=(a.rows, a.cols))
    scipy.io.mmwrite(path, m, symmetry="general")

"""MPO types of the drop-in API and their device residency.

``Mpo`` / ``SparseCore`` keep the reference's host-side semantics
(/root/reference/pkg/src/mposvd/mpo.py:63-204): validation, shapes, ranks,
``densify`` guard.  ``DeviceMpo`` is the same chain resident in HBM behind a
C-ABI handle (include/mpo_b200.h ``mpo_dev``), cores F-ordered exactly like
the serialized layout (mpo.py:17-23), so upload/download is one memcpy per
core.  All arithmetic on MPOs goes through the device (rsvd.py wrappers).
"""

from __future__ import annotations

import ctypes as C
from math import prod

import numpy as np

from . import _lib

__all__ = [
    "Mpo", "SparseCore", "DeviceMpo", "mpo_transpose", "random_unit_rank_mpo",
    "random_mpo", "identity_mpo", "zero_mpo", "mpo_add", "mpo_round",
    "contract_to_matrix", "CONTRACT_GUARD", "DENSIFY_GUARD",
]

CONTRACT_GUARD = 1 << 26   # mpo.py:56
DENSIFY_GUARD = 1 << 24    # mpo.py:58


class SparseCore:
    """A 4-way core holding only explicit nonzeros as parallel 0-based COO
    index arrays (mpo.py:63-108)."""

    __slots__ = ("shape", "left", "row", "col", "right", "values")

    def __init__(self, shape, left, row, col, right, values):
        self.shape = tuple(int(n) for n in shape)
        if len(self.shape) != 4 or min(self.shape) < 1:
            raise ValueError(f"bad core shape {shape}")
        self.left = np.asarray(left, dtype=np.int64).reshape(-1)
        self.row = np.asarray(row, dtype=np.int64).reshape(-1)
        self.col = np.asarray(col, dtype=np.int64).reshape(-1)
        self.right = np.asarray(right, dtype=np.int64).reshape(-1)
        self.values = np.asarray(values, dtype=np.float64).reshape(-1)

    @property
    def nnz(self) -> int:
        return self.values.size

    @property
    def size(self) -> int:
        return prod(self.shape)

    def to_dense(self) -> np.ndarray:
        out = np.zeros(self.shape)
        np.add.at(out, (self.left, self.row, self.col, self.right), self.values)
        return out

    def transpose(self) -> "SparseCore":
        r, i, j, s = self.shape
        return SparseCore((r, j, i, s), self.left, self.col, self.row, self.right,
                          self.values)

    def __repr__(self):
        return f"SparseCore(shape={self.shape}, nnz={self.nnz})"


def _dense(c):
    return c.to_dense() if isinstance(c, SparseCore) else c


class Mpo:
    """Chain of 4-way cores (R_k, I_k, J_k, R_{k+1}) with unit boundary
    ranks (mpo.py:119-204)."""

    __slots__ = ("cores",)

    def __init__(self, cores):
        cores = list(cores)
        if not cores:
            raise ValueError("an MPO needs at least one core")
        out = []
        for k, c in enumerate(cores):
            if not isinstance(c, SparseCore):
                c = np.asarray(c, dtype=np.float64)
                if c.ndim != 4:
                    raise ValueError(f"core {k} is {c.ndim}-way, expected 4")
                if min(c.shape) < 1:
                    raise ValueError(f"core {k} has empty extent {c.shape}")
            out.append(c)
        if out[0].shape[0] != 1 or out[-1].shape[3] != 1:
            raise ValueError("boundary ranks must be 1")
        for k in range(len(out) - 1):
            if out[k].shape[3] != out[k + 1].shape[0]:
                raise ValueError(
                    f"rank mismatch between cores {k} and {k + 1}: "
                    f"{out[k].shape[3]} vs {out[k + 1].shape[0]}")
        self.cores = out

    num_cores = property(lambda self: len(self.cores))
    row_dims = property(lambda self: tuple(c.shape[1] for c in self.cores))
    col_dims = property(lambda self: tuple(c.shape[2] for c in self.cores))
    num_rows = property(lambda self: prod(self.row_dims))
    num_cols = property(lambda self: prod(self.col_dims))

    @property
    def ranks(self) -> tuple:
        return tuple(c.shape[0] for c in self.cores) + (1,)

    @property
    def max_rank(self) -> int:
        return max(self.ranks)

    @property
    def is_sparse(self) -> bool:
        return any(isinstance(c, SparseCore) for c in self.cores)

    def copy(self) -> "Mpo":
        return Mpo([c if isinstance(c, SparseCore) else c.copy() for c in self.cores])

    def densify(self, limit: int | None = DENSIFY_GUARD) -> "Mpo":
        """Plain ndarray cores; refuses above ``limit`` entries (mpo.py:184-197)."""
        if not self.is_sparse:
            return self
        total = sum(prod(c.shape) for c in self.cores)
        if limit is not None and total > limit:
            raise ValueError(f"densifying needs {total} entries (> {limit}); "
                             "round the MPO or raise the limit")
        return Mpo([_dense(c) for c in self.cores])

    def to_device(self, device: int | None = None) -> "DeviceMpo":
        return DeviceMpo.from_host(self, device)

    def __add__(self, other):
        return mpo_add(self, other)

    def __repr__(self):
        return (f"Mpo(d={self.num_cores}, shape={self.num_rows}x{self.num_cols}, "
                f"ranks={list(self.ranks)})")


_PACK_LIMIT = 1 << 22   # doubles (32 MB): packed single-transfer up/downloads below this


class DeviceMpo:
    """An MPO resident in HBM (C-ABI handle ``mpo_dev``).  Cores are F-ordered
    FP64 device buffers owned by the library; freed with the handle."""

    __slots__ = ("handle", "ctx", "shapes")

    def __init__(self, handle, ctx):
        self.handle = handle
        self.ctx = ctx
        lib = _lib.load()
        d = C.c_int()
        _lib.check(lib.mpo_dev_num_cores(handle, C.byref(d)))
        sh = np.zeros(4 * d.value, dtype=np.int64)
        _lib.check(lib.mpo_dev_shapes(handle, sh.ctypes.data_as(_lib._I64P)))
        self.shapes = [tuple(int(x) for x in sh[4 * k:4 * k + 4]) for k in range(d.value)]

    @classmethod
    def from_host(cls, m: "Mpo", device: int | None = None) -> "DeviceMpo":
        m = m.densify()
        ctx = _lib.context(device)
        cores = [np.asarray(c, dtype=np.float64) for c in m.cores]
        shapes = np.array([s for c in cores for s in c.shape], dtype=np.int64)
        h = C.c_void_p()
        if sum(c.size for c in cores) <= _PACK_LIMIT:
            # one packed upload (small MPOs: per-core transfers are latency)
            packed = np.concatenate([c.ravel(order="F") for c in cores])
            _lib.call("mpo_dev_create_packed", ctx, len(cores),
                      shapes.ctypes.data_as(_lib._I64P), C.c_void_p(packed.ctypes.data), 1,
                      C.byref(h))
        else:
            cores = [np.asfortranarray(c) for c in cores]
            ptrs = (C.c_void_p * len(cores))(*[c.ctypes.data for c in cores])
            _lib.call("mpo_dev_create", ctx, len(cores), shapes.ctypes.data_as(_lib._I64P),
                      ptrs, 1, C.byref(h))
        return cls(h, ctx)

    @classmethod
    def from_device_ptrs(cls, shapes, ptrs, device: int | None = None) -> "DeviceMpo":
        """Build from device buffers (e.g. torch CUDA tensors' data_ptr())."""
        ctx = _lib.context(device)
        sh = np.array([s for shp in shapes for s in shp], dtype=np.int64)
        arr = (C.c_void_p * len(ptrs))(*[int(p) for p in ptrs])
        h = C.c_void_p()
        _lib.call("mpo_dev_create", ctx, len(ptrs), sh.ctypes.data_as(_lib._I64P), arr, 0,
                  C.byref(h))
        return cls(h, ctx)

    num_cores = property(lambda self: len(self.shapes))
    row_dims = property(lambda self: tuple(s[1] for s in self.shapes))
    col_dims = property(lambda self: tuple(s[2] for s in self.shapes))

    @property
    def ranks(self) -> tuple:
        return tuple(s[0] for s in self.shapes) + (1,)

    def core_ptr(self, k: int) -> int:
        p = C.c_void_p()
        _lib.call("mpo_dev_core_ptr", self.handle, k, C.byref(p))
        return int(p.value or 0)

    def core(self, k: int) -> np.ndarray:
        shp = self.shapes[k]
        out = _host_buffer(shp)
        _lib.call("mpo_dev_copy_core", self.ctx, self.handle, k, C.c_void_p(out.ctypes.data), 1)
        return out

    def to_host(self) -> Mpo:
        # cores stay in the device's F order (same values and shapes; a C-order
        # copy would be a strided transpose of every core on the host).  Small
        # MPOs come down in ONE packed transfer, the cores as views of it.
        sizes = [int(np.prod(s)) for s in self.shapes]
        if sum(sizes) > _PACK_LIMIT:
            return Mpo([self.core(k) for k in range(self.num_cores)])
        buf = np.empty(sum(sizes), dtype=np.float64)
        _lib.call("mpo_dev_copy_all", self.ctx, self.handle, C.c_void_p(buf.ctypes.data), 1)
        out, off = [], 0
        for s, n in zip(self.shapes, sizes):
            out.append(buf[off:off + n].reshape(s, order="F"))
            off += n
        return Mpo(out)

    def free(self):
        if self.handle is not None and self.handle.value:
            _lib.load().mpo_dev_free(self.handle)
        self.handle = None

    def __del__(self):
        try:
            self.free()
        except Exception:  # pragma: no cover - interpreter shutdown
            pass

    def __repr__(self):
        return f"DeviceMpo(d={self.num_cores}, ranks={list(self.ranks)})"


def _host_buffer(shape) -> np.ndarray:
    """F-ordered float64 (pinned when CUDA is up) host array for a download."""
    return _lib.host_empty(shape, np.float64, order="F")


def _wrap(ctx, handle) -> DeviceMpo:
    return DeviceMpo(handle, ctx)


def _to_dev(m) -> DeviceMpo:
    return m if isinstance(m, DeviceMpo) else DeviceMpo.from_host(m)


def mpo_transpose(m):
    """Swap row/col axes of every core (mpo.py:402-410)."""
    if isinstance(m, DeviceMpo):
        h = C.c_void_p()
        _lib.call("mpo_transpose", m.ctx, m.handle, C.byref(h))
        return _wrap(m.ctx, h)
    cores = []
    for c in m.cores:
        if isinstance(c, SparseCore):
            cores.append(c.transpose())
        else:
            cores.append(np.ascontiguousarray(c.transpose(0, 2, 1, 3)))
    return Mpo(cores)


def mpo_add(a, b):
    """Sum over the same index grid by block-diagonal stacking (mpo.py:264-294),
    computed on the device."""
    host = not isinstance(a, DeviceMpo)
    if host:
        if a.num_cores != b.num_cores:
            raise ValueError(f"core counts differ: {a.num_cores} vs {b.num_cores}")
        if a.row_dims != b.row_dims or a.col_dims != b.col_dims:
            raise ValueError("per-core row/col extents differ")
    da, db = _to_dev(a), _to_dev(b)
    h = C.c_void_p()
    _lib.call("mpo_add", da.ctx, da.handle, db.handle, C.byref(h))
    out = _wrap(da.ctx, h)
    return out.to_host() if host else out


def mpo_round(m, rel_tol: float):
    """Rank truncation within rel_tol * ||m||_F (mpo.py:323-354) on the device."""
    if rel_tol < 0:
        raise ValueError("rel_tol must be >= 0")
    host = not isinstance(m, DeviceMpo)
    dm = _to_dev(m)
    h = C.c_void_p()
    _lib.call("mpo_round", dm.ctx, dm.handle, float(rel_tol), C.byref(h))
    out = _wrap(dm.ctx, h)
    return out.to_host() if host else out


def random_unit_rank_mpo(row_dims, k: int, seed=None) -> Mpo:
    """Random k-column unit-rank MPO; draws the reference's exact numpy
    stream (mpo.py:413-433) so sketches are bit-identical."""
    row_dims = [int(n) for n in row_dims]
    if not row_dims or min(row_dims) < 1:
        raise ValueError(f"bad row dims {row_dims}")
    if not 1 <= k <= row_dims[0]:
        raise ValueError(f"k = {k} exceeds the leading extent {row_dims[0]}; "
                         "merge leading cores first")
    rng = np.random.default_rng(seed)
    cores = [rng.standard_normal((1, row_dims[0], k, 1))]
    cores += [rng.standard_normal((1, n, 1, 1)) for n in row_dims[1:]]
    return Mpo(cores)


def random_mpo(row_dims, col_dims, interior_ranks, seed=None) -> Mpo:
    """Dense N(0,1) MPO, same draw order as mpo.py:436-449."""
    row_dims = [int(n) for n in row_dims]
    col_dims = [int(n) for n in col_dims]
    if len(col_dims) != len(row_dims):
        raise ValueError("row/col dim lists must have equal length")
    ranks = [1] + [int(r) for r in interior_ranks] + [1]
    if len(ranks) != len(row_dims) + 1:
        raise ValueError(f"need {len(row_dims) - 1} interior ranks, got {len(ranks) - 2}")
    rng = np.random.default_rng(seed)
    return Mpo([rng.standard_normal((ranks[k], row_dims[k], col_dims[k], ranks[k + 1]))
                for k in range(len(row_dims))])


def identity_mpo(dims) -> Mpo:
    return Mpo([np.eye(int(n)).reshape(1, int(n), int(n), 1) for n in dims])


def zero_mpo(row_dims, col_dims) -> Mpo:
    """Canonical all-zero MPO (mpo.py:457-462)."""
    if len(row_dims) != len(col_dims):
        raise ValueError("row/col dim lists must have equal length")
    return Mpo([np.zeros((1, int(i), int(j), 1)) for i, j in zip(row_dims, col_dims)])


def contract_to_matrix(m: Mpo, guard: int = CONTRACT_GUARD) -> np.ndarray:
    """Dense matrix of a desk-scale MPO (verification helper, mpo.py:214-238;
    host numpy, not part of the device path)."""
    rows, cols = m.num_rows, m.num_cols
    if rows * cols > guard:
        raise ValueError(f"contraction would create {rows}x{cols} entries (> {guard})")
    cores = [_dense(c) for c in m.cores]
    t = cores[0][0]
    for c in cores[1:]:
        a_, b_, _ = t.shape
        _, i_, j_, s_ = c.shape
        n = np.tensordot(t, c, axes=(2, 0)).transpose(0, 2, 1, 3, 4)
        t = n.reshape(a_ * i_, b_ * j_, s_, order="F")
    return t[:, :, 0].copy()

"""Sparse -> MPO conversion drop-in (reference:
/root/reference/pkg/src/mposvd/sparse.py:43-93 and :207-275).

``matrix_to_mpo`` runs Algorithm 1 on the device: the per-nonzero
mixed-radix split, block keying, the atomics-free radix sort-and-segment
that yields block ids, and the core scatter (convert.cu).  The returned
``Mpo`` has exactly the reference's structure: dense cores when their total
footprint fits ``densify_limit`` (densified on the device), else a
``SparseCore`` chain whose index arrays are bit-identical to the
reference's.  The capped path (rank_cap) runs the reference's chunked
accumulation with the device ``mpo_add`` / ``mpo_round``.
"""

from __future__ import annotations

import ctypes as C
from math import prod

import numpy as np

from . import _lib
from .mpo import DENSIFY_GUARD, DeviceMpo, Mpo, SparseCore, mpo_add, mpo_round, zero_mpo
from .partition import PartitionPlan

__all__ = ["SparseMatrixCoo", "matrix_to_mpo", "ConversionResult", "convert_structure",
           "min_rank_lower_bound"]


class SparseMatrixCoo:
    """1-based (row, col, value) coordinate matrix (sparse.py:43-93).
    Duplicates and out-of-range coordinates are rejected; stored zeros are
    kept but do not count as nonzeros."""

    __slots__ = ("rows", "cols", "row", "col", "val")

    def __init__(self, rows, cols, row, col, val):
        self.rows = int(rows)
        self.cols = int(cols)
        if self.rows < 1 or self.cols < 1:
            raise ValueError("matrix dimensions must be >= 1")
        self.row = np.asarray(row, dtype=np.int64).reshape(-1)
        self.col = np.asarray(col, dtype=np.int64).reshape(-1)
        self.val = np.asarray(val, dtype=np.float64).reshape(-1)
        if not (self.row.size == self.col.size == self.val.size):
            raise ValueError("row/col/val arrays must have equal length")
        if self.row.size:
            if self.row.min() < 1 or self.row.max() > self.rows:
                raise ValueError("row index out of range")
            if self.col.min() < 1 or self.col.max() > self.cols:
                raise ValueError("col index out of range")
            keys = (self.row - 1) * self.cols + (self.col - 1)
            keys.sort()
            if keys.size > 1 and bool(np.any(keys[1:] == keys[:-1])):
                raise ValueError("duplicate (row, col) entries rejected")

    @property
    def nnz(self) -> int:
        return int(np.count_nonzero(self.val))

    @classmethod
    def from_dense(cls, arr) -> "SparseMatrixCoo":
        arr = np.asarray(arr, dtype=np.float64)
        r, c = np.nonzero(arr)
        return cls(arr.shape[0], arr.shape[1], r + 1, c + 1, arr[r, c])

    def to_scipy(self):
        import scipy.sparse as sp
        return sp.coo_matrix((self.val, (self.row - 1, self.col - 1)),
                             shape=(self.rows, self.cols))

    def to_dense(self) -> np.ndarray:
        out = np.zeros((self.rows, self.cols))
        out[self.row - 1, self.col - 1] = self.val
        return out

    def __repr__(self):
        return f"SparseMatrixCoo({self.rows}x{self.cols}, nnz={self.nnz})"


def min_rank_lower_bound(z: int, i1: int, j1: int) -> int:
    """ceil(z / (I1*J1)) (sparse.py:163-170)."""
    if i1 < 1 or j1 < 1:
        raise ValueError("block dimensions must be >= 1")
    if z < 0:
        raise ValueError("nonzero count must be >= 0")
    return -(-z // (i1 * j1))


class ConversionResult:
    """Device-resident conversion structure (C-ABI handle ``mpo_conv``):
    per kept nonzero i1, j1, ti, values (masked input order) and the sorted
    unique block keys; the rank is the nonzero block count (Lemma 4.2)."""

    __slots__ = ("handle", "ctx", "plan", "nkept", "rank")

    def __init__(self, handle, ctx, plan):
        self.handle, self.ctx, self.plan = handle, ctx, plan
        nk, rk = C.c_int64(), C.c_int64()
        _lib.check(_lib.load().mpo_conv_info(handle, C.byref(nk), C.byref(rk)))
        self.nkept, self.rank = int(nk.value), int(rk.value)

    def arrays(self):
        """(i1, j1, ti, values, uniq) as host arrays."""
        n, r = self.nkept, self.rank
        i1, j1, ti = (_lib.host_empty(n, np.int64) for _ in range(3))
        v = _lib.host_empty(n, np.float64)
        u = _lib.host_empty(r, np.int64)
        _lib.call("mpo_conv_copy", self.ctx, self.handle, _lib.ptr(i1), _lib.ptr(j1),
                  _lib.ptr(ti), _lib.ptr(v), _lib.ptr(u), 1)
        return i1, j1, ti, v, u

    def level(self, k: int):
        """Block digits (row, col) of core k >= 1 (sparse.py:249-250)."""
        rd = _lib.host_empty(self.rank, np.int64); cd = _lib.host_empty(self.rank, np.int64)
        _lib.call("mpo_conv_level", self.ctx, self.handle, int(k), _lib.ptr(rd), _lib.ptr(cd), 1)
        return rd, cd

    def dense_core(self, k: int) -> np.ndarray:
        rf, cf, d, r = self.plan.row_factors, self.plan.col_factors, self.plan.d, self.rank
        shape = (1, rf[0], cf[0], r) if k == 0 else (r, rf[k], cf[k], r if k < d - 1 else 1)
        out = np.empty(shape, dtype=np.float64, order="F")
        _lib.call("mpo_conv_dense_core", self.ctx, self.handle, int(k),
                  C.c_void_p(out.ctypes.data), 1)
        return np.ascontiguousarray(out)

    def free(self):
        if self.handle is not None and self.handle.value:
            _lib.load().mpo_conv_free(self.handle)
        self.handle = None

    def __del__(self):
        try:
            self.free()
        except Exception:  # pragma: no cover
            pass


def convert_structure(row1, col1, val, plan: PartitionPlan, device=None,
                      n_device: int | None = None) -> ConversionResult:
    """Run the device conversion on 1-based COO arrays.  With ``n_device``
    set, the three arguments are device pointers (ints, e.g. torch CUDA
    tensors' data_ptr()) holding that many entries; else host arrays."""
    ctx = _lib.context(device)
    rf = _lib.as_i64(plan.row_factors)
    cf = _lib.as_i64(plan.col_factors)
    h = C.c_void_p()
    if n_device is not None:
        _lib.call("mpo_sparse_convert", ctx, C.c_void_p(row1), C.c_void_p(col1),
                  C.c_void_p(val), int(n_device), 0, plan.d, rf.ctypes.data_as(_lib._I64P),
                  cf.ctypes.data_as(_lib._I64P), C.byref(h))
    else:
        r = _lib.as_i64(row1); c = _lib.as_i64(col1)
        v = np.ascontiguousarray(val, dtype=np.float64)
        _lib.call("mpo_sparse_convert", ctx, _lib.ptr(r), _lib.ptr(c), _lib.ptr(v), r.size, 1,
                  plan.d, rf.ctypes.data_as(_lib._I64P), cf.ctypes.data_as(_lib._I64P),
                  C.byref(h))
    return ConversionResult(h, ctx, plan)


class _LevelCore(SparseCore):
    """Block core k >= 1 of the SparseCore chain (sparse.py:195-203) whose
    per-block digit arrays (``row``, ``col``) stay on the device until first
    read: the reference materialises all 2(d-1) of them (10.9 GB at config
    5), most callers touch none or a few."""

    __slots__ = ("_res", "_k", "_rd", "_cd")

    def __init__(self, shape, left, right, values, res, k):
        SparseCore.__init__(self, shape, left, _EMPTY, _EMPTY, right, values)
        self._res, self._k, self._rd, self._cd = res, k, None, None

    def _fetch(self):
        if self._rd is None:
            self._rd, self._cd = self._res.level(self._k)
        return self._rd, self._cd

    @property
    def row(self):
        return self._fetch()[0]

    @row.setter
    def row(self, v):
        pass

    @property
    def col(self):
        return self._fetch()[1]

    @col.setter
    def col(self, v):
        pass

    def transpose(self) -> SparseCore:
        r, i, j, s = self.shape
        return SparseCore((r, j, i, s), self.left, self.col, self.row, self.right, self.values)


_EMPTY = np.zeros(0, dtype=np.int64)


def _sparse_cores(res: ConversionResult, i1, j1, ti, values, rank):
    plan = res.plan
    d = plan.d
    cores = [SparseCore((1, plan.row_factors[0], plan.col_factors[0], rank),
                        np.zeros_like(ti), i1, j1, ti, values)]
    # shared by every block core, as in the reference (sparse.py:194-195)
    t = np.arange(rank, dtype=np.int64)
    ones = np.ones(rank)
    zero = np.zeros_like(t)
    for k in range(1, d):
        last = k == d - 1
        cores.append(_LevelCore((rank, plan.row_factors[k], plan.col_factors[k],
                                 1 if last else rank),
                                t, zero if last else t, ones, res, k))
    return cores


def matrix_to_mpo(a: SparseMatrixCoo, plan: PartitionPlan, rank_cap: int | None = None,
                  round_tol: float | None = None,
                  densify_limit: int | None = DENSIFY_GUARD) -> Mpo:
    """Algorithm 1 (sparse.py:207-275) on the device."""
    if rank_cap is not None and rank_cap < 1:
        raise ValueError("rank_cap must be >= 1")
    if plan.rows < a.rows or plan.cols < a.cols:
        raise ValueError(f"plan covers {plan.rows}x{plan.cols} but the matrix is "
                         f"{a.rows}x{a.cols}")
    if not np.any(a.val != 0):
        return zero_mpo(plan.row_factors, plan.col_factors)
    res = convert_structure(a.row, a.col, a.val, plan)
    rank = res.rank
    d = plan.d
    if rank_cap is None or rank <= rank_cap or d == 1:
        total = plan.row_factors[0] * plan.col_factors[0] * rank + sum(
            rank * plan.row_factors[k] * plan.col_factors[k] * (rank if k < d - 1 else 1)
            for k in range(1, d))
        if densify_limit is None or total <= densify_limit:
            return Mpo([res.dense_core(k) for k in range(d)])
        i1, j1, ti, values, _ = res.arrays()
        return Mpo(_sparse_cores(res, i1, j1, ti, values, rank))
    # capped accumulation (sparse.py:260-275): chunks of rank_cap unit-rank
    # terms built as dense device cores straight from the conversion handle
    # (mpo_conv_chunk), stacked with mpo_add and rounded, all on the device
    tol = 1e-14 if round_tol is None else round_tol
    acc = None
    for start in range(0, rank, rank_cap):
        stop = min(start + rank_cap, rank)
        h = C.c_void_p()
        _lib.call("mpo_conv_chunk", res.ctx, res.handle, int(start), int(stop), C.byref(h))
        chunk = DeviceMpo(h, res.ctx)
        acc = chunk if acc is None else mpo_add(acc, chunk)
        if max(acc.ranks) >= rank_cap:
            acc = mpo_round(acc, tol)
    return acc.to_host()

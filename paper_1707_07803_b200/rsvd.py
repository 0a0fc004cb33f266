"""TNrSVD drop-in API (reference: /root/reference/pkg/src/mposvd/rsvd.py).

Same names, signatures, defaults and ValueError preconditions as the
reference; the work runs on the B200 through the C-ABI (include/mpo_b200.h).
Host-side logic kept here is integer bookkeeping only: the sketch width
K (rsvd.py:235), the leading-core merge count (rsvd.py:236-243) and the
sketch O drawn from numpy's generator in the reference's call order
(mpo.py:430-432) so that both paths consume a bit-identical sketch.

Each function accepts host ``Mpo`` objects (results come back as host
``Mpo``) or ``DeviceMpo`` handles (results stay in HBM).
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from math import ceil

import numpy as np

from . import _lib
from .mpo import (DeviceMpo, Mpo, contract_to_matrix, mpo_transpose,
                  random_unit_rank_mpo, CONTRACT_GUARD)

__all__ = ["LowRankSvd", "mpo_matmul", "merge_leading_cores", "mpo_qr", "mpo_svd",
           "subspace_iteration", "tnrsvd", "reconstruct_matrix", "DEFAULT_ROUND_TOL",
           "sketch_width", "merge_count"]

DEFAULT_ROUND_TOL = 1e-9   # rsvd.py:43


@dataclass
class LowRankSvd:
    """U diag(s) V^T with MPO factors (rsvd.py:46-59)."""

    u: object
    s: np.ndarray
    v: object
    k_target: int
    k_oversampled: int


def _dev(m) -> tuple[DeviceMpo, bool]:
    if isinstance(m, DeviceMpo):
        return m, False
    return DeviceMpo.from_host(m), True


def _out(ctx, h, host: bool):
    d = DeviceMpo(h, ctx)
    return d.to_host() if host else d


def _tol(round_tol):
    return (0.0, 0) if round_tol is None else (float(round_tol), 1)


def mpo_matmul(a, o):
    """Per-core product; interior ranks multiply (rsvd.py:62-79)."""
    if a.num_cores != o.num_cores:
        raise ValueError("operands must have the same number of cores")
    if tuple(a.col_dims) != tuple(o.row_dims):
        raise ValueError(f"inner dims differ per core: {a.col_dims} vs {o.row_dims}")
    da, host = _dev(a)
    do, _ = _dev(o)
    h = C.c_void_p()
    _lib.call("mpo_matmul", da.ctx, da.handle, 0, do.handle, 0, C.byref(h))
    return _out(da.ctx, h, host)


def merge_leading_cores(m, count: int):
    """Contract the first ``count`` cores into one (rsvd.py:82-99);
    count == 1 returns ``m`` itself."""
    if not 1 <= count <= m.num_cores:
        raise ValueError(f"count {count} out of range [1, {m.num_cores}]")
    if count == 1:
        return m
    dm, host = _dev(m)
    h = C.c_void_p()
    _lib.call("mpo_merge_leading_cores", dm.ctx, dm.handle, int(count), C.byref(h))
    return _out(dm.ctx, h, host)


def mpo_qr(y, round_tol: float | None = None):
    """Thin QR of a tall MPO (Algorithm 3, rsvd.py:139-166): (Q, R[K x K])."""
    r0, i1, k, _ = (y.cores[0].shape if isinstance(y, Mpo) else y.shapes[0])
    if i1 < k:
        raise ValueError(f"first core has I1 = {i1} < K = {k}; merge leading cores first")
    dy, host = _dev(y)
    tol, has = _tol(round_tol)
    r = np.zeros((k, k), dtype=np.float64, order="F")
    h = C.c_void_p()
    _lib.call("mpo_qr", dy.ctx, dy.handle, tol, has, C.byref(h),
              r.ctypes.data_as(_lib._DP))
    return _out(dy.ctx, h, host), np.ascontiguousarray(r)


def mpo_svd(b, round_tol: float | None = None):
    """Economical SVD of a short-wide MPO (Algorithm 4, rsvd.py:169-193):
    (W[K x K], s[K], tall V)."""
    _, k, j1, _ = (b.cores[0].shape if isinstance(b, Mpo) else b.shapes[0])
    if j1 < k:
        raise ValueError(f"first core has J1 = {j1} < K = {k}; merge leading cores first")
    db, host = _dev(b)
    tol, has = _tol(round_tol)
    w = np.zeros((k, k), dtype=np.float64, order="F")
    s = np.zeros(k, dtype=np.float64)
    h = C.c_void_p()
    _lib.call("mpo_svd", db.ctx, db.handle, tol, has, w.ctypes.data_as(_lib._DP),
              s.ctypes.data_as(_lib._DP), C.byref(h))
    return np.ascontiguousarray(w), s, _out(db.ctx, h, host)


def subspace_iteration(a, o, q: int = 2, round_tol: float | None = DEFAULT_ROUND_TOL):
    """Randomized MPO subspace iteration (Algorithm 5, rsvd.py:196-214)."""
    if q < 0:
        raise ValueError("q must be >= 0")
    da, host = _dev(a)
    do, _ = _dev(o)
    tol, has = _tol(round_tol)
    h = C.c_void_p()
    _lib.call("mpo_subspace_iteration", da.ctx, da.handle, do.handle, int(q), tol, has,
              C.byref(h))
    return _out(da.ctx, h, host)


def sketch_width(k_target: int, oversample: float) -> int:
    """K = max(k, ceil(oversample * k)) (rsvd.py:235)."""
    return max(int(k_target), int(ceil(oversample * k_target)))


def merge_count(row_dims, col_dims, k: int) -> int:
    """First core count whose cumulative row and column extents reach K
    (rsvd.py:236-243)."""
    rc = cc = 1
    for idx, (r, c) in enumerate(zip(row_dims, col_dims)):
        rc *= int(r)
        cc *= int(c)
        if rc >= k and cc >= k:
            return idx + 1
    raise ValueError(f"matrix {rc}x{cc} cannot host a width-{k} sketch")


def _merged_col_dims(col_dims, count):
    lead = 1
    for c in col_dims[:count]:
        lead *= int(c)
    return (lead,) + tuple(int(c) for c in col_dims[count:])


def tnrsvd(a, k_target: int, q: int = 2, round_tol: float | None = DEFAULT_ROUND_TOL,
           oversample: float = 2.0, seed=None) -> LowRankSvd:
    """Randomized rank-``k_target`` SVD in MPO form (Algorithm 2,
    rsvd.py:217-259), computed on the device."""
    if k_target < 1:
        raise ValueError("k_target must be >= 1")
    kk = sketch_width(k_target, oversample)
    cnt = merge_count(a.row_dims, a.col_dims, kk)
    host = not isinstance(a, DeviceMpo)
    if host:
        a = a.densify()   # rsvd.py:243 (guarded like Mpo.densify)
    da, _ = _dev(a)
    if cnt > 1:
        h = C.c_void_p()
        _lib.call("mpo_merge_leading_cores", da.ctx, da.handle, cnt, C.byref(h))
        am = DeviceMpo(h, da.ctx)
    else:
        am = da
    o = random_unit_rank_mpo(_merged_col_dims(a.col_dims, cnt), kk, seed)
    do = DeviceMpo.from_host(o)
    s = np.zeros(k_target, dtype=np.float64)
    hu, hv = C.c_void_p(), C.c_void_p()
    tol, has = _tol(round_tol)
    _lib.call("mpo_tnrsvd", da.ctx, am.handle, do.handle, int(k_target), int(q), tol, has,
              C.byref(hu), s.ctypes.data_as(_lib._DP), C.byref(hv))
    u = _out(da.ctx, hu, host)
    v = _out(da.ctx, hv, host)
    return LowRankSvd(u=u, s=s, v=v, k_target=int(k_target), k_oversampled=kk)


def prepare(a, k_target: int, oversample: float = 2.0, seed=None):
    """Device-resident inputs of one TNrSVD: the merged operator and the
    sketch (rsvd.py:235-244), so a timed step starts with both in HBM."""
    kk = sketch_width(k_target, oversample)
    cnt = merge_count(a.row_dims, a.col_dims, kk)
    da, _ = _dev(a if isinstance(a, DeviceMpo) else a.densify())
    am = merge_leading_cores(da, cnt) if cnt > 1 else da
    o = DeviceMpo.from_host(random_unit_rank_mpo(_merged_col_dims(a.col_dims, cnt), kk, seed))
    return am, o, kk


def tnrsvd_prepared(am: DeviceMpo, o: DeviceMpo, k_target: int, q: int = 2,
                    round_tol: float | None = DEFAULT_ROUND_TOL):
    """The device pipeline of rsvd.py:244-259 on prepared inputs; returns
    (U, s, V) with U, V resident in HBM."""
    s = np.zeros(k_target, dtype=np.float64)
    hu, hv = C.c_void_p(), C.c_void_p()
    tol, has = _tol(round_tol)
    _lib.call("mpo_tnrsvd", am.ctx, am.handle, o.handle, int(k_target), int(q), tol, has,
              C.byref(hu), s.ctypes.data_as(_lib._DP), C.byref(hv))
    return DeviceMpo(hu, am.ctx), s, DeviceMpo(hv, am.ctx)


def reconstruct_matrix(lr: LowRankSvd, guard: int | None = None) -> np.ndarray:
    """Dense U diag(s) V^T (desk-scale verification helper)."""
    g = CONTRACT_GUARD if guard is None else guard
    u = contract_to_matrix(lr.u if isinstance(lr.u, Mpo) else lr.u.to_host(), g)
    v = contract_to_matrix(lr.v if isinstance(lr.v, Mpo) else lr.v.to_host(), g)
    return (u * lr.s) @ v.T


# re-export for the rsvd namespace (reference rsvd.py imports it)
mpo_transpose = mpo_transpose

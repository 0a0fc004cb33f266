"""CPU ORACLE -- TEST INFRASTRUCTURE ONLY.

This module is the checker for the B200 hot path.  Only ``tests/``,
``__graft_entry__.smoke()`` and the ``cpu_baseline`` / ``--impl reference``
legs of ``bench.py`` may import it; the product package
(``paper_1707_07803_b200``) never does, and fails loudly when its CUDA
library is missing instead of falling back to anything here.

It restates, in plain numpy (LAPACK dgeqrf/dorgqr via ``np.linalg.qr``,
dgesdd via ``np.linalg.svd``, dgemm via ``@``), the reference algorithms of
arXiv 1707.07803 as implemented by the reference package ``mposvd``
(/root/reference/pkg/src/mposvd).  Each function cites the reference
file:line it follows.  Cores are numpy arrays indexed (R, I, J, S);
reshapes use first-index-fastest ("F") order exactly like the reference.

Parity pin: ``tests/golden/*.npz`` were produced by importing the
unmodified reference in the build container (``tests/golden/make_golden.py``)
and ``tests/test_oracle_golden.py`` checks this restatement against them
(bit-exact for the conversion structure, <= 1e-12 relative for TNrSVD).
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass, field

import numpy as np

# ---------------------------------------------------------------------------
# flop ledger: algorithmic work the reference performs
# ---------------------------------------------------------------------------


@dataclass
class Ledger:
    """Counts the FP64 work of the reference's LAPACK/BLAS calls.

    qr(m x n): 2*(2*M*N^2 - 2*N^3/3) with M = max, N = min (dgeqrf+dorgqr);
    svd(m x n): 6*M*N^2 + 20*N^3; gemm: 2*out*contracted; einsum: 2*out*J.
    """

    qr: float = 0.0
    svd: float = 0.0
    gemm: float = 0.0
    einsum: float = 0.0
    calls: list = field(default_factory=list)
    keep_calls: bool = False

    @property
    def total(self) -> float:
        return self.qr + self.svd + self.gemm + self.einsum

    def add(self, kind: str, flops: float, shape):
        setattr(self, kind, getattr(self, kind) + float(flops))
        if self.keep_calls:
            self.calls.append((kind, tuple(shape), float(flops)))


def _qr_flops(m, n):
    big, small = max(m, n), min(m, n)
    return 2.0 * (2.0 * big * small * small - 2.0 * small ** 3 / 3.0)


def _svd_flops(m, n):
    big, small = max(m, n), min(m, n)
    return 6.0 * big * small * small + 20.0 * small ** 3


# ---------------------------------------------------------------------------
# MPO helpers (mpo.py)
# ---------------------------------------------------------------------------


def check_chain(cores):
    """Validation of mpo.py:119-145 (4-way cores, unit boundary ranks)."""
    if not cores:
        raise ValueError("an MPO needs at least one core")
    for k, c in enumerate(cores):
        if c.ndim != 4:
            raise ValueError(f"core {k} is {c.ndim}-way, expected 4")
    if cores[0].shape[0] != 1 or cores[-1].shape[3] != 1:
        raise ValueError("boundary ranks must be 1")
    for k in range(len(cores) - 1):
        if cores[k].shape[3] != cores[k + 1].shape[0]:
            raise ValueError(f"rank mismatch between cores {k} and {k + 1}")


def ranks_of(cores):
    return tuple(c.shape[0] for c in cores) + (1,)


def random_mpo(row_dims, col_dims, interior_ranks, seed=None):
    """N(0,1) cores drawn core by core in C order (mpo.py:436-449)."""
    rng = np.random.default_rng(seed)
    rk = [1] + [int(r) for r in interior_ranks] + [1]
    return [rng.standard_normal((rk[k], int(row_dims[k]), int(col_dims[k]),
                                 rk[k + 1])) for k in range(len(row_dims))]


def random_unit_rank_mpo(row_dims, k, seed=None):
    """Sketch O: core 0 (1,J1,k,1) then (1,n,1,1) per level (mpo.py:413-433)."""
    row_dims = [int(n) for n in row_dims]
    if not row_dims or min(row_dims) < 1:
        raise ValueError(f"bad row dims {row_dims}")
    if not 1 <= k <= row_dims[0]:
        raise ValueError(f"k = {k} exceeds the leading extent {row_dims[0]}")
    rng = np.random.default_rng(seed)
    out = [rng.standard_normal((1, row_dims[0], k, 1))]
    for n in row_dims[1:]:
        out.append(rng.standard_normal((1, n, 1, 1)))
    return out


def transpose_cores(cores):
    """Swap row/col axes per core (mpo.py:402-410)."""
    return [np.ascontiguousarray(c.transpose(0, 2, 1, 3)) for c in cores]


def contract(cores, guard=1 << 26):
    """Dense matrix of an MPO (mpo.py:214-238): row index i1 + I1*i2 + ...,
    rank slices multiplied last core leftmost."""
    rows = math.prod(c.shape[1] for c in cores)
    cols = math.prod(c.shape[2] for c in cores)
    if rows * cols > guard:
        raise ValueError("contraction too large")
    t = cores[0][0]                       # (A, B, r)
    for c in cores[1:]:
        a_, b_, r_ = t.shape
        _, i_, j_, s_ = c.shape
        n = np.tensordot(t, c, axes=(2, 0))           # (A, B, I, J, S)
        n = n.transpose(0, 2, 1, 3, 4)                 # (A, I, B, J, S)
        t = n.reshape(a_ * i_, b_ * j_, s_, order="F")
    return t[:, :, 0]


def mpo_add(x, y):
    """Block-diagonal stacking sum (mpo.py:264-294)."""
    d = len(x)
    if d == 1:
        return [x[0] + y[0]]
    out = []
    for k, (a, b) in enumerate(zip(x, y)):
        ra, i_, j_, sa = a.shape
        rb, _, _, sb = b.shape
        r = 1 if k == 0 else ra + rb
        s = 1 if k == d - 1 else sa + sb
        c = np.zeros((r, i_, j_, s))
        if k == 0:
            c[:, :, :, :sa] = a
            c[:, :, :, sa:] = b
        elif k == d - 1:
            c[:ra] = a
            c[ra:] = b
        else:
            c[:ra, :, :, :sa] = a
            c[ra:, :, :, sa:] = b
        out.append(c)
    return out


def mpo_frobenius(cores):
    """||M||_F by a left-to-right QR sweep: the norm ends up in the last
    core, so no cancellation (used for the MPO-form residual)."""
    cs = [c.copy() for c in cores]
    for k in range(len(cs) - 1):
        r, i_, j_, s = cs[k].shape
        _, rm = np.linalg.qr(cs[k].reshape(r * i_ * j_, s, order="F"))
        cs[k + 1] = np.tensordot(rm, cs[k + 1], axes=(1, 0))
    return float(np.linalg.norm(cs[-1]))


def scale_first(cores, alpha):
    out = [c.copy() for c in cores]
    out[0] = out[0] * alpha
    return out


def truncation_rank(s, delta, rel_tol):
    """mpo.py:297-304: smallest r whose discarded tail sum of s^2 is
    <= delta^2 (ties toward smaller r), floor 1; rel_tol == 0 keeps the
    nonzeros."""
    if rel_tol == 0.0:
        return max(int(np.count_nonzero(s)), 1)
    sq = s * s
    tail = np.append(np.cumsum(sq[::-1])[::-1], 0.0)
    ok = np.nonzero(tail <= delta * delta)[0]
    return max(int(ok[0]), 1)


# ---------------------------------------------------------------------------
# TNrSVD pipeline (rsvd.py)
# ---------------------------------------------------------------------------


def mpo_matmul(a, b, ledger=None):
    """Per-core product, bond index a + Ra*c (rsvd.py:62-79)."""
    if len(a) != len(b):
        raise ValueError("operands must have the same number of cores")
    if tuple(c.shape[2] for c in a) != tuple(c.shape[1] for c in b):
        raise ValueError("inner dims differ per core")
    out = []
    for ca, cb in zip(a, b):
        ra, i_, j_, sa = ca.shape
        rc, _, k_, sc = cb.shape
        n = np.einsum("aijb,cjkd->acikbd", ca, cb)
        if ledger is not None:
            ledger.add("einsum", 2.0 * n.size * j_, n.shape)
        out.append(n.reshape(ra * rc, i_, k_, sa * sc, order="F"))
    return out


def merge_leading(cores, count, ledger=None):
    """Contract cores 0..count-1 into one (rsvd.py:82-99); merged row
    index a + A*i."""
    if not 1 <= count <= len(cores):
        raise ValueError(f"count {count} out of range")
    if count == 1:
        return list(cores)
    t = cores[0]
    for c in cores[1:count]:
        _, a_, b_, r_ = t.shape
        _, i_, j_, s_ = c.shape
        n = t.reshape(a_ * b_, r_, order="F") @ c.reshape(r_, i_ * j_ * s_,
                                                          order="F")
        if ledger is not None:
            ledger.add("gemm", 2.0 * n.size * r_, n.shape)
        n = n.reshape(a_, b_, i_, j_, s_, order="F").transpose(0, 2, 1, 3, 4)
        t = n.reshape(1, a_ * i_, b_ * j_, s_, order="F")
    return [t] + list(cores[count:])


def _l2r(cores, ledger):
    """rsvd.py:102-108: reduced QR of the (R*I*J x S) unfolding per core,
    R factor absorbed into the next core."""
    for k in range(len(cores) - 1):
        r, i_, j_, s = cores[k].shape
        q, rm = np.linalg.qr(cores[k].reshape(r * i_ * j_, s, order="F"))
        if ledger is not None:
            ledger.add("qr", _qr_flops(r * i_ * j_, s), (r * i_ * j_, s))
        cores[k] = q.reshape(r, i_, j_, q.shape[1], order="F")
        nxt = np.tensordot(rm, cores[k + 1], axes=(1, 0))
        if ledger is not None:
            ledger.add("gemm", 2.0 * nxt.size * rm.shape[1], nxt.shape)
        cores[k + 1] = nxt


def _r2l(cores, round_tol, ledger, ranks_out=None):
    """rsvd.py:111-136: optional L2R pass + per-bond truncated SVD
    (delta = tol*||last||/sqrt(d-1)) or exact RQ, carry absorbed leftward."""
    d = len(cores)
    if d == 1:
        return
    delta = 0.0
    if round_tol is not None:
        _l2r(cores, ledger)
        delta = round_tol * np.linalg.norm(cores[-1]) / math.sqrt(d - 1)
    for k in range(d - 1, 0, -1):
        r, i_, j_, s = cores[k].shape
        m = cores[k].reshape(r, i_ * j_ * s, order="F")
        if round_tol is not None:
            u, sv, vh = np.linalg.svd(m, full_matrices=False)
            if ledger is not None:
                ledger.add("svd", _svd_flops(*m.shape), m.shape)
            rr = truncation_rank(sv, delta, round_tol)
            head, carry = vh[:rr], u[:, :rr] * sv[:rr]
        else:
            qt, rt = np.linalg.qr(m.T)
            if ledger is not None:
                ledger.add("qr", _qr_flops(*m.shape), m.shape)
            head, carry = qt.T, rt.T
            rr = head.shape[0]
        cores[k] = head.reshape(rr, i_, j_, s, order="F")
        prev = np.tensordot(cores[k - 1], carry, axes=(3, 0))
        if ledger is not None:
            ledger.add("gemm", 2.0 * prev.size * carry.shape[0], prev.shape)
        cores[k - 1] = prev


def mpo_qr(y, round_tol=None, ledger=None):
    """Algorithm 3 with fused rounding (rsvd.py:139-166)."""
    _, i1, kk, _ = y[0].shape
    if i1 < kk:
        raise ValueError(f"first core has I1 = {i1} < K = {kk}")
    cores = [c.copy() for c in y]
    _r2l(cores, round_tol, ledger)
    _, i1, kk, r2 = cores[0].shape
    b = (cores[0].reshape(i1, kk, r2, order="F").transpose(1, 0, 2)
         .reshape(kk, i1 * r2, order="F"))
    qt, rt = np.linalg.qr(b.T)
    if ledger is not None:
        ledger.add("qr", _qr_flops(i1 * r2, kk), (i1 * r2, kk))
    cores[0] = (qt.T.reshape(kk, i1, r2, order="F").transpose(1, 0, 2)
                .reshape(1, i1, kk, r2, order="F"))
    return cores, rt


def mpo_svd(b, round_tol=None, ledger=None):
    """Algorithm 4 (rsvd.py:169-193): returns W, s and the tall V cores."""
    _, kk, j1, _ = b[0].shape
    if j1 < kk:
        raise ValueError(f"first core has J1 = {j1} < K = {kk}")
    cores = [c.copy() for c in b]
    _r2l(cores, round_tol, ledger)
    _, kk, j1, r2 = cores[0].shape
    m = cores[0].reshape(kk, j1 * r2, order="F")
    w, s, q1h = np.linalg.svd(m, full_matrices=False)
    if ledger is not None:
        ledger.add("svd", _svd_flops(*m.shape), m.shape)
    cores[0] = q1h.reshape(1, kk, j1, r2, order="F")
    return w, s, transpose_cores(cores)


def subspace_iteration(a, o, q=2, round_tol=1e-9, ledger=None):
    """Algorithm 5 (rsvd.py:196-214)."""
    if q < 0:
        raise ValueError("q must be >= 0")
    qm, _ = mpo_qr(mpo_matmul(a, o, ledger), round_tol, ledger)
    at = transpose_cores(a)
    for _ in range(q):
        qm, _ = mpo_qr(mpo_matmul(at, qm, ledger), round_tol, ledger)
        qm, _ = mpo_qr(mpo_matmul(a, qm, ledger), round_tol, ledger)
    return qm


def sketch_width(k_target, oversample):
    """rsvd.py:235: K = max(k, ceil(oversample*k))."""
    return max(int(k_target), int(np.ceil(oversample * k_target)))


def merge_count(row_dims, col_dims, kk):
    """rsvd.py:236-243: first core count whose cumulative row and column
    extents both reach K."""
    rc = np.cumprod(row_dims)
    cc = np.cumprod(col_dims)
    ok = np.nonzero((rc >= kk) & (cc >= kk))[0]
    if ok.size == 0:
        raise ValueError(f"matrix cannot host a width-{kk} sketch")
    return int(ok[0]) + 1


@dataclass
class OracleSvd:
    u: list
    s: np.ndarray
    v: list
    k_target: int
    k_oversampled: int


def tnrsvd(a, k_target, q=2, round_tol=1e-9, oversample=2.0, seed=None,
           ledger=None):
    """Algorithm 2 driver (rsvd.py:217-259)."""
    if k_target < 1:
        raise ValueError("k_target must be >= 1")
    kk = sketch_width(k_target, oversample)
    cnt = merge_count([c.shape[1] for c in a], [c.shape[2] for c in a], kk)
    am = merge_leading(a, cnt, ledger)
    o = random_unit_rank_mpo([c.shape[2] for c in am], kk, seed)
    qm = subspace_iteration(am, o, q, round_tol, ledger)
    b = mpo_matmul(transpose_cores(qm), am, ledger)
    w, s, v = mpo_svd(b, round_tol, ledger)
    u = [c.copy() for c in qm]
    u[0] = np.einsum("xikr,kl->xilr", u[0], w)
    v = [c.copy() for c in v]
    for col in range(k_target):
        nz = np.nonzero(w[:, col])[0]
        if nz.size and w[nz[0], col] < 0:
            u[0][:, :, col, :] *= -1.0
            v[0][:, :, col, :] *= -1.0
    u[0] = np.ascontiguousarray(u[0][:, :, :k_target, :])
    v[0] = np.ascontiguousarray(v[0][:, :, :k_target, :])
    return OracleSvd(u, s[:k_target].copy(), v, k_target, kk)


def lowrank_residual(a, u, s, v):
    """||A.V - U.diag(s)||_F / ||U.diag(s)||_F in MPO form (no densify):
    the difference MPO is built by stacking and its norm taken by a QR sweep."""
    av = mpo_matmul(a, v)
    us = [c.copy() for c in u]
    us[0] = us[0] * s[None, None, :, None]
    diff = mpo_add(av, scale_first(us, -1.0))
    return mpo_frobenius(diff) / mpo_frobenius(us)


def lowrank_difference(u1, s1, v1, u2, s2, v2):
    """||U1 S1 V1^T - U2 S2 V2^T||_F / ||U2 S2 V2^T||_F in MPO form."""
    def usv(u, s, v):
        us = [c.copy() for c in u]
        us[0] = us[0] * s[None, None, :, None]
        return mpo_matmul(us, transpose_cores(v))
    x = usv(u1, s1, v1)
    y = usv(u2, s2, v2)
    return mpo_frobenius(mpo_add(x, scale_first(y, -1.0))) / mpo_frobenius(y)


# ---------------------------------------------------------------------------
# sparse -> MPO conversion structure (sparse.py)
# ---------------------------------------------------------------------------


@dataclass
class ConversionStructure:
    i1: np.ndarray      # per kept nonzero, row offset inside its block
    j1: np.ndarray      # per kept nonzero, col offset inside its block
    ti: np.ndarray      # per kept nonzero, block id in [0, rank)
    values: np.ndarray  # kept values, masked input order
    uniq: np.ndarray    # sorted unique block keys br + nrb*bc
    rank: int


def digits(idx, extents):
    """Level digits, level-2 fastest (sparse.py:173-180)."""
    out = []
    rest = np.asarray(idx, dtype=np.int64).copy()
    for n in extents:
        out.append(rest % n)
        rest //= n
    return out


def conversion_structure(row1, col1, val, row_factors, col_factors):
    """sparse.py:234-250 on 1-based COO input: drop explicit zeros, split
    each coordinate into (in-block offset, block coordinate), key blocks
    column-block-major, unique with inverse."""
    row1 = np.asarray(row1, dtype=np.int64)
    col1 = np.asarray(col1, dtype=np.int64)
    val = np.asarray(val, dtype=np.float64)
    keep = val != 0
    r0 = row1[keep] - 1
    c0 = col1[keep] - 1
    i1_, j1_ = int(row_factors[0]), int(col_factors[0])
    nrb = math.prod(int(f) for f in row_factors[1:])
    br, bc = r0 // i1_, c0 // j1_
    key = br + nrb * bc
    uniq, ti = np.unique(key, return_inverse=True)
    return ConversionStructure(r0 % i1_, c0 % j1_, ti.astype(np.int64),
                               val[keep], uniq.astype(np.int64), int(uniq.size))


def coo_validate(rows, cols, row1, col1, val):
    """SparseMatrixCoo.__init__ checks (sparse.py:53-70): lengths, 1-based
    ranges and the duplicate-coordinate rejection (np.unique of the keys).
    CPU-baseline port of the constructor bench.py times separately."""
    row1 = np.asarray(row1, dtype=np.int64).reshape(-1)
    col1 = np.asarray(col1, dtype=np.int64).reshape(-1)
    val = np.asarray(val, dtype=np.float64).reshape(-1)
    if not (row1.size == col1.size == val.size):
        raise ValueError("row/col/val arrays must have equal length")
    if row1.size:
        if row1.min() < 1 or row1.max() > rows:
            raise ValueError("row index out of range")
        if col1.min() < 1 or col1.max() > cols:
            raise ValueError("col index out of range")
        keys = (row1 - 1) * cols + (col1 - 1)
        if np.unique(keys).size != keys.size:
            raise ValueError("duplicate (row, col) entries rejected")
    return row1, col1, val


def matrix_to_mpo_arrays(row1, col1, val, row_factors, col_factors):
    """The whole uncapped matrix_to_mpo with sparse cores
    (sparse.py:207-258 + _build_cores :183-204), as parallel index arrays
    per core (left, row, col, right, values): the same numpy work the
    reference does, including its per-nonzero level digits (:243-244), whose
    results it never uses.  CPU-baseline port (bench.py)."""
    keep = val != 0
    r0 = row1[keep] - 1
    c0 = col1[keep] - 1
    values = val[keep]
    i1_, j1_ = int(row_factors[0]), int(col_factors[0])
    i1, br = r0 % i1_, r0 // i1_
    j1, bc = c0 % j1_, c0 // j1_
    digits(br, row_factors[1:])          # sparse.py:243-244 (dead in the reference too)
    digits(bc, col_factors[1:])
    nrb = math.prod(int(f) for f in row_factors[1:])
    key = br + nrb * bc
    uniq, ti = np.unique(key, return_inverse=True)
    rank = uniq.size
    u_row = digits(uniq % nrb, row_factors[1:])
    u_col = digits(uniq // nrb, col_factors[1:])
    d = len(row_factors)
    cores = [(np.zeros_like(ti), i1, j1, ti, values)]
    t = np.arange(rank, dtype=np.int64)
    ones = np.ones(rank)
    for k in range(1, d):
        cores.append((t, u_row[k - 1], u_col[k - 1], t if k < d - 1 else np.zeros_like(t), ones))
    return cores


def block_digits(uniq, row_factors, col_factors):
    """u_row / u_col of sparse.py:249-250."""
    nrb = math.prod(int(f) for f in row_factors[1:])
    return (digits(uniq % nrb, row_factors[1:]),
            digits(uniq // nrb, col_factors[1:]))


def conversion_dense_cores(st: ConversionStructure, row_factors, col_factors):
    """Dense cores of sparse.py:183-204 (desk scale only)."""
    d = len(row_factors)
    rank = st.rank
    c0 = np.zeros((1, row_factors[0], col_factors[0], rank))
    np.add.at(c0, (np.zeros_like(st.ti), st.i1, st.j1, st.ti), st.values)
    cores = [c0]
    ur, uc = block_digits(st.uniq, row_factors, col_factors)
    t = np.arange(rank)
    for k in range(1, d):
        s = rank if k < d - 1 else 1
        c = np.zeros((rank, row_factors[k], col_factors[k], s))
        c[t, ur[k - 1], uc[k - 1], t if k < d - 1 else 0] = 1.0
        cores.append(c)
    return cores


# ---------------------------------------------------------------------------
# CPU baseline timing helper (bench.py:148-155 convention)
# ---------------------------------------------------------------------------


def timed(fn, repeats=3):
    times, res = [], None
    for _ in range(repeats):
        t0 = time.perf_counter()
        res = fn()
        times.append(time.perf_counter() - t0)
    times.sort()
    return res, times[len(times) // 2]


def gram_first_index(x, y):
    """X^T Y (K x K) for two tall MPOs whose first cores carry the K column
    index (shape (1, I1, K, R)); contracted by transfer matrices, never
    densified."""
    t = None
    for k in range(len(x) - 1, 0, -1):
        cx, cy = x[k], y[k]            # (Rx, I, Kx=1.., Sx), (Ry, I, .., Sy)
        cx2 = cx.reshape(cx.shape[0], -1, cx.shape[3], order="F")
        cy2 = cy.reshape(cy.shape[0], -1, cy.shape[3], order="F")
        if t is None:
            t = np.tensordot(cx2, cy2, axes=([1, 2], [1, 2]))
        else:
            t = np.tensordot(np.tensordot(cx2, t, axes=(2, 0)), cy2, axes=([1, 2], [1, 2]))
    c0x, c0y = x[0][0], y[0][0]        # (I1, K, R)
    if t is not None:
        c0x = np.tensordot(c0x, t, axes=(2, 0))      # (I1, Kx, Sy)
    return np.tensordot(c0x, c0y, axes=([0, 2], [0, 2]))


def aligned_factor_error(x, y):
    """max over columns of ||x_k - sign_k y_k|| for two tall MPOs with
    orthonormal columns, sign_k from x^T y; computed via the Gram matrices
    of the stacked difference (no cancellation beyond ~1e-8 absolute, so
    use the explicit difference MPO for tight bounds)."""
    p = gram_first_index(x, y)
    sg = np.where(np.diag(p) < 0, -1.0, 1.0)
    ys = [c.copy() for c in y]
    ys[0] = ys[0] * sg[None, None, :, None]
    diff = mpo_add(x, scale_first(ys, -1.0))
    return mpo_frobenius(diff), sg

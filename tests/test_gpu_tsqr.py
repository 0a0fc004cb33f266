"""Row-sharded TSQR / SVD (paper_1707_07803_b200/tsqr.py) with the device
primitives (C-ABI mpo_dense_qr / mpo_dense_svd / mpo_dense_gemm): the
P-rank exchange emulated in lock step on one GPU, and the one-rank path,
against numpy/LAPACK (rsvd.py:106, :128)."""

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


def _ops():
    from paper_1707_07803_b200.tsqr import DenseDeviceOps
    return DenseDeviceOps(0)


@pytest.mark.parametrize("world,m,n", [(2, 700, 64), (4, 4096, 256), (8, 65536, 512)])
def test_tsqr_emulated_device(world, m, n):
    from paper_1707_07803_b200.tsqr import tsqr_emulated, tsqr_svd_emulated
    rng = np.random.default_rng(m + n)
    a = rng.standard_normal((m, n))
    a[:, 3] = a[:, 1]            # rank deficient
    b = np.linspace(0, m, world + 1).astype(int)
    shards = [torch.from_numpy(a[b[i]:b[i + 1]]).cuda() for i in range(world)]
    ops = _ops()
    res = tsqr_emulated(shards, ops)
    qm = np.concatenate([x[0].cpu().numpy() for x in res])
    r = res[0][1].cpu().numpy()
    assert np.linalg.norm(qm.T @ qm - np.eye(n)) <= 1e-13 * n
    assert np.linalg.norm(qm @ r - a) <= 1e-13 * np.linalg.norm(a)
    assert np.abs(np.tril(r, -1)).max() == 0.0
    sa = np.linalg.svd(a, compute_uv=False)
    us, s, vt = tsqr_svd_emulated(shards, ops)
    s = s.cpu().numpy()
    np.testing.assert_allclose(s, sa, rtol=0, atol=1e-13 * sa[0])
    um = np.concatenate([u.cpu().numpy() for u in us])
    assert np.linalg.norm(um.T @ um - np.eye(n)) <= 1e-12 * n
    assert np.linalg.norm((um * s) @ vt.cpu().numpy() - a) <= 1e-13 * np.linalg.norm(a)


def test_tsqr_single_rank_and_dense_ops():
    from paper_1707_07803_b200.tsqr import tsqr, tsqr_svd
    rng = np.random.default_rng(2)
    a = rng.standard_normal((3000, 200))
    q, r = tsqr(torch.from_numpy(a).cuda(), _ops())
    q, r = q.cpu().numpy(), r.cpu().numpy()
    assert np.linalg.norm(q @ r - a) <= 1e-13 * np.linalg.norm(a)
    rl = np.linalg.qr(a, mode="r")
    np.testing.assert_allclose(np.abs(r), np.abs(rl), atol=1e-11 * np.abs(rl).max())
    u, s, vt = tsqr_svd(torch.from_numpy(a).cuda(), _ops())
    np.testing.assert_allclose(s.cpu().numpy(), np.linalg.svd(a, compute_uv=False), rtol=1e-12)
    x, y = rng.standard_normal((300, 70)), rng.standard_normal((70, 90))
    c = _ops().matmul(torch.from_numpy(x).cuda(), torch.from_numpy(y).cuda()).cpu().numpy()
    np.testing.assert_allclose(c, x @ y, rtol=0, atol=1e-12 * np.abs(x @ y).max())


def test_dense_svd_tall_and_square():
    """mpo_dense_svd: square (one-sided Jacobi, U from Ucarry / s) and tall
    (QR first, U = Q U_R) against LAPACK, incl. a rank-deficient tall case."""
    rng = np.random.default_rng(4)
    ops = _ops()
    for m, n in ((300, 300), (3000, 200), (1000, 64)):
        a = rng.standard_normal((m, n))
        if m == 1000:
            a[:, 10] = a[:, 2]
        u, s, vt = ops.svd(torch.from_numpy(a).cuda())
        u, s, vt = u.cpu().numpy(), s.cpu().numpy(), vt.cpu().numpy()
        sl = np.linalg.svd(a, compute_uv=False)
        np.testing.assert_allclose(s, sl, rtol=0, atol=1e-13 * sl[0])
        assert np.linalg.norm(u.T @ u - np.eye(n)) <= 1e-12 * n
        assert np.linalg.norm(vt @ vt.T - np.eye(n)) <= 1e-12 * n
        assert np.linalg.norm((u * s) @ vt - a) <= 1e-13 * np.linalg.norm(a)

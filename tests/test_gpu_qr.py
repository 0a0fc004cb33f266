"""The blocked Householder QR (qr.cu: cluster panels, compact-WY trailing
updates) through the C-ABI mpo_qr on a
one-core MPO, i.e. np.linalg.qr(mode="reduced") of an m x n matrix
(rsvd.py:158-163): Q orthonormal, Q R = A, R upper triangular and equal to
LAPACK's up to row signs -- also for rank-deficient and graded columns."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _qr(a):
    import paper_1707_07803_b200 as m
    mm, nn = a.shape
    q, r = m.mpo_qr(m.Mpo([a.reshape(1, mm, nn, 1)]))
    return q.cores[0].reshape(mm, nn), np.asarray(r)


@pytest.mark.parametrize("shape", [(700, 96), (2048, 512), (8192, 256), (3000, 300), (520, 520),
                                   (70000, 128), (40001, 1024)])
def test_qr_random(shape):
    a = np.random.default_rng(sum(shape)).standard_normal(shape)
    q, r = _qr(a)
    n = shape[1]
    assert np.linalg.norm(q.T @ q - np.eye(n)) <= 1e-13 * np.sqrt(n)
    assert np.linalg.norm(q @ r - a) <= 1e-13 * np.linalg.norm(a)
    assert np.abs(np.tril(r, -1)).max() == 0.0
    rl = np.linalg.qr(a, mode="r")
    np.testing.assert_allclose(np.abs(r), np.abs(rl), atol=1e-11 * np.abs(rl).max())


@pytest.mark.parametrize("shape", [(257, 257), (1000, 999), (1025, 33), (2047, 129), (4097, 511),
                                   (8300, 64), (12000, 700), (16385, 130), (20000, 300)])
def test_qr_odd_shapes(shape):
    """Shapes off every blocking boundary: partial 32-column panels, partial
    128-column outer blocks, CTA slices of more than 512 rows (the multi-pass
    panel paths), panels on either side of the 16384-row limit of the
    clustered reflector application, narrow (16 / 8 column) cluster panels."""
    a = np.random.default_rng(sum(shape)).standard_normal(shape)
    q, r = _qr(a)
    n = shape[1]
    assert np.linalg.norm(q.T @ q - np.eye(n)) <= 1e-13 * np.sqrt(n)
    assert np.linalg.norm(q @ r - a) <= 1e-13 * np.linalg.norm(a)
    assert np.abs(np.tril(r, -1)).max() == 0.0


def test_qr_rank_deficient_and_graded():
    rng = np.random.default_rng(3)
    a = rng.standard_normal((1500, 200))
    a[:, 7] = a[:, 3] * 2.0            # exactly dependent column
    a[:, 50] = 0.0                     # zero column
    a[:, 100:] *= 1e-9                 # graded block
    q, r = _qr(a)
    assert np.linalg.norm(q.T @ q - np.eye(200)) <= 1e-13 * np.sqrt(200)
    assert np.linalg.norm(q @ r - a) <= 1e-13 * np.linalg.norm(a)


def test_qr_tall_rank_deficient():
    """Very tall (row-block TSQR path) with dependent, zero and graded columns."""
    rng = np.random.default_rng(9)
    a = rng.standard_normal((50000, 96))
    a[:, 7] = a[:, 3] * 2.0
    a[:, 50] = 0.0
    a[:, 60:] *= 1e-9
    q, r = _qr(a)
    assert np.linalg.norm(q.T @ q - np.eye(96)) <= 1e-13 * np.sqrt(96)
    assert np.linalg.norm(q @ r - a) <= 1e-13 * np.linalg.norm(a)
    assert np.abs(np.tril(r, -1)).max() == 0.0

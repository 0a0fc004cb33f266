"""Row-sharded TSQR / SVD of one tall unfolding (paper_1707_07803_b200/tsqr.py,
SURVEY.md 8(f).4) with world size 2 and 3 over gloo on CPU.  The per-rank
dense primitives are replaced by torch CPU stand-ins (test infrastructure);
the exchange and the assembly of Q / U are the product code.  Checked
against numpy/LAPACK on the gathered matrix (rsvd.py:106, :128)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


class CpuDenseOps:
    """torch CPU stand-ins for tsqr.DenseDeviceOps (test infrastructure)."""

    def qr(self, a):
        return torch.linalg.qr(a.to(torch.float64), mode="reduced")

    def svd(self, a):
        u, s, vt = torch.linalg.svd(a, full_matrices=False)
        return u, s, vt

    def matmul(self, a, b):
        return a @ b

    def cat(self, parts):
        return torch.cat(list(parts), 0)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _matrix(world):
    rng = np.random.default_rng(7)
    a = rng.standard_normal((90 * world + 13, 24))
    a[:, 5] = a[:, 2] * 3.0          # rank deficient
    a[:, 20:] *= 1e-7                # graded
    return a


def _rows(n, world, rank):
    b = np.linspace(0, n, world + 1).astype(int)
    return b[rank], b[rank + 1]


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1707_07803_b200.tsqr import tsqr, tsqr_svd
        a = _matrix(world)
        lo, hi = _rows(a.shape[0], world, rank)
        ql, r = tsqr(torch.from_numpy(a[lo:hi]), CpuDenseOps())
        ul, s, vt = tsqr_svd(torch.from_numpy(a[lo:hi]), CpuDenseOps())
        q.put((rank, ql.numpy(), r.numpy(), ul.numpy(), s.numpy(), vt.numpy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_tsqr_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = sorted([q.get(timeout=180) for _ in range(world)], key=lambda x: x[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    a = _matrix(world)
    n = a.shape[1]
    qm = np.concatenate([o[1] for o in out])
    r = out[0][2]
    assert all(np.array_equal(o[2], r) for o in out)          # R identical on every rank
    assert np.linalg.norm(qm.T @ qm - np.eye(n)) <= 1e-13 * n
    assert np.linalg.norm(qm @ r - a) <= 1e-13 * np.linalg.norm(a)
    assert np.abs(np.tril(r, -1)).max() == 0.0
    # R is unique only up to the arbitrary direction the dependent column
    # leaves; its singular values are A's
    np.testing.assert_allclose(np.linalg.svd(r, compute_uv=False),
                               np.linalg.svd(a, compute_uv=False), rtol=0,
                               atol=1e-13 * np.linalg.norm(a, 2))
    um = np.concatenate([o[3] for o in out])
    s, vt = out[0][4], out[0][5]
    sl = np.linalg.svd(a, compute_uv=False)
    np.testing.assert_allclose(s, sl, rtol=0, atol=1e-13 * sl[0])
    assert np.linalg.norm(um.T @ um - np.eye(n)) <= 1e-12 * n
    assert np.linalg.norm((um * s) @ vt - a) <= 1e-13 * np.linalg.norm(a)


@pytest.mark.parametrize("world", [2, 4, 8])
def test_tsqr_emulated(world):
    from paper_1707_07803_b200.tsqr import tsqr_emulated, tsqr_svd_emulated
    a = _matrix(world)
    shards = [torch.from_numpy(a[slice(*_rows(a.shape[0], world, r))]) for r in range(world)]
    res = tsqr_emulated(shards, CpuDenseOps())
    qm = np.concatenate([x[0].numpy() for x in res])
    r = res[0][1].numpy()
    assert np.linalg.norm(qm @ r - a) <= 1e-13 * np.linalg.norm(a)
    assert np.linalg.norm(qm.T @ qm - np.eye(a.shape[1])) <= 1e-13 * a.shape[1]
    us, s, vt = tsqr_svd_emulated(shards, CpuDenseOps())
    um = np.concatenate([u.numpy() for u in us])
    assert np.linalg.norm((um * s.numpy()) @ vt.numpy() - a) <= 1e-13 * np.linalg.norm(a)


def test_tsqr_shard_too_short():
    from paper_1707_07803_b200.tsqr import tsqr_emulated
    a = np.random.default_rng(1).standard_normal((40, 24))
    with pytest.raises(ValueError, match="at least n = 24 rows"):
        tsqr_emulated([torch.from_numpy(a[:30]), torch.from_numpy(a[30:])], CpuDenseOps())

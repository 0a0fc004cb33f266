"""Multi-GPU factorisation of ONE tall unfolding whose rows are sharded over
the ranks: communication-avoiding TSQR and the SVD built
on it.  These replace, for a single instance too large or too slow for one
GPU, the per-core factorisations of the sweeps -- np.linalg.qr at
/root/reference/pkg/src/mposvd/rsvd.py:106 (L2R sweep, tall unfolding
(R*I*J x S)) and np.linalg.svd at rsvd.py:128 (R2L truncation, whose
unfolding is tall after the transpose) -- with the same results up to the
column-sign gauge of Q / U (R's diagonal and the singular values are
unique).

Per rank r, holding rows A_r (m_r x n, m_r >= n) of A = [A_0; ...; A_{P-1}]:

1. local Householder QR  A_r = Q_r R_r            (mpo_dense_qr, qr.cu)
2. all-gather of the n x n factors R_r -> S = [R_0; ...; R_{P-1}]   (NCCL)
3. QR of S on every rank  S = Q_S R               (same inputs, same device
   code: every rank holds the same R bit for bit)
4. Q's rows  Q_r Q_S[r n : (r + 1) n, :]           (mpo_dense_gemm, DMMA)

One collective of P n^2 doubles per factorisation, all flops local.
tsqr_svd continues with the n x n SVD of R (replicated): A = (Q U_R) s V^T.

The algorithm is written once per rank over injected primitives (``ops``)
and one collective request: ``DenseDeviceOps`` runs the C-ABI kernels on
torch CUDA tensors; ``tsqr`` services the all-gather with torch.distributed
(NCCL on the GPU box, gloo in the CPU tests) and ``tsqr_emulated`` runs the
P shards in lock step in one process (the single-GPU test of the exchange).
"""

from __future__ import annotations

from . import _lib

__all__ = ["DenseDeviceOps", "tsqr", "tsqr_svd", "tsqr_emulated", "tsqr_svd_emulated"]


class DenseDeviceOps:
    """Local dense primitives on torch CUDA tensors through the C-ABI.
    Matrices are torch tensors of shape (m, n) in row-major torch layout;
    the C-ABI is column-major, so each call works on the transposed view
    (a row-major (m, n) tensor's storage is a column-major (n, m) matrix)."""

    def __init__(self, device=None):
        import torch
        self.torch = torch
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None
                                   else int(device))
        self.ctx = _lib.context(self.device.index)

    def _f(self, a):
        """column-major copy of a (m, n): a (n, m) row-major tensor"""
        return a.t().contiguous()

    def qr(self, a):
        torch = self.torch
        m, n = a.shape
        af = self._f(a.to(self.device, torch.float64))
        qf = torch.empty((n, m), dtype=torch.float64, device=self.device)
        rf = torch.empty((n, n), dtype=torch.float64, device=self.device)
        _lib.call("mpo_dense_qr", self.ctx, m, n, af.data_ptr(), m, qf.data_ptr(), m,
                  rf.data_ptr(), n)
        return qf.t(), rf.t()

    def svd(self, a):
        torch = self.torch
        m, n = a.shape
        af = self._f(a.to(self.device, torch.float64))
        s = torch.empty(n, dtype=torch.float64, device=self.device)
        uf = torch.empty((n, m), dtype=torch.float64, device=self.device)
        vtf = torch.empty((n, n), dtype=torch.float64, device=self.device)
        _lib.call("mpo_dense_svd", self.ctx, m, n, af.data_ptr(), m, s.data_ptr(),
                  uf.data_ptr(), m, vtf.data_ptr(), n)
        return uf.t(), s, vtf.t()

    def matmul(self, a, b):
        """a (m, k) @ b (k, n) on the DMMA GEMM: in column-major terms
        C^T (n x m) = B^T A^T, i.e. the row-major operands as they lie"""
        torch = self.torch
        m, k = a.shape
        n = b.shape[1]
        ac, bc = a.contiguous(), b.contiguous()
        c = torch.empty((m, n), dtype=torch.float64, device=self.device)
        _lib.call("mpo_dense_gemm", self.ctx, 0, 0, n, m, k, 1.0, bc.data_ptr(), n,
                  ac.data_ptr(), k, 0.0, c.data_ptr(), n)
        return c

    def cat(self, parts):
        return self.torch.cat(list(parts), 0)


def _rank_steps(a, ops, world, me):
    """One rank's TSQR; yields its collective request, returns (Q_r, R)."""
    m, n = a.shape
    if m < n:
        raise ValueError(f"tsqr: every shard needs at least n = {n} rows (rank {me} has {m})")
    q_loc, r_loc = ops.qr(a)
    rs = yield ("all_gather", r_loc)
    q_s, r = ops.qr(ops.cat(rs))
    return ops.matmul(q_loc, q_s[me * n:(me + 1) * n]), r


def _serve(gen, group):
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group)
    res = None
    while True:
        try:
            req = gen.send(res)
        except StopIteration as fin:
            return fin.value
        t = req[1].contiguous()
        out = [torch.empty_like(t) for _ in range(world)]
        dist.all_gather(out, t, group=group)
        res = out


def tsqr(a_local, ops=None, group=None):
    """Reduced QR of the row-sharded A: returns (this rank's rows of Q, R).
    Without an initialised process group it is the single-GPU QR."""
    import torch.distributed as dist
    ops = ops or DenseDeviceOps()
    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return ops.qr(a_local)
    return _serve(_rank_steps(a_local, ops, dist.get_world_size(group), dist.get_rank(group)),
                  group)


def tsqr_svd(a_local, ops=None, group=None):
    """Thin SVD of the row-sharded A = U diag(s) V^T: returns (this rank's
    rows of U, s, V^T); s and V^T are the same on every rank."""
    ops = ops or DenseDeviceOps()
    q, r = tsqr(a_local, ops, group)
    u_r, s, vt = ops.svd(r)
    return ops.matmul(q, u_r), s, vt


def tsqr_emulated(shards, ops):
    """All ranks' TSQR in lock step in one process (the collective is a
    list): the single-device test of the exchange."""
    gens = [_rank_steps(a, ops, len(shards), i) for i, a in enumerate(shards)]
    reqs = [g.send(None) for g in gens]
    gathered = [r[1] for r in reqs]
    out = []
    for g in gens:
        try:
            g.send(gathered)
        except StopIteration as fin:
            out.append(fin.value)
    return out


def tsqr_svd_emulated(shards, ops):
    res = tsqr_emulated(shards, ops)
    u_r, s, vt = ops.svd(res[0][1])
    return [ops.matmul(q, u_r) for q, _ in res], s, vt

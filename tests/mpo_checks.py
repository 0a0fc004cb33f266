"""MPO-form accuracy checks of a TNrSVD result -- TEST INFRASTRUCTURE ONLY.

Used by ``tests/golden/make_golden.py`` (on the reference's outputs, torch on
the CPU) and by the ``-m gpu`` parity tests (on the device path's outputs,
torch on the GPU as a plain FP64 contraction engine), so both sides evaluate
the same formulas.  Nothing here is densified: every quantity is a chain of
transfer-matrix contractions from the right end (where the column index K is
absent), so memory is bounded by the bond ranks, never by 2^20 rows.

Operands: ``a`` is the MERGED operator (the cores TNrSVD actually multiplies,
rsvd.py:243), ``u`` / ``v`` the tall factors of ``LowRankSvd`` (first core
(1, I1, k, R), later cores (R, n, 1, S)), ``s`` the singular values.

* ``uav(u, a, v)``      U^T A V                   (k x k; = diag(s) up to rounding)
* ``quad(x, a, t)``     X^T A^T A X (t=False) or X^T A A^T X (t=True)   (k x k)
* ``residuals``         ||A V - U S||_F / ||U S||_F   (BASELINE.json config 2's
                        "MPO-form residual ... contracted in TT format") and the
                        transposed ||A^T U - V S||_F / ||V S||_F, in Gram form:
                        ||AV - US||^2 = tr(V^T A^T A V) - 2 sum_i s_i (U^T A V)_ii + sum s_i^2
* ``probe(x, p)``       X^T P for a unit-rank probe MPO P (k x m)
"""

from __future__ import annotations

import math

import numpy as np


def _torch():
    import torch
    return torch


def _t(c, dev):
    torch = _torch()
    return torch.as_tensor(np.ascontiguousarray(np.asarray(c)), dtype=torch.float64, device=dev)


def _cores(m, dev):
    cores = m.cores if hasattr(m, "cores") else m
    return [_t(c, dev) for c in cores]


def uav(u, a, v, dev="cpu"):
    """U^T A V (k_u x k_v), contracted right to left with the 3-layer
    environment E[u, a, v] (bond ranks rU x rA x rV)."""
    torch = _torch()
    U, A, V = _cores(u, dev), _cores(a, dev), _cores(v, dev)
    d = len(U)
    assert len(A) == d and len(V) == d, "A must be the merged operator (same core count as U, V)"
    E = torch.ones((1, 1, 1), dtype=torch.float64, device=dev)
    for j in range(d - 1, 0, -1):
        Uj, Vj, Aj = U[j][:, :, 0, :], V[j][:, :, 0, :], A[j]
        X = torch.einsum("vjw,uaw->vjua", Vj, E)
        Y = torch.einsum("vjua,bija->vubi", X, Aj)
        E = torch.einsum("uix,vxbi->ubv", Uj, Y)
        del X, Y
    U0, A0, V0 = U[0][0], A[0][0], V[0][0]          # (I1,k,u) (I1,J1,a) (J1,k,v)
    X = torch.einsum("jkv,uav->jkua", V0, E)
    Y = torch.einsum("jlua,ija->ilu", X, A0)
    return torch.einsum("iku,ilu->kl", U0, Y).cpu().numpy()


def quad(x, a, transpose=False, dev="cpu"):
    """X^T M^T M X with M = A (X is V: contracted with A's column index) or
    M = A^T (transpose=True, X is U).  Environment E[x, a, y, b] (rX^2 rA^2
    doubles), updated one right bond index b at a time to bound temporaries."""
    torch = _torch()
    X, A = _cores(x, dev), _cores(a, dev)
    if transpose:
        A = [c.permute(0, 2, 1, 3) for c in A]   # M = A^T: (a, out=j, in=i, a')
    d = len(X)
    E = torch.ones((1, 1, 1, 1), dtype=torch.float64, device=dev)
    for j in range(d - 1, 0, -1):
        Xj, Mj = X[j][:, :, 0, :], A[j]           # (x, in, x'), (a, out, in, a')
        rx, ra = Xj.shape[0], Mj.shape[0]
        En = torch.zeros((rx, ra, rx, ra), dtype=torch.float64, device=dev)
        for b2 in range(Mj.shape[3]):
            Eb = E[:, :, :, b2]                                   # (x2, a2, y2)
            P = torch.einsum("xjw,wav->xjav", Xj, Eb)             # (x, in, a2, y2)
            Q = torch.einsum("xjav,cija->xvci", P, Mj)            # (x, y2, a, out)
            del P
            T = torch.einsum("xvci,ykv->xciyk", Q, Xj)            # (x, a, out, y, in')
            del Q
            En += torch.einsum("xciyk,bik->xcyb", T, Mj[:, :, :, b2])
            del T
        E = En
    X0, M0 = X[0][0], A[0][0]                     # (in1, k, x), (out1, in1, a)
    Z = torch.einsum("jkx,xayb->jkayb", X0, E)
    W = torch.einsum("jkayb,ija->ikyb", Z, M0)
    del Z
    R = torch.einsum("imb,mly->ibly", M0, X0)
    return torch.einsum("ikyb,ibly->kl", W, R).cpu().numpy()


def residuals(u, s, v, a, dev="cpu", av=True, atu=True):
    """Gram-form relative residuals; returns dict with the k x k pieces."""
    s = np.asarray(s, dtype=np.float64)
    g2 = uav(u, a, v, dev)
    ns2 = float(np.sum(s * s))
    cross = float(np.sum(s * np.diag(g2)))
    out = {"uav": g2}
    if av:
        g1 = quad(v, a, False, dev)
        out["vaav"] = g1
        out["res_av"] = math.sqrt(max(np.trace(g1) - 2.0 * cross + ns2, 0.0) / ns2)
    if atu:
        g3 = quad(u, a, True, dev)
        out["uaau"] = g3
        out["res_atu"] = math.sqrt(max(np.trace(g3) - 2.0 * cross + ns2, 0.0) / ns2)
    return out


def probe_mpo(row_dims, m, seed):
    """Unit-rank probe with m columns: core 0 (1, I1, m, 1), cores (1, n, 1, 1)."""
    rng = np.random.default_rng(seed)
    cores = [rng.standard_normal((1, row_dims[0], m, 1))]
    cores += [rng.standard_normal((1, n, 1, 1)) for n in row_dims[1:]]
    return cores


def probe(x, p, dev="cpu"):
    """X^T P (k x m) for tall MPOs with the column index in core 0."""
    torch = _torch()
    X, P = _cores(x, dev), _cores(p, dev)
    E = torch.ones((1, 1), dtype=torch.float64, device=dev)
    for j in range(len(X) - 1, 0, -1):
        E = torch.einsum("xiw,piq,wq->xp", X[j][:, :, 0, :], P[j][:, :, 0, :], E)
    return torch.einsum("ikx,imp,xp->km", X[0][0], P[0][0], E).cpu().numpy()


def row_dims(x):
    cores = x.cores if hasattr(x, "cores") else x
    return [int(c.shape[1]) for c in cores]


def summary(u, s, v, a, dev="cpu", av=True, atu=True, probes=(101, 102)):
    """Every quantity the full-size parity tests compare."""
    out = residuals(u, s, v, a, dev, av=av, atu=atu)
    pu = probe_mpo(row_dims(u), 8, probes[0])
    pv = probe_mpo(row_dims(v), 8, probes[1])
    out["utp"] = probe(u, pu, dev)
    out["vtp"] = probe(v, pv, dev)
    # P_u^T (U S V^T) P_v: invariant under the common per-triplet sign flip
    out["rec_probe"] = out["utp"].T @ (np.asarray(s)[:, None] * out["vtp"])
    return out


def sign_alignment(got, ref):
    """Per-triplet signs D with got ~ ref D from the probe products (U and V
    must agree: a triplet flips as a whole)."""
    du = np.sign(np.sum(got["utp"] * ref["utp"], axis=1))
    dv = np.sign(np.sum(got["vtp"] * ref["vtp"], axis=1))
    return du, dv

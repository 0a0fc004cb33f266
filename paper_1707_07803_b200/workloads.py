"""Seeded synthetic workloads of BASELINE.json's five configs.

No public dataset is involved: every input is generated on the host from
``numpy.random.default_rng(seed)`` with the shapes / value distributions the
configs name, identically for the device path, the oracle and the bench.
"""

from __future__ import annotations

import math

import numpy as np

from .mpo import Mpo, random_mpo
from .partition import PartitionPlan

__all__ = ["config_mpo", "TNRSVD_ARGS", "band_scatter_coo", "powerlaw_coo", "dedup_sum"]

# tnrsvd arguments per config (additive oversampling p -> multiplicative
# oversample = (k + p) / k, rsvd.py:235)
TNRSVD_ARGS = {
    "c1": dict(k_target=10, q=0, round_tol=1e-9, oversample=2.0, seed=2),
    "c2": dict(k_target=20, q=1, round_tol=1e-9, oversample=1.5, seed=2),
    "c3": dict(k_target=32, q=2, round_tol=1e-9, oversample=1.5, seed=4),
    "c3q0": dict(k_target=32, q=0, round_tol=1e-9, oversample=1.5, seed=4),
    "c5inst": dict(k_target=16, q=1, round_tol=1e-9, oversample=1.5, seed=51),
    "c5inst_q0": dict(k_target=16, q=0, round_tol=1e-9, oversample=1.5, seed=51),
}


def config_mpo(name: str, instance: int = 0) -> Mpo:
    """The operator A of a TNrSVD config (random_mpo draw order, mpo.py:436-449)."""
    if name == "c1":
        return random_mpo([2] * 10, [2] * 10, [3] * 9, seed=1)
    if name == "c2":
        a = random_mpo([2] * 20, [2] * 20, [8] * 19, seed=1)
        return Mpo([c / math.sqrt(8.0) for c in a.cores])
    if name in ("c3", "c3q0"):
        a = random_mpo([4] * 12, [4] * 12, [64] * 11, seed=3)
        cores = [c / 8.0 for c in a.cores]
        # geometric decay imposed on the middle bond (core 5's right rank)
        cores[5] = cores[5] * (0.5 ** np.arange(64))[None, None, None, :]
        return Mpo(cores)
    if name in ("c5inst", "c5inst_q0"):
        return random_mpo([2] * 20, [2] * 20, [16] * 19, seed=50 + instance)
    raise KeyError(name)


def dedup_sum(n_rows, r0, c0, v):
    """Merge duplicate 0-based coordinates by summation (the reference rejects
    duplicates, sparse.py:68-70); returns sorted-by-key 1-based COO."""
    key = r0.astype(np.int64) * np.int64(n_rows) + c0.astype(np.int64)
    uk, inv = np.unique(key, return_inverse=True)
    vs = np.zeros(uk.size)
    np.add.at(vs, inv, v)
    return uk // n_rows + 1, uk % n_rows + 1, vs


def band_scatter_coo(n: int, extra: int, seed: int):
    """Config 4: tridiagonal band + ``extra`` uniform scattered N(0,1)
    entries, duplicates summed.  Returns (row1, col1, val)."""
    rng = np.random.default_rng(seed)
    main = np.arange(n)
    r = np.concatenate([main, main[:-1], main[1:]])
    c = np.concatenate([main, main[1:], main[:-1]])
    v = rng.standard_normal(r.size)
    rr = rng.integers(0, n, extra)
    cc = rng.integers(0, n, extra)
    vv = rng.standard_normal(extra)
    return dedup_sum(n, np.concatenate([r, rr]), np.concatenate([c, cc]),
                     np.concatenate([v, vv]))


def powerlaw_coo(n: int, seed: int, alpha: float = 2.1):
    """Config 5: row degrees floor(Pareto(alpha, xmin=1)) capped at n,
    uniform columns, values U(-1, 1), duplicates summed.  The mean degree is
    ~7.9, i.e. ~33M nonzeros at n = 2^22 (SURVEY.md 8(d) calibration note)."""
    rng = np.random.default_rng(seed)
    deg = np.floor((1.0 - rng.random(n)) ** (-1.0 / (alpha - 1.0))).astype(np.int64)
    deg = np.minimum(deg, n)
    rows = np.repeat(np.arange(n, dtype=np.int64), deg)
    cols = rng.integers(0, n, rows.size)
    vals = rng.uniform(-1.0, 1.0, rows.size)
    return dedup_sum(n, rows, cols, vals)


def square_plan(log2n: int) -> PartitionPlan:
    return PartitionPlan((2,) * log2n, (2,) * log2n)

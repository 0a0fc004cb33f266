"""Randomised parity of the fused rank-bounded sweeps (csrc/sweep.cu) against
the oracle restatement of the reference (materialised products), on MPOs
whose product ranks exceed the bond extents -- rectangular row/col
factors, mixed mode sizes, q = 0..2, several tolerances.  Checks: every
output rank equal, singular values within 1e-8 relative, U S V^T within
1e-10 relative (MPO form), U and V orthonormal."""

import numpy as np
import pytest

from oracle import mposvd_oracle as orc

pytestmark = pytest.mark.gpu

CASES = [
    # row_dims, col_dims, ranks, k, q, tol, oversample, seed
    ([2, 3, 2, 2, 3, 2], [3, 2, 2, 3, 2, 2], [4, 5, 6, 5, 4], 6, 1, 1e-9, 2.0, 1),
    ([4, 2, 2, 2, 2, 2, 2], [2, 2, 4, 2, 2, 2, 2], [3, 6, 6, 6, 6, 3], 5, 2, 1e-9, 1.5, 2),
    ([2] * 9, [2] * 9, [6] * 8, 8, 1, 1e-6, 1.5, 3),
    ([3, 3, 3, 3, 3], [2, 4, 2, 4, 2], [5, 9, 9, 5], 7, 1, 1e-12, 2.0, 4),
    ([2] * 10, [2] * 10, [5] * 9, 10, 2, 1e-9, 1.3, 5),
    ([4, 4, 4, 4], [4, 4, 4, 4], [8, 16, 8], 12, 1, 1e-9, 1.5, 6),
]


def _ortho(cores):
    g = orc.gram_first_index(cores, cores)
    return np.linalg.norm(g - np.eye(g.shape[0]))


@pytest.mark.parametrize("case", CASES, ids=[f"c{i}" for i in range(len(CASES))])
def test_fused_sweeps_match_oracle(case):
    import paper_1707_07803_b200 as m
    rd, cd, rk, k, q, tol, os_, seed = case
    a = m.random_mpo(rd, cd, rk, seed=seed)
    lr = m.tnrsvd(a, k, q=q, round_tol=tol, oversample=os_, seed=seed + 100)
    ref = orc.tnrsvd([c.copy() for c in a.cores], k, q=q, round_tol=tol, oversample=os_,
                     seed=seed + 100)
    assert lr.u.ranks == orc.ranks_of(ref.u) and lr.v.ranks == orc.ranks_of(ref.v)
    np.testing.assert_allclose(lr.s, ref.s, rtol=1e-8)
    diff = orc.lowrank_difference(lr.u.cores, lr.s, lr.v.cores, ref.u, ref.s, ref.v)
    assert diff <= 1e-10
    assert _ortho(lr.u.cores) <= 1e-12 and _ortho(lr.v.cores) <= 1e-12

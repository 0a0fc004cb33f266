"""B200-native TNrSVD + sparse->MPO hot path of arXiv 1707.07803.

Drop-in for the reference package ``mposvd``'s hot-path API
(/root/reference/pkg/src/mposvd/__init__.py:13-50): same names, signatures,
defaults and errors; the arithmetic runs in hand-written sm_100a CUDA
kernels behind the C-ABI library ``lib/libmpo_b200.so``
(include/mpo_b200.h).  There is no CPU fallback.
"""

from .mpo import (CONTRACT_GUARD, DENSIFY_GUARD, DeviceMpo, Mpo, SparseCore,
                  contract_to_matrix, identity_mpo, mpo_add, mpo_round, mpo_transpose,
                  random_mpo, random_unit_rank_mpo, zero_mpo)
from .partition import PartitionPlan, next_pow2, plan_partition, prime_factorize
from .rsvd import (DEFAULT_ROUND_TOL, LowRankSvd, merge_leading_cores, mpo_matmul, mpo_qr,
                   mpo_svd, reconstruct_matrix, subspace_iteration, tnrsvd)
from .sparse import (ConversionResult, SparseMatrixCoo, convert_structure, matrix_to_mpo,
                     min_rank_lower_bound)
from .io import load_mpo, read_matrix_market, save_mpo, write_matrix_market

__version__ = "0.1.0"

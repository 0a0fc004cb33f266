"""Target for compute-sanitizer (memcheck / racecheck / synccheck): one
config-1 TNrSVD (the single-CTA QR/Jacobi paths and the multi-kernel sweeps)
and one 2^16 power-law conversion (bucketed fast path, look-back), each
checked against the oracle so a silent corruption also fails.
    compute-sanitizer --tool memcheck python tools/sanitize_target.py"""
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_1707_07803_b200 as m
from paper_1707_07803_b200.distributed import DeviceOps, convert_sharded
from paper_1707_07803_b200.workloads import TNRSVD_ARGS, config_mpo, powerlaw_coo, square_plan
from oracle import mposvd_oracle as orc

kw = dict(TNRSVD_ARGS["c1"])
a = config_mpo("c1")
lr = m.tnrsvd(a, **kw)
ref = orc.tnrsvd([c.copy() for c in a.cores], kw.pop("k_target"), **kw)
assert np.max(np.abs(lr.s - ref.s) / ref.s) < 1e-8
print("c1 tnrsvd ok")

r, c, v = powerlaw_coo(1 << 16, seed=55)
plan = square_plan(16)
for order in ("row_sorted", "shuffled"):
    if order == "shuffled":
        p = np.random.default_rng(1).permutation(r.size)
        r, c, v = r[p], c[p], v[p]
    tr, tc, tv = (torch.from_numpy(x).cuda() for x in (r, c, v))
    res = convert_sharded(tr, tc, tv, plan, DeviceOps(0))
    st = orc.conversion_structure(r, c, v, plan.row_factors, plan.col_factors)
    assert np.array_equal(st.ti, res.ti.cpu().numpy()) and np.array_equal(st.uniq, res.uniq.cpu().numpy())
    assert np.array_equal(st.i1, res.i1.cpu().numpy()) and np.array_equal(st.j1, res.j1.cpu().numpy())
    print(f"conversion {order} ok: nnz {r.size} blocks {res.rank}")

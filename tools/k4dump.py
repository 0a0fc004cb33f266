"""One config-5 conversion (row-sorted, or shuffled with argv[1] == 'shuffled')
for the k4prof variant's per-bucket dump (MPO_K4DUMP)."""
import sys
import numpy as np
sys.path.insert(0, ".")
import torch
from paper_1707_07803_b200.distributed import DeviceOps, convert_sharded
from paper_1707_07803_b200.workloads import powerlaw_coo, square_plan
r, c, v = powerlaw_coo(1 << 22, seed=55)
if len(sys.argv) > 1 and sys.argv[1] == "shuffled":
    p = np.random.default_rng(1).permutation(r.size)
    r, c, v = r[p], c[p], v[p]
tr, tc, tv = (torch.from_numpy(x).cuda() for x in (r, c, v))
ops = DeviceOps(0)
for _ in range(3):
    convert_sharded(tr, tc, tv, square_plan(22), ops)
torch.cuda.synchronize()

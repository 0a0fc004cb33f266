"""Device conversion of config 5 (2^22, power-law rows) with device-resident input."""
import sys, time
import numpy as np
sys.path.insert(0, ".")
import torch
import paper_1707_07803_b200 as m
from paper_1707_07803_b200.workloads import powerlaw_coo, square_plan
log2n = int(sys.argv[1]) if len(sys.argv) > 1 else 22
r, c, v = powerlaw_coo(1 << log2n, seed=55)
tr, tc, tv = (torch.from_numpy(x).cuda() for x in (r, c, v))
plan = square_plan(log2n)
for it in range(3):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    res = m.convert_structure(tr.data_ptr(), tc.data_ptr(), tv.data_ptr(), plan, n_device=r.size)
    torch.cuda.synchronize(); dt = time.perf_counter() - t0
    print(f"nnz {r.size} rank {res.rank} {dt*1e3:.2f} ms {r.size/dt/1e9:.2f} Gnnz/s")

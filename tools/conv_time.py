"""Time the device conversion of config 5 (2^22 power-law rows) on resident
input: row-sorted (bench input) and shuffled order; CUDA events, 10 reps.
    python tools/conv_time.py [log2n] [reps]"""
import sys
import numpy as np
sys.path.insert(0, ".")
import torch
from paper_1707_07803_b200.distributed import DeviceOps, convert_sharded
from paper_1707_07803_b200.workloads import powerlaw_coo, square_plan
log2n = int(sys.argv[1]) if len(sys.argv) > 1 else 22
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
r, c, v = powerlaw_coo(1 << log2n, seed=55)
plan = square_plan(log2n)
ops = DeviceOps(0)
for order in ("row_sorted", "shuffled"):
    if order == "shuffled":
        p = np.random.default_rng(1).permutation(r.size)
        r, c, v = r[p], c[p], v[p]
    tr, tc, tv = (torch.from_numpy(x).cuda() for x in (r, c, v))
    for _ in range(3):
        res = convert_sharded(tr, tc, tv, plan, ops)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        res = convert_sharded(tr, tc, tv, plan, ops)
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1) / reps
    byt = 32.0 * r.size + 8.0 * res.rank
    print(f"{order}: nnz {r.size} blocks {res.rank} {ms:.3f} ms  {r.size / ms / 1e6:.2f} G nnz/s  "
          f"{byt / ms / 1e6:.0f} GB/s compulsory ({byt / ms / 1e6 / 6518:.3f} of 6518)", flush=True)

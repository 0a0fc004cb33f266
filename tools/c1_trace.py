"""Config-1 TNrSVD latency: wall/device time per call and (MPO_B200_TRACE=1)
the per-stage trace of one call."""
import os
import sys
import time
sys.path.insert(0, ".")
import torch
import paper_1707_07803_b200 as m
from paper_1707_07803_b200 import _lib
from paper_1707_07803_b200.rsvd import prepare, tnrsvd_prepared
from paper_1707_07803_b200.workloads import TNRSVD_ARGS, config_mpo
name = sys.argv[1] if len(sys.argv) > 1 else "c1"
kw = TNRSVD_ARGS[name]
a = config_mpo(name)
am, o, _ = prepare(a, kw["k_target"], kw["oversample"], kw["seed"])
for _ in range(5):
    tnrsvd_prepared(am, o, kw["k_target"], kw["q"], kw["round_tol"])
torch.cuda.synchronize()
n = 20
l0 = _lib.launch_count()
t0 = time.perf_counter()
for _ in range(n):
    tnrsvd_prepared(am, o, kw["k_target"], kw["q"], kw["round_tol"])
torch.cuda.synchronize()
dt = (time.perf_counter() - t0) / n
print(f"{name}: {dt * 1e3:.3f} ms per call, {(_lib.launch_count() - l0) / n:.0f} launches per call")

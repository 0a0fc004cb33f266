"""Config 3 (d=12, n=4, rank 64, decaying middle bond; K=32, p=16) at q=1 or
q=2 on the device: time, output ranks, orthonormality; or the allocation
that fails.  python tools/c3_q.py [q]"""
import sys
import time
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_1707_07803_b200 as m
from paper_1707_07803_b200.workloads import config_mpo
q = int(sys.argv[1]) if len(sys.argv) > 1 else 1
a = config_mpo("c3")
t0 = time.perf_counter()
try:
    lr = m.tnrsvd(a, 32, q=q, round_tol=1e-9, oversample=1.5, seed=4)
except Exception as e:  # noqa: BLE001
    print(f"c3 q={q}: FAILED after {time.perf_counter() - t0:.1f} s: {type(e).__name__}: {e}")
    print("peak allocated GB", torch.cuda.max_memory_allocated() / 1e9)
    sys.exit(0)
dt = time.perf_counter() - t0
print(f"c3 q={q}: {dt:.1f} s  s[:4]={lr.s[:4]}  s[-1]={lr.s[-1]}")
print("U ranks", lr.u.ranks)
print("V ranks", lr.v.ranks)
sys.path.insert(0, "tests")
from oracle import mposvd_oracle as orc
g = orc.gram_first_index(lr.u.cores, lr.u.cores)
print("U ortho", np.linalg.norm(g - np.eye(g.shape[0])))
g = orc.gram_first_index(lr.v.cores, lr.v.cores)
print("V ortho", np.linalg.norm(g - np.eye(g.shape[0])))

"""Host-side phase timing of one public-API TNrSVD call (diagnostic)."""
import sys, time
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_1707_07803_b200 as m
from paper_1707_07803_b200 import rsvd
from paper_1707_07803_b200.workloads import TNRSVD_ARGS, config_mpo
name = sys.argv[1] if len(sys.argv) > 1 else "c2"
a = config_mpo(name)
kw = TNRSVD_ARGS[name]
for rep in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    am, o, kk = rsvd.prepare(a, kw["k_target"], kw["oversample"], kw["seed"])
    torch.cuda.synchronize()
    t1 = time.perf_counter()
    u, s, v = rsvd.tnrsvd_prepared(am, o, kw["k_target"], kw["q"], kw["round_tol"])
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    uh, vh = u.to_host(), v.to_host()
    t3 = time.perf_counter()
    lr = m.tnrsvd(a, **kw)
    t4 = time.perf_counter()
    nb = sum(c.nbytes for c in uh.cores) + sum(c.nbytes for c in vh.cores)
    print(f"prepare {t1-t0:.3f}s device {t2-t1:.3f}s to_host {t3-t2:.3f}s ({nb/1e6:.0f} MB) "
          f"public api {t4-t3:.3f}s", flush=True)

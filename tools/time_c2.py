"""Time one config end to end through the public API (diagnostic)."""
import sys, time
import numpy as np
sys.path.insert(0, ".")
import paper_1707_07803_b200 as m
from paper_1707_07803_b200.workloads import TNRSVD_ARGS, config_mpo
name = sys.argv[1] if len(sys.argv) > 1 else "c2"
a = config_mpo(name)
m.tnrsvd(m.random_mpo([2] * 10, [2] * 10, [3] * 9, seed=1), 10, q=0)  # warm-up / context
import os
for rep in range(int(os.environ.get("REPS", "1"))):
    t = time.time()
    lr = m.tnrsvd(a, **TNRSVD_ARGS[name])
    print(name, "seconds", time.time() - t, "ranks", lr.u.ranks, lr.v.ranks, flush=True)
print("s", lr.s)
try:
    z = np.load(f"tests/golden/big_{name}.npz")
    print("max rel s err", np.max(np.abs(lr.s - z["s"]) / z["s"]),
          "ranks equal", lr.u.ranks == tuple(z["u_ranks"]), lr.v.ranks == tuple(z["v_ranks"]))
except FileNotFoundError:
    pass

"""One config-2 TNrSVD through the prepared (device-resident) path, after a
small warm-up: the target for launch-list captures (ncu -c / --launch-skip)."""
import sys
sys.path.insert(0, ".")
import paper_1707_07803_b200 as m
from paper_1707_07803_b200 import rsvd
from paper_1707_07803_b200.workloads import TNRSVD_ARGS, config_mpo
name = sys.argv[1] if len(sys.argv) > 1 else "c2"
kw = TNRSVD_ARGS[name]
am, o, kk = rsvd.prepare(config_mpo(name), kw["k_target"], kw["oversample"], kw["seed"])
u, s, v = rsvd.tnrsvd_prepared(am, o, kw["k_target"], kw["q"], kw["round_tol"])
print("ok", s[:3])

"""cProfile of the config-1 end-to-end call (host side of tnrsvd(host Mpo))."""
import cProfile
import pstats
import sys
sys.path.insert(0, ".")
import torch
import paper_1707_07803_b200 as m
from paper_1707_07803_b200.workloads import TNRSVD_ARGS, config_mpo
kw = TNRSVD_ARGS["c1"]
a = config_mpo("c1")
for _ in range(5):
    m.tnrsvd(a, **kw)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(50):
    m.tnrsvd(a, **kw)
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)

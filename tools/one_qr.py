"""One device QR of a random m x n matrix (profiling target)."""
import sys
import numpy as np
sys.path.insert(0, ".")
import paper_1707_07803_b200 as m
mm, nn = int(sys.argv[1]), int(sys.argv[2])
a = np.random.default_rng(0).standard_normal((mm, nn))
q, r = m.mpo_qr(m.Mpo([a.reshape(1, mm, nn, 1)]))
print("ok", r[0, 0])

"""Residual / orthogonality of the device QR on a list of shapes: python tools/qr_check.py m,n m,n ..."""
import sys
import numpy as np
sys.path.insert(0, ".")
import paper_1707_07803_b200 as m
for sh in sys.argv[1:]:
    mm, nn = map(int, sh.split(","))
    a = np.random.default_rng(mm + nn).standard_normal((mm, nn))
    q, r = m.mpo_qr(m.Mpo([a.reshape(1, mm, nn, 1)]))
    q = q.cores[0].reshape(mm, nn); r = np.asarray(r)
    print(sh, "orth", np.linalg.norm(q.T @ q - np.eye(nn)), "resid", np.linalg.norm(q @ r - a) / np.linalg.norm(a), flush=True)

"""Device SVD of random (optionally graded) k x k matrices vs numpy: max
relative singular-value error and wall time (MPO_B200_MP=0/1 to compare)."""
import sys, time
import numpy as np
sys.path.insert(0, ".")
import paper_1707_07803_b200 as m
k = int(sys.argv[1]) if len(sys.argv) > 1 else 2048
grade = float(sys.argv[2]) if len(sys.argv) > 2 else 0.0
rng = np.random.default_rng(0)
a = rng.standard_normal((k, k)) * np.logspace(0, -grade, k)[None, :]
mpo = m.Mpo([a.reshape(1, k, k, 1)])
m.mpo_svd(mpo)   # warm-up
t = time.perf_counter()
w, s, v = m.mpo_svd(mpo)
dt = time.perf_counter() - t
ref = np.linalg.svd(a, compute_uv=False)
vt = v.cores[0]                     # V (n x k) as core (1, n, k, 1)
vm = vt.reshape(vt.shape[1], vt.shape[2])
rec = (w * s) @ vm.T
bwd = np.linalg.norm(rec - a) / np.linalg.norm(a)
vorth = np.linalg.norm(vm.T @ vm - np.eye(k))
# Weyl: |s_i - s_i(A)| <= ||A - rec|| + ||A|| * (loss of orthogonality)
print(f"backward error {bwd:.2e}  V orth {vorth:.1e}")
print(f"k={k} grade={grade} {dt*1e3:.1f} ms  max rel s err {np.max(np.abs(s - ref) / ref):.2e}  "
      f"abs err/s0 {np.max(np.abs(s - ref)) / ref[0]:.2e}  W orth {np.linalg.norm(w.T @ w - np.eye(k)):.1e}")

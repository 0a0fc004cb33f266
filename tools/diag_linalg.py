"""Diagnostic: accuracy of the device QR / SVD on single-core MPOs."""
import sys, time
import numpy as np
sys.path.insert(0, ".")
import paper_1707_07803_b200 as m

rng = np.random.default_rng(0)
for (mm, nn) in [(24, 8192), (256, 512), (512, 1024), (300, 700), (1024, 2048)]:
    a = rng.standard_normal((mm, nn)) * (0.8 ** np.arange(mm))[:, None]
    b = m.Mpo([a.reshape(1, mm, nn, 1)])
    t = time.time()
    w, s, v = m.mpo_svd(b)
    dt = time.time() - t
    vm = v.cores[0].reshape(nn, mm)
    sref = np.linalg.svd(a, compute_uv=False)
    print(f"svd {mm}x{nn}: {dt*1e3:.1f} ms  |WtW-I|={np.linalg.norm(w.T@w-np.eye(mm)):.2e} "
          f"|VtV-I|={np.linalg.norm(vm.T@vm-np.eye(mm)):.2e} "
          f"rec={np.linalg.norm(w@np.diag(s)@vm.T-a)/np.linalg.norm(a):.2e} "
          f"s_abs={np.max(np.abs(s-sref))/sref[0]:.2e}", flush=True)
for (mm, nn) in [(8192, 24), (512, 256), (2048, 1024)]:
    a = rng.standard_normal((mm, nn))
    y = m.Mpo([a.reshape(1, mm, nn, 1)])
    t = time.time()
    q, r = m.mpo_qr(y)
    dt = time.time() - t
    qm = q.cores[0].reshape(mm, nn)
    print(f"qr {mm}x{nn}: {dt*1e3:.1f} ms |QtQ-I|={np.linalg.norm(qm.T@qm-np.eye(nn)):.2e} "
          f"rec={np.linalg.norm(qm@r-a)/np.linalg.norm(a):.2e}", flush=True)

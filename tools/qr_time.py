"""Device time of mpo_qr on a one-core MPO (QR of an m x n matrix), CUDA events.
    python tools/qr_time.py m n [reps]"""
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_1707_07803_b200 as m
mm, nn = int(sys.argv[1]), int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
a = m.DeviceMpo.from_host(m.Mpo([np.random.default_rng(0).standard_normal((mm, nn)).reshape(1, mm, nn, 1)]))
m.mpo_qr(a)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    m.mpo_qr(a)
e1.record()
e1.synchronize()
print(f"qr {mm}x{nn}: {e0.elapsed_time(e1) / reps:.3f} ms")

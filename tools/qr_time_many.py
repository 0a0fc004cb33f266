"""CUDA-event time of the device QR on several shapes: python tools/qr_time_many.py m,n ..."""
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_1707_07803_b200 as m
for sh in sys.argv[1:]:
    mm, nn = map(int, sh.split(","))
    a = m.DeviceMpo.from_host(m.Mpo([np.random.default_rng(0).standard_normal((mm, nn)).reshape(1, mm, nn, 1)]))
    m.mpo_qr(a)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        m.mpo_qr(a)
    e1.record()
    e1.synchronize()
    print(f"qr {mm}x{nn}: {e0.elapsed_time(e1) / 5:.3f} ms", flush=True)

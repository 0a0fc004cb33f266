"""QR device time and ledger rate over the sweeps' shapes (dense, one GPU).
    python tools/qr_sweep.py"""
import sys
sys.path.insert(0, ".")
import torch
from paper_1707_07803_b200.tsqr import DenseDeviceOps
from paper_1707_07803_b200 import _lib
import ctypes as C
ops = DenseDeviceOps(0)
shapes = [(1024, 512), (2048, 512), (4096, 512), (8192, 512), (16384, 512), (65536, 512),
          (2048, 2048), (4096, 2048), (8192, 2048), (4096, 4096), (8192, 4096), (16384, 4096),
          (24576, 4096), (32768, 1024), (65536, 256), (196608, 48), (8192, 8192)]
for m, n in shapes:
    a = torch.randn(m, n, dtype=torch.float64, device="cuda")
    ops.qr(a)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 3
    e0.record()
    for _ in range(reps):
        ops.qr(a)
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1) / reps
    fl = 2.0 * (2.0 * m * n * n - 2.0 * n ** 3 / 3.0)
    print(f"qr {m:7d} x {n:5d}: {ms:9.3f} ms  {fl / ms / 1e9:6.2f} TFLOP/s", flush=True)
    del a

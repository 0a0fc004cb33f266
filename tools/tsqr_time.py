"""Per-rank work of the row-sharded TSQR vs the one-GPU QR of the whole
unfolding (device time, CUDA events): python tools/tsqr_time.py m n world"""
import sys
sys.path.insert(0, ".")
import numpy as np
import torch
from paper_1707_07803_b200.tsqr import DenseDeviceOps, tsqr_emulated
m, n, world = (int(x) for x in sys.argv[1:4])
a = torch.from_numpy(np.random.default_rng(0).standard_normal((m, n))).cuda()
ops = DenseDeviceOps(0)
b = np.linspace(0, m, world + 1).astype(int)
shards = [a[b[i]:b[i + 1]].contiguous() for i in range(world)]


def timed(f, reps=5):
    f()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        f()
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / reps


full = timed(lambda: ops.qr(a))
local = timed(lambda: ops.qr(shards[0]))
rs = torch.cat([ops.qr(s)[1] for s in shards])
tree = timed(lambda: ops.qr(rs))
q0, r0 = ops.qr(shards[0])
qs = ops.qr(rs)[0]
assemble = timed(lambda: ops.matmul(q0, qs[:n]))
emul = timed(lambda: tsqr_emulated(shards, ops), reps=2)
print(f"m={m} n={n} P={world}: one-GPU QR {full:.2f} ms | per rank: local QR {local:.2f} + "
      f"tree QR ({world * n}x{n}) {tree:.2f} + Q assembly {assemble:.2f} = "
      f"{local + tree + assemble:.2f} ms (+ all-gather of {world * n * n * 8 / 1e6:.1f} MB) | "
      f"all {world} ranks serialised on one GPU {emul:.2f} ms")

"""Device time of the dense QR (mpo_dense_qr) of an m x n random matrix on
torch's current stream, CUDA events.  python tools/qr_time2.py m n [reps]"""
import sys
sys.path.insert(0, ".")
import torch
from paper_1707_07803_b200.tsqr import DenseDeviceOps
mm, nn = int(sys.argv[1]), int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
ops = DenseDeviceOps(0)
a = torch.randn(mm, nn, dtype=torch.float64, device="cuda")
ops.qr(a)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    ops.qr(a)
e1.record()
e1.synchronize()
print(f"dense qr {mm}x{nn}: {e0.elapsed_time(e1) / reps:.3f} ms (stream {torch.cuda.current_stream().cuda_stream})")

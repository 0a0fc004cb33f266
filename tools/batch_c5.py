"""Config-5 batched TNrSVD: N independent instances (CFG=c5inst_q0 or
c5inst for q=1), run with T host threads, each on its own CUDA stream
(diagnostic)."""
import os, sys, time, threading
sys.path.insert(0, ".")
import numpy as np
import torch
import paper_1707_07803_b200 as m
from paper_1707_07803_b200.rsvd import prepare, tnrsvd_prepared
from paper_1707_07803_b200.workloads import TNRSVD_ARGS, config_mpo
T = int(sys.argv[1]) if len(sys.argv) > 1 else 8
N = int(sys.argv[2]) if len(sys.argv) > 2 else 64
CFG = os.environ.get("CFG", "c5inst_q0")
kw = dict(TNRSVD_ARGS[CFG])
inst = [config_mpo(CFG, i) for i in range(N)]
streams = [torch.cuda.Stream() for _ in range(T)]
prepared = [None] * N
def prep(i, s):
    with torch.cuda.stream(s):
        prepared[i] = prepare(inst[i], kw["k_target"], kw["oversample"], kw["seed"])
for i in range(N): prep(i, streams[i % T])
torch.cuda.synchronize()
out = [None] * N
def worker(tid):
    with torch.cuda.stream(streams[tid]):
        for i in range(tid, N, T):
            am, o, _ = prepared[i]
            out[i] = tnrsvd_prepared(am, o, kw["k_target"], kw["q"], kw["round_tol"])[1]
for rep in range(2):
    t0 = time.perf_counter()
    th = [threading.Thread(target=worker, args=(t,)) for t in range(T)]
    for x in th: x.start()
    for x in th: x.join()
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"rep {rep}: {dt:.3f} s", flush=True)
print(f"threads {T} instances {N} seconds {dt:.3f} per-instance {dt/N*1e3:.1f} ms; s0 {out[0][:3]}")

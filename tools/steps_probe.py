import sys, time
sys.path.insert(0, ".")
import torch
import paper_1707_07803_b200 as m
from paper_1707_07803_b200 import rsvd
from paper_1707_07803_b200.workloads import TNRSVD_ARGS, config_mpo
kw = TNRSVD_ARGS["c2"]
am, o, kk = rsvd.prepare(config_mpo("c2"), kw["k_target"], kw["oversample"], kw["seed"])
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device="cuda")
st = torch.cuda.current_stream()
for rnd in range(3):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
    hs = []
    ev[0].record(st)
    for i in range(4):
        t0 = time.perf_counter()
        if rnd > 0: flush.zero_()
        rsvd.tnrsvd_prepared(am, o, kw["k_target"], kw["q"], kw["round_tol"])
        ev[i + 1].record(st)
        hs.append(time.perf_counter() - t0)
    ev[4].synchronize()
    print("round", rnd, "device ms", [round(ev[i].elapsed_time(ev[i + 1]), 1) for i in range(4)],
          "host s", [round(h, 3) for h in hs], flush=True)
    time.sleep(1.0 if rnd == 1 else 0.0)

"""Record the reference algorithm's FP64 work (SURVEY.md 8(d) ledger) for the
bench workloads by running the oracle restatement with its flop ledger.
Run in the build container; writes bench_data/ledger.json (committed)."""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle import mposvd_oracle as orc  # noqa: E402
from paper_1707_07803_b200.workloads import TNRSVD_ARGS, config_mpo  # noqa: E402

out = {}
for name in sys.argv[1:] or ["c1", "c5inst_q0", "c2"]:
    a = [c.copy() for c in config_mpo(name).cores]
    kw = dict(TNRSVD_ARGS[name])
    led = orc.Ledger()
    t0 = time.perf_counter()
    res = orc.tnrsvd(a, kw.pop("k_target"), ledger=led, **kw)
    secs = time.perf_counter() - t0
    out[name] = {"flops": led.total, "qr": led.qr, "svd": led.svd, "gemm": led.gemm,
                 "einsum": led.einsum, "oracle_seconds_build_container": secs}
    print(name, out[name], flush=True)
path = os.path.join(ROOT, "bench_data", "ledger.json")
old = json.load(open(path)) if os.path.exists(path) else {}
old.update(out)
json.dump(old, open(path, "w"), indent=1, sort_keys=True)

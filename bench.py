"""Benchmark of the B200 TNrSVD / sparse->MPO hot path (BASELINE.json).

Headline workload (N=1): config 2 of BASELINE.json -- TNrSVD of the
2^20 x 2^20 random MPO (d=20, n=2, rank 8, cores N(0,1)/sqrt(8)), K=20,
p=10 (oversample 1.5), q=1, round_tol 1e-9.  A "step" is one full TNrSVD
(time-to-K-triplets).  ``value`` is the reference algorithm's FP64 work
(the oracle's LAPACK/BLAS flop ledger, bench_data/ledger.json, SURVEY.md
8(d)) divided by the device time per step, summed over ranks (each rank
runs an independent replica: TNrSVD does not shard, "replicas only").

The line also carries the conversion metric of BASELINE.json (sparse->MPO
nnz/s, config 5's 2^22 power-law matrix sharded by nonzeros over the
ranks with one NCCL all-gather), the FP64 roofline of the dominant kernel,
the host-CPU baseline (the oracle restatement, numpy/OpenBLAS on this
box's cores) and the end-to-end number through the public API.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
"""

from __future__ import annotations

import argparse
import datetime
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

LEDGER = os.path.join(ROOT, "bench_data", "ledger.json")
METRIC = "TNrSVD time-to-K-triplets as FP64 TFLOP/s (reference flop ledger / device time)"
UNIT = "TFLOP/s"


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=3)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="b200", choices=["b200", "reference"])
    p.add_argument("--workload", default="c2")
    p.add_argument("--no-conversion", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--no-batched", action="store_true")
    p.add_argument("--no-c3", action="store_true")
    return p.parse_args()


def ledger_flops(name):
    return float(json.load(open(LEDGER))[name]["flops"])


# ---------------------------------------------------------------------------
# CPU baseline samples (oracle = test infrastructure, only here and in tests)
# ---------------------------------------------------------------------------

def blas_info():
    """OpenBLAS/MKL build and thread count numpy uses on this host."""
    try:
        from threadpoolctl import threadpool_info
        for x in threadpool_info():
            if x.get("user_api") == "blas":
                return {"library": f"{x.get('internal_api')} {x.get('version')}",
                        "threads": int(x.get("num_threads") or 0)}
    except Exception:  # pragma: no cover
        pass
    return {"library": "unknown", "threads": host_cores()}


def cpu_c2_full(progress=None):
    """The reference algorithm end to end on config 2 (the oracle
    restatement of rsvd.py:217-259, same numpy/LAPACK calls, OpenBLAS on all
    host cores): one complete tnrsvd, its ledger flops counted live.
    ``progress(ledger_total)`` is called after every LAPACK/BLAS call."""
    from oracle import mposvd_oracle as orc
    from paper_1707_07803_b200.workloads import TNRSVD_ARGS, config_mpo
    kw = dict(TNRSVD_ARGS["c2"])
    a = [np.ascontiguousarray(c) for c in config_mpo("c2").cores]
    led = orc.Ledger()
    if progress is not None:
        add = led.add

        def hooked(kind, flops, shape):
            add(kind, flops, shape)
            progress(led.total)
        led.add = hooked
    t0 = time.perf_counter()
    res = orc.tnrsvd(a, kw.pop("k_target"), ledger=led, **kw)
    secs = time.perf_counter() - t0
    return led.total, secs, res


def cpu_c1_median():
    """Config 1 through the oracle, median of 3 (reference bench.py:148-155)."""
    from oracle import mposvd_oracle as orc
    from paper_1707_07803_b200.workloads import TNRSVD_ARGS, config_mpo
    kw = dict(TNRSVD_ARGS["c1"])
    a = [np.ascontiguousarray(c) for c in config_mpo("c1").cores]
    k = kw.pop("k_target")
    _, secs = orc.timed(lambda: orc.tnrsvd([c.copy() for c in a], k, **kw), repeats=3)
    return secs


def cpu_conversion_full(log2n=22):
    """Config 5's whole conversion through the oracle port of matrix_to_mpo
    (sparse.py:207-258 with SparseCore index arrays, single-threaded numpy,
    as the reference) and, separately, the SparseMatrixCoo constructor's
    validation (sparse.py:53-70)."""
    from oracle import mposvd_oracle as orc
    from paper_1707_07803_b200.workloads import powerlaw_coo
    n = 1 << log2n
    r, c, v = powerlaw_coo(n, seed=55)
    t0 = time.perf_counter()
    orc.coo_validate(n, n, r, c, v)
    t_ctor = time.perf_counter() - t0
    t0 = time.perf_counter()
    orc.matrix_to_mpo_arrays(r, c, v, (2,) * log2n, (2,) * log2n)
    t_conv = time.perf_counter() - t0
    return r.size, t_conv, t_ctor


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


# ---------------------------------------------------------------------------
# clocks sampled during the timed region
# ---------------------------------------------------------------------------

class Clocks:
    """nvidia-smi sampler (200 ms).  It is started before the warm-up (its
    start-up would otherwise land inside the first timed step) and only the
    samples stamped inside [start(), stop()] — the timed region — count."""
    FIELDS = ("timestamp,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.path = None
        self.t0 = self.t1 = None

    def start(self):
        self.t0 = datetime.datetime.now()

    def stop(self):
        self.t1 = datetime.datetime.now()

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        if os.environ.get("BENCH_NO_CLOCKS"):   # diagnostics only: no sampler
            return self
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:  # pragma: no cover
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        try:
            for line in open(self.path):
                f = [x.strip() for x in line.split(",")]
                if len(f) < 9:
                    continue
                try:
                    ts = datetime.datetime.strptime(f[0], "%Y/%m/%d %H:%M:%S.%f")
                    if (self.t0 and ts < self.t0) or (self.t1 and ts > self.t1):
                        continue
                    clk, cmax = float(f[1]), float(f[2])
                except ValueError:
                    continue
                sm.append(clk)
                mx = cmax
                for nm, val in zip(names, f[5:9]):
                    if val.lower() == "active":
                        reasons.add(nm)
        finally:
            os.unlink(self.path)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx,
                "sm_min_mhz": min(sm) if sm else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# reference arm
# ---------------------------------------------------------------------------

def run_reference(args, rank, world):
    """The reference's CPU implementation of the headline path on this
    box's host cores: config 2's tnrsvd end to end (the oracle restatement,
    same numpy/OpenBLAS calls; /root/reference does not travel to the GPU
    box).  Warm-up: W config-1 runs.  Timed region: ONE complete config-2
    run (~2 min) -- the --steps K are K equal slices of its flop ledger, so
    ms_per_step = total / K and value = ledger flops / total time."""
    if rank != 0:
        return
    from oracle import mposvd_oracle as orc
    from paper_1707_07803_b200.workloads import TNRSVD_ARGS, config_mpo
    kw1 = dict(TNRSVD_ARGS["c1"])
    a1 = [np.ascontiguousarray(c) for c in config_mpo("c1").cores]
    k1 = kw1.pop("k_target")
    for _ in range(max(args.warmup, 0)):
        orc.tnrsvd([c.copy() for c in a1], k1, **kw1)
    total = ledger_flops("c2")
    marks = []
    steps = max(args.steps, 1)

    def progress(done):
        while len(marks) < steps and done >= total * (len(marks) + 1) / steps * (1 - 1e-12):
            marks.append(time.perf_counter())

    t0 = time.perf_counter()
    flops, secs, res = cpu_c2_full(progress)
    step_s = [b - a for a, b in zip([t0] + marks[:-1], marks)] if len(marks) == steps else []
    value = flops / secs / 1e12
    blas = blas_info()
    sample = (f"one complete config-2 tnrsvd (oracle port of rsvd.py:217-259, numpy "
              f"{np.__version__}, {blas['library']}, {blas['threads']} threads), timed as "
              f"{steps} equal-ledger steps; ledger {flops:.4g} flops")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": world, "steps": steps, "warmup": args.warmup,
        "ms_per_step": 1e3 * secs / steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": "c2: TNrSVD of random MPO d=20 n=2 rank 8 (N(0,1)/sqrt(8)), "
                               "K=20 p=10 q=1 round_tol=1e-9",
                   "time_to_k_triplets_s": secs},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": blas["threads"], "kind": "port",
                         "sample": sample, "seconds": secs},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "step_seconds": step_s,
        "s_head": [float(x) for x in res.s[:3]],
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# B200 arm
# ---------------------------------------------------------------------------

def fp64_peak_tflops(torch):
    """cuBLAS DGEMM 8192^3 (torch.matmul float64), best of 5: the FP64
    denominator MEASURED_PEAKS.json lacks."""
    n = 8192
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    torch.matmul(a, b)
    torch.cuda.synchronize()
    best = 1e30
    for _ in range(5):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        torch.matmul(a, b)
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1) / 1e3)
    del a, b
    return 2.0 * n ** 3 / best / 1e12


def run_b200(args, rank, world, local_rank):
    import torch
    import torch.distributed as dist
    import paper_1707_07803_b200 as m
    from paper_1707_07803_b200 import _lib
    from paper_1707_07803_b200.rsvd import prepare, tnrsvd_prepared
    from paper_1707_07803_b200.workloads import TNRSVD_ARGS, config_mpo

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    name = args.workload
    kw = dict(TNRSVD_ARGS[name])
    flops = ledger_flops(name)
    a_host = config_mpo(name)

    def barrier():
        if world > 1:
            dist.barrier()

    def max_over_ranks(x):
        if world == 1:
            return x
        t = torch.tensor([x], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    peak = fp64_peak_tflops(torch)
    try:
        traffic = json.load(open(os.path.join(ROOT, "profiles", "r02_traffic.json")))
    except (OSError, ValueError):
        traffic = {}
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)  # 256 MB > 126 MB L2

    am, o, kk = prepare(a_host, kw["k_target"], kw["oversample"], kw["seed"])

    def step():
        u, s, v = tnrsvd_prepared(am, o, kw["k_target"], kw["q"], kw["round_tol"])
        return s

    clk = Clocks(local_rank).__enter__()   # sampler up before the warm-up
    for _ in range(args.warmup):   # same loop body as the timed one (lazy-loaded fill kernel)
        flush.zero_()
        step()
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    l0 = _lib.launch_count()
    stream = torch.cuda.current_stream()
    try:
        clk.start()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        marks = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
        e0.record(stream)
        for i in range(args.steps):
            flush.zero_()
            s = step()
            marks[i].record(stream)
        e1.record(stream)
        e1.synchronize()
        clk.stop()
    finally:
        clk.__exit__(None, None, None)
    step_ms = [e0.elapsed_time(marks[0])] + [marks[i - 1].elapsed_time(marks[i])
                                             for i in range(1, args.steps)]
    print("[bench] c2 device ms per step:", " ".join(f"{x:.1f}" for x in step_ms), file=sys.stderr)
    torch.cuda.synchronize()
    barrier()
    launches = _lib.launch_count() - l0
    secs = max_over_ranks(e0.elapsed_time(e1) / 1e3)
    per_step = secs / args.steps
    value = world * flops / per_step / 1e12

    # end to end through the public API: host Mpo in, host Mpo out.  Same
    # warm-up rule as above (the first calls populate the pinned host pool
    # the downloads land in)
    for _ in range(args.warmup):
        flush.zero_()
        lr = m.tnrsvd(a_host, **kw)
    del lr
    barrier()
    torch.cuda.synchronize()
    h2d = sum(c.nbytes for c in a_host.cores)
    d2h = 0
    e2 = torch.cuda.Event(enable_timing=True)
    e3 = torch.cuda.Event(enable_timing=True)
    e2.record(stream)
    for _ in range(args.steps):
        flush.zero_()
        lr = m.tnrsvd(a_host, **kw)
        d2h = sum(c.nbytes for c in lr.u.cores) + sum(c.nbytes for c in lr.v.cores) + lr.s.nbytes
    e3.record(stream)
    e3.synchronize()
    e2e_secs = max_over_ranks(e2.elapsed_time(e3) / 1e3) / args.steps
    e2e_value = world * flops / e2e_secs / 1e12

    # roofline of the dominant kernel family: CUDA events around every
    # Jacobi round kernel, DGEMM launch and QR panel of one extra step
    _lib.call("mpo_b200_profile_enable", 1)
    step()
    torch.cuda.synchronize()
    prof = {}
    import ctypes as C
    names = ["jacobi_gram_kernel", "jacobi_eig_kernel", "jacobi_apply_kernel", "dgemm_kernel",
             "qr_panel_cluster_kernel", "qr_inblock_cluster_kernel"]
    for idx, kname in enumerate(names):
        ms, fl, n = C.c_double(), C.c_double(), C.c_ulonglong()
        _lib.call("mpo_b200_profile_read", idx, C.byref(ms), C.byref(fl), C.byref(n))
        prof[kname] = (ms.value, fl.value, n.value)
    _lib.call("mpo_b200_profile_enable", 0)
    # the tensor-pipe kernel with the most time (the QR panel is latency
    # bound: its share is reported, not a roofline)
    dom = max(("jacobi_gram_kernel", "jacobi_apply_kernel", "dgemm_kernel"),
              key=lambda k: prof[k][0])
    ms_d, fl_d, n_d = prof[dom]
    achieved = fl_d / (ms_d / 1e3) / 1e12 if ms_d > 0 else 0.0
    step_ms = per_step * 1e3
    roofline = {
        "bound": "tensor", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "TFLOP/s",
        "frac": achieved / peak if peak else None,
        "traffic": traffic.get("dram_bytes_per_launch") if dom == traffic.get("kernel") else None,
        "traffic_note": traffic.get("note"),
        "peak_source": "measured in this run: cuBLAS DGEMM 8192^3 (torch.matmul float64); "
                       "MEASURED_PEAKS.json has no FP64 figure",
        "avg_launch_us": 1e3 * ms_d / max(n_d, 1), "launches_per_step": n_d,
        "flops_per_step": fl_d,
        "share_of_step": (ms_d / step_ms) if step_ms else None,
        "kernel_ms_per_step": {k: v[0] for k, v in prof.items()},
        "kernel_launches_per_step": {k: v[2] for k, v in prof.items()},
        "timing": "CUDA events around every launch of one extra (profiling) step; each "
                  "timed launch synchronises its stream, so shares are of serialised time",
    }

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": per_step * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded numpy generators of BASELINE.json configs; no dataset)",
        "config": {"workload": f"{name}: TNrSVD of random MPO d=20 n=2 rank 8 (N(0,1)/sqrt(8)), "
                               "K=20 p=10 q=1 round_tol=1e-9" if name == "c2" else name,
                   "parallelism": f"replicas x{world} (independent instances)",
                   "ledger_flops_per_step": flops, "l2": "flushed (256 MB write) before each step",
                   "time_to_k_triplets_s": per_step},
        "roofline": roofline,
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h), "seconds_per_step": e2e_secs,
                "api": "paper_1707_07803_b200.tnrsvd(host Mpo) -> host U, s, V"},
        "gpu_launches": int(launches),
        "clocks": clk.summary(),
        "s_head": [float(x) for x in s[:3]],
    }

    if not args.no_conversion:
        line["conversion"] = bench_conversion(args, torch, dist, rank, world, dev, barrier,
                                              max_over_ranks)
    line["c1"] = bench_c1(args, torch, rank, world, barrier, max_over_ranks)
    line["tsqr"] = bench_tsqr(args, torch, rank, world, dev, barrier, max_over_ranks)
    if not args.no_c3:
        line["tnrsvd_c3q0"] = bench_c3q0(args, torch, rank, world, barrier, max_over_ranks)
    if not args.no_batched:
        line["tnrsvd_batched"] = bench_batched(args, torch, rank, world, barrier, max_over_ranks,
                                               cfg="c5inst")
        line["tnrsvd_batched_q0"] = bench_batched(args, torch, rank, world, barrier,
                                                  max_over_ranks, cfg="c5inst_q0")
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        fl, secs, _ = cpu_c2_full()
        blas = blas_info()
        line["cpu_baseline"] = {
            "value": fl / secs / 1e12, "unit": UNIT, "cores": blas["threads"], "kind": "port",
            "sample": f"one complete config-2 tnrsvd, oracle port of rsvd.py:217-259 (numpy "
                      f"{np.__version__}, {blas['library']}); {secs:.1f} s to K triplets vs "
                      f"{per_step:.3f} s on the B200", "seconds": secs}
        if "c1" in line:
            cs1 = cpu_c1_median()
            line["c1"]["cpu_baseline"] = {"value": cs1 * 1e3, "unit": "ms", "cores": blas["threads"],
                                          "kind": "port", "sample": "config-1 tnrsvd, oracle, "
                                          "median of 3 (reference bench.py:148-155)"}
        if "conversion" in line:
            nnz, tc, tctor = cpu_conversion_full()
            line["conversion"]["cpu_baseline"] = {
                "value": nnz / tc, "unit": "nnz/s", "cores": 1, "kind": "port",
                "sample": "config 5 at 2^22 (32.7M nnz): oracle port of the whole uncapped "
                          "matrix_to_mpo (sparse.py:207-258, SparseCore index arrays), "
                          "single-threaded numpy as the reference",
                "seconds": tc, "coo_constructor_seconds": tctor}
    if rank == 0:
        print(json.dumps(line), flush=True)


def bench_tsqr(args, torch, rank, world, dev, barrier, max_over_ranks, m=131072, n=512):
    """one tall unfolding (m x n, the L2R sweep's QR at
    rsvd.py:106) whose rows are sharded over the ranks, factored by the
    row-distributed TSQR (tsqr.py: local QR, one NCCL all-gather of the
    n x n factors, tree QR, Q assembly).  Strong scaling: the same matrix at
    every N.  value = the reference's QR ledger flops 2 (2 m n^2 - 2 n^3 / 3)
    per second of device time (max over ranks)."""
    from paper_1707_07803_b200.tsqr import DenseDeviceOps, tsqr
    rng = np.random.default_rng(77)
    b = np.linspace(0, m, world + 1).astype(int)
    lo, hi = int(b[rank]), int(b[rank + 1])
    full = rng.standard_normal((m, n))
    a = torch.from_numpy(full[lo:hi]).to(dev)
    del full
    ops = DenseDeviceOps(dev.index)
    for _ in range(max(args.warmup, 1)):
        q, r = tsqr(a, ops)
    torch.cuda.synchronize()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = max(args.steps, 3)
    e0.record()
    for _ in range(reps):
        q, r = tsqr(a, ops)
    e1.record()
    e1.synchronize()
    secs = max_over_ranks(e0.elapsed_time(e1) / 1e3) / reps
    flops = 2.0 * (2.0 * m * n * n - 2.0 * n ** 3 / 3.0)
    return {"metric": f"row-sharded TSQR of a {m}x{n} unfolding (rsvd.py:106), ledger FP64 TFLOP/s",
            "value": flops / secs / 1e12, "unit": "TFLOP/s", "seconds": secs, "n_gpus": world,
            "scaling": "strong", "rows_per_rank": hi - lo,
            "exchange": "one all-gather of the n x n R factors" if world > 1 else "none (one GPU)"}


def bench_c1(args, torch, rank, world, barrier, max_over_ranks, steps=20):
    """Config 1 (BASELINE configs[0]: d=10 n=2 rank 3, K=10, p=10, q=0) --
    the latency-bound regime: device time per tnrsvd on resident inputs and
    end to end through tnrsvd(host Mpo) (upload + download inside)."""
    import paper_1707_07803_b200 as m
    from paper_1707_07803_b200.rsvd import prepare, tnrsvd_prepared
    from paper_1707_07803_b200.workloads import TNRSVD_ARGS, config_mpo
    kw = TNRSVD_ARGS["c1"]
    a = config_mpo("c1")
    am, o, _ = prepare(a, kw["k_target"], kw["oversample"], kw["seed"])
    for _ in range(3):
        tnrsvd_prepared(am, o, kw["k_target"], kw["q"], kw["round_tol"])
        m.tnrsvd(a, **kw)
    torch.cuda.synchronize()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        tnrsvd_prepared(am, o, kw["k_target"], kw["q"], kw["round_tol"])
    e1.record()
    e1.synchronize()
    dev_ms = max_over_ranks(e0.elapsed_time(e1) / steps)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(steps):
        lr = m.tnrsvd(a, **kw)
    torch.cuda.synchronize()
    e2e_ms = max_over_ranks((time.perf_counter() - t0) * 1e3 / steps)
    return {"metric": "config-1 TNrSVD time-to-K-triplets", "value": dev_ms, "unit": "ms",
            "higher_is_better": False, "n_gpus": world, "scaling": "weak",
            "e2e": {"value": e2e_ms, "unit": "ms",
                    "h2d_bytes_per_step": int(sum(c.nbytes for c in a.cores)),
                    "d2h_bytes_per_step": int(sum(c.nbytes for c in lr.u.cores) +
                                              sum(c.nbytes for c in lr.v.cores) + lr.s.nbytes),
                    "api": "paper_1707_07803_b200.tnrsvd(host Mpo)"},
            "s_head": [float(x) for x in lr.s[:3]]}


def bench_c3q0(args, torch, rank, world, barrier, max_over_ranks):
    """Config 3 (d=12, n=4, rank 64, decaying middle bond; K=32, p=16) at
    q=0, the largest setting the reference finishes (213 s on 8 cores in
    the build container; q=2 needs a 1.5 TiB product core at rsvd.py:77).
    One replica per rank, device-resident inputs, CUDA-event timed."""
    from paper_1707_07803_b200.rsvd import prepare, tnrsvd_prepared
    from paper_1707_07803_b200.workloads import TNRSVD_ARGS, config_mpo
    kw = TNRSVD_ARGS["c3q0"]
    am, o, _ = prepare(config_mpo("c3q0"), kw["k_target"], kw["oversample"], kw["seed"])
    tnrsvd_prepared(am, o, kw["k_target"], kw["q"], kw["round_tol"])   # warm-up
    torch.cuda.synchronize()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    steps = 2
    e0.record()
    for _ in range(steps):
        _, s, _ = tnrsvd_prepared(am, o, kw["k_target"], kw["q"], kw["round_tol"])
    e1.record()
    e1.synchronize()
    secs = max_over_ranks(e0.elapsed_time(e1) / 1e3 / steps)
    try:
        flops = ledger_flops("c3q0")
    except (KeyError, OSError, ValueError):
        flops = None
    return {"metric": "config-3 TNrSVD (q=0) time-to-K-triplets", "seconds": secs,
            "value": (flops / secs / 1e12 * world) if flops else None, "unit": "TFLOP/s",
            "ledger_flops_per_step": flops, "n_gpus": world, "scaling": "weak",
            "reference_seconds_build_container": 213.2, "s_head": [float(x) for x in s[:3]],
            "note": "q=0: the BASELINE q=2 is infeasible for the reference and for any faithful "
                    "implementation (exact bond ranks 16384 at rank-64x16384 products)"}


def bench_batched(args, torch, rank, world, barrier, max_over_ranks, n_inst=64, threads=8,
                  cfg="c5inst"):
    """Config 5's batched TNrSVD: 64 independent instances (d=20, n=2,
    rank 16, K=16, p=8, q=1 as BASELINE.json states it; cfg="c5inst_q0" for
    the q=0 variant) split over the ranks; on each GPU the rank's instances
    run concurrently from `threads` host threads, one CUDA stream each.  q=1
    is infeasible for the reference (48 GiB product core at rsvd.py:77); the
    device runs it through the fused rank-bounded sweeps (csrc/sweep.cu)."""
    import threading
    from paper_1707_07803_b200.rsvd import prepare, tnrsvd_prepared
    from paper_1707_07803_b200.workloads import TNRSVD_ARGS, config_mpo
    kw = dict(TNRSVD_ARGS[cfg])
    mine = [i for i in range(n_inst) if i % world == rank]
    streams = [torch.cuda.Stream() for _ in range(threads)]
    prepared = {}
    for j, i in enumerate(mine):
        with torch.cuda.stream(streams[j % threads]):
            prepared[i] = prepare(config_mpo(cfg, i), kw["k_target"], kw["oversample"],
                                  kw["seed"])
    torch.cuda.synchronize()
    out = {}

    def worker(tid, todo):
        with torch.cuda.stream(streams[tid]):
            for j in range(tid, len(todo), threads):
                am, o, _ = prepared[todo[j]]
                out[todo[j]] = tnrsvd_prepared(am, o, kw["k_target"], kw["q"], kw["round_tol"])[1]

    def run_all(todo):
        th = [threading.Thread(target=worker, args=(t, todo)) for t in range(threads)]
        for x in th:
            x.start()
        for x in th:
            x.join()
        torch.cuda.synchronize()

    # warm-up: one instance per host thread (q=1 instances take seconds each)
    run_all(mine[:threads] if kw["q"] > 0 else mine)
    barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    run_all(mine)
    secs = max_over_ranks(time.perf_counter() - t0)
    res = {"metric": f"config-5 batched TNrSVD instances/s (64 instances, q={kw['q']})",
           "value": n_inst / secs, "unit": "instances/s", "n_gpus": world, "scaling": "strong",
           "seconds": secs, "host_threads_per_gpu": threads,
           "s0_head": [float(x) for x in out[mine[0]][:3]],
           "note": "wall clock of the whole batch (host threads + streams), max over ranks"}
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        from oracle import mposvd_oracle as orc
        kq = dict(TNRSVD_ARGS["c5inst_q0"])
        a = [c.copy() for c in config_mpo("c5inst_q0", 0).cores]
        t1 = time.perf_counter()
        orc.tnrsvd(a, kq.pop("k_target"), **kq)
        cs = time.perf_counter() - t1
        res["cpu_baseline"] = {
            "value": 1.0 / cs, "unit": "instances/s", "cores": host_cores(), "kind": "port",
            "sample": "one config-5 instance at q=0, oracle" +
                      ("; q=1 is oracle-infeasible (MemoryError: 48 GiB product core, "
                       "rsvd.py:77)" if kw["q"] > 0 else "")}
    return res


def bench_conversion(args, torch, dist, rank, world, dev, barrier, max_over_ranks):
    """Config 5's conversion: 2^22 square, power-law rows (alpha 2.1), uniform
    columns, U(-1,1) values, plan ([2]*22, [2]*22); nnz sharded over ranks
    (contiguous input ranges), block keys exchanged by key range
    (distributed.py: samples -> splitters, one all-to-all of keys, one back
    of global ids).  The timed region covers the whole sharded conversion
    incl. the exchange; the input (785 MB of COO) exceeds the 126 MB L2."""
    from paper_1707_07803_b200.distributed import DeviceOps, convert_sharded, shard_range
    from paper_1707_07803_b200.workloads import powerlaw_coo, square_plan
    r, c, v = powerlaw_coo(1 << 22, seed=55)
    n = r.size
    lo, hi = shard_range(n, world, rank)
    tr = torch.from_numpy(r[lo:hi]).to(dev)
    tc = torch.from_numpy(c[lo:hi]).to(dev)
    tv = torch.from_numpy(v[lo:hi]).to(dev)
    plan = square_plan(22)
    ops = DeviceOps(dev.index)
    for _ in range(args.warmup):
        res = convert_sharded(tr, tc, tv, plan, ops)
    torch.cuda.synchronize()
    barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(args.steps):
        res = convert_sharded(tr, tc, tv, plan, ops)
    e1.record()
    e1.synchronize()
    secs = max_over_ranks(e0.elapsed_time(e1) / 1e3) / args.steps
    blocks = res.rank
    compulsory = 32.0 * n + 8.0 * blocks   # read 24 B/nnz, write ti 8 B, uniq 8 B
    # the same shard in shuffled order (a COO in no particular order takes the
    # full-key in-bucket sort); reported beside the row-sorted headline
    perm = torch.from_numpy(np.random.default_rng(1).permutation(hi - lo)).to(dev)
    sr, sc, sv = tr[perm], tc[perm], tv[perm]
    del perm
    for _ in range(args.warmup):
        convert_sharded(sr, sc, sv, plan, ops)
    torch.cuda.synchronize()
    barrier()
    e0.record()
    for _ in range(args.steps):
        convert_sharded(sr, sc, sv, plan, ops)
    e1.record()
    e1.synchronize()
    secs_shuf = max_over_ranks(e0.elapsed_time(e1) / 1e3) / args.steps
    del sr, sc, sv
    peak_hbm = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6521.1
    achieved = compulsory / secs / 1e9 / world   # per GPU
    try:
        ctraffic = json.load(open(os.path.join(ROOT, "profiles", "r02_conv_traffic.json")))
    except (OSError, ValueError):
        ctraffic = {}
    # end to end through the sharded path: this rank's host COO shard
    # (pinned) -> HBM, conversion + exchange, (i1, j1, ti, values, uniq
    # shard) -> pinned host
    pin = lambda x: torch.from_numpy(x).pin_memory()
    hr, hc, hv = pin(r[lo:hi]), pin(c[lo:hi]), pin(v[lo:hi])
    outs = None

    def e2e_step():
        nonlocal outs
        res = convert_sharded(hr.to(dev, non_blocking=True), hc.to(dev, non_blocking=True),
                              hv.to(dev, non_blocking=True), plan, ops)
        arrs = (res.i1, res.j1, res.ti, res.values, res.uniq)
        if outs is None or any(o.numel() != a.numel() for o, a in zip(outs, arrs)):
            outs = [torch.empty(a.numel(), dtype=a.dtype, pin_memory=True) for a in arrs]
        for o, a in zip(outs, arrs):
            o.copy_(a, non_blocking=True)
        torch.cuda.synchronize()
        return sum(o.numel() * o.element_size() for o in outs)

    for _ in range(args.warmup):
        d2h = e2e_step()
    barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        d2h = e2e_step()
    e2e = max_over_ranks((time.perf_counter() - t0) / args.steps)
    return {
        "metric": "sparse->MPO conversion nnz/s (config 5, 2^22 power-law, d=22)",
        "value": n / secs, "unit": "nnz/s", "n_gpus": world, "scaling": "strong",
        "nnz": int(n), "blocks": int(blocks), "ms_per_step": secs * 1e3,
        "input_order": "row-sorted COO (deduplicated by np.unique)",
        "shuffled_input": {"value": n / secs_shuf, "unit": "nnz/s", "ms_per_step": secs_shuf * 1e3,
                           "note": "same shard, randomly permuted entries"},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak_hbm, "unit": "GB/s",
                     "frac": achieved / peak_hbm,
                     "traffic": ctraffic.get("dram_bytes_per_step"),
                     "traffic_source": ctraffic.get("source"),
                     "algorithmic_bytes_per_step": compulsory,
                     "note": "whole conversion (compaction + radix passes + segment + ids) "
                             "timed; compulsory bytes 32 B/nnz + 8 B/block (SURVEY 8(d))"},
        "e2e": {"value": n / e2e, "unit": "nnz/s",
                "h2d_bytes_per_step": int(24 * (hi - lo)) * world,
                "d2h_bytes_per_step": int(d2h) * world,
                "api": "distributed.convert_sharded on each rank's pinned host shard "
                       "(H2D, convert + key-range exchange, D2H of i1/j1/ti/values/uniq)"},
    }


def main():
    args = parse()
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: relaunch under torchrun (rank 0 prints the line)
        import socket
        sk = socket.socket()
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
        sk.close()
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
               f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
        sys.exit(subprocess.call(cmd))
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world != args.gpus and rank == 0:
        print(f"[bench] note: --gpus {args.gpus} but WORLD_SIZE={world}; reporting n_gpus={world}",
              file=sys.stderr)
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    try:
        run_b200(args, rank, world, local_rank)
    finally:
        if world > 1:
            import torch.distributed as dist
            dist.destroy_process_group()


if __name__ == "__main__":
    main()

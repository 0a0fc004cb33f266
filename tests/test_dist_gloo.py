"""World-size-2 gloo test of the sharded conversion's exchange logic
(paper_1707_07803_b200/distributed.py) on CPU.  The per-rank device
primitives are replaced by oracle-backed CPU equivalents; the all-gather,
padding, global merge and id remap are the product code."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle import mposvd_oracle as orc


class CpuOps:
    """Oracle-backed stand-ins for DeviceOps (test infrastructure)."""

    def local(self, row1, col1, val, plan):
        st = orc.conversion_structure(row1.numpy(), col1.numpy(), val.numpy(),
                                      plan.row_factors, plan.col_factors)
        t = lambda a: torch.from_numpy(np.ascontiguousarray(a))
        return t(st.i1), t(st.j1), t(st.ti), t(st.values), t(st.uniq)

    def unique(self, keys, max_key):
        return torch.from_numpy(np.unique(keys.numpy()))

    def lookup(self, table, q):
        idx = np.searchsorted(table.numpy(), q.numpy())
        return torch.from_numpy(idx.astype(np.int64))

    def remap(self, mapping, ti):
        return mapping[ti]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1707_07803_b200.distributed import convert_sharded, shard_range
        from paper_1707_07803_b200.workloads import powerlaw_coo, square_plan
        r, c, v = powerlaw_coo(1 << 12, seed=11)
        v[::7] = 0.0   # explicit zeros are dropped before keying (sparse.py:234)
        lo, hi = shard_range(r.size, world, rank)
        res = convert_sharded(torch.from_numpy(r[lo:hi]), torch.from_numpy(c[lo:hi]),
                              torch.from_numpy(v[lo:hi]), square_plan(12), CpuOps())
        q.put((rank, res.ti.numpy(), res.i1.numpy(), res.uniq.numpy(), res.rank,
               res.kept_offset, res.nkept_total))
    finally:
        dist.destroy_process_group()


def test_sharded_conversion_matches_single_device_world2():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = sorted([q.get(timeout=180) for _ in range(world)], key=lambda x: x[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    from paper_1707_07803_b200.workloads import powerlaw_coo, square_plan
    r, c, v = powerlaw_coo(1 << 12, seed=11)
    v[::7] = 0.0
    plan = square_plan(12)
    ref = orc.conversion_structure(r, c, v, plan.row_factors, plan.col_factors)
    ti = np.concatenate([o[1] for o in out])
    i1 = np.concatenate([o[2] for o in out])
    assert np.array_equal(ti, ref.ti)
    assert np.array_equal(i1, ref.i1)
    for o in out:
        assert np.array_equal(o[3], ref.uniq)
        assert o[4] == ref.rank
        assert o[6] == ref.ti.size
    assert out[0][5] == 0 and out[1][5] == out[0][1].size

"""Multi-process gloo tests (world size 2 and 3) of the sharded conversion's
key-range exchange (paper_1707_07803_b200/distributed.py) on CPU, plus the
lock-step emulation of 2/4/8 ranks.  The per-rank device primitives are
replaced by oracle-backed CPU equivalents; the sampling, splitters,
all-to-all exchange, range merge, id assignment and remap are the product
code."""

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
        from paper_1707_07803_b200.distributed import Entries
        t = lambda a: torch.from_numpy(np.ascontiguousarray(a))
        return Entries(t(st.i1), t(st.j1), t(st.values)), t(st.ti), t(st.uniq)

    def unique(self, keys, max_key):
        return torch.from_numpy(np.unique(keys.numpy()))

    def search(self, table, q, offset=0, exact=False):
        t, x = table.numpy(), q.numpy()
        idx = np.searchsorted(t, x).astype(np.int64)
        if exact:
            ok = (idx < t.size) & (t[np.minimum(idx, max(t.size - 1, 0))] == x) if t.size else \
                np.zeros(x.size, bool)
            return torch.from_numpy(np.where(ok, idx + offset, -1))
        return torch.from_numpy(idx + offset)

    def remap(self, mapping, ti):
        return mapping[ti]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _input():
    from paper_1707_07803_b200.workloads import powerlaw_coo, square_plan
    r, c, v = powerlaw_coo(1 << 12, seed=11)
    v[::7] = 0.0   # explicit zeros are dropped before keying (sparse.py:234)
    return r, c, v, square_plan(12)


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1707_07803_b200.distributed import convert_sharded, shard_range
        r, c, v, plan = _input()
        lo, hi = shard_range(r.size, world, rank)
        res = convert_sharded(torch.from_numpy(r[lo:hi]), torch.from_numpy(c[lo:hi]),
                              torch.from_numpy(v[lo:hi]), plan, CpuOps())
        full = convert_sharded(torch.from_numpy(r[lo:hi]), torch.from_numpy(c[lo:hi]),
                               torch.from_numpy(v[lo:hi]), plan, CpuOps(), replicate=True)
        q.put((rank, res.ti.numpy(), res.i1.numpy(), res.uniq.numpy(), res.rank,
               res.kept_offset, res.nkept_total, res.uniq_offset, full.uniq.numpy()))
    finally:
        dist.destroy_process_group()


def _check(out, world):
    r, c, v, plan = _input()
    ref = orc.conversion_structure(r, c, v, plan.row_factors, plan.col_factors)
    ti = np.concatenate([o[1] for o in out])
    i1 = np.concatenate([o[2] for o in out])
    assert np.array_equal(ti, ref.ti)
    assert np.array_equal(i1, ref.i1)
    # key-range shards of uniq concatenate to the global list, offsets agree
    assert np.array_equal(np.concatenate([o[3] for o in out]), ref.uniq)
    off = 0
    for o in out:
        assert o[7] == off
        off += o[3].size
        assert o[4] == ref.rank
        assert o[6] == ref.ti.size
        assert np.array_equal(o[8], ref.uniq)
    # balanced key ranges (256 samples per rank): no rank holds > 2x its share
    assert max(o[3].size for o in out) <= 2 * ref.rank / world + 64
    kept = np.cumsum([0] + [o[1].size for o in out])
    assert [o[5] for o in out] == list(kept[:-1])


@pytest.mark.parametrize("world", [2, 3])
def test_sharded_conversion_matches_single_device_gloo(world):
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
    _check(out, world)


@pytest.mark.parametrize("world", [2, 4, 8])
def test_sharded_conversion_emulated(world):
    """The same per-rank code driven in lock step (collectives emulated)."""
    from paper_1707_07803_b200.distributed import convert_sharded_emulated, shard_range
    r, c, v, plan = _input()
    shards = []
    for k in range(world):
        lo, hi = shard_range(r.size, world, k)
        shards.append((torch.from_numpy(r[lo:hi]), torch.from_numpy(c[lo:hi]),
                       torch.from_numpy(v[lo:hi])))
    res = convert_sharded_emulated(shards, plan, CpuOps())
    full = convert_sharded_emulated(shards, plan, CpuOps(), replicate=True)
    out = [(k, x.ti.numpy(), x.i1.numpy(), x.uniq.numpy(), x.rank, x.kept_offset,
            x.nkept_total, x.uniq_offset, f.uniq.numpy()) for k, (x, f) in enumerate(zip(res, full))]
    _check(out, world)


def test_sharded_conversion_empty_shard():
    """A rank with no entries (more ranks than useful) still joins every
    collective and the result is unchanged."""
    from paper_1707_07803_b200.distributed import convert_sharded_emulated
    r, c, v, plan = _input()
    e = torch.zeros(0, dtype=torch.int64)
    shards = [(torch.from_numpy(r), torch.from_numpy(c), torch.from_numpy(v)),
              (e, e, torch.zeros(0, dtype=torch.float64))]
    res = convert_sharded_emulated(shards, plan, CpuOps(), replicate=True)
    ref = orc.conversion_structure(r, c, v, plan.row_factors, plan.col_factors)
    assert np.array_equal(res[0].ti.numpy(), ref.ti)
    assert res[1].ti.numel() == 0 and np.array_equal(res[1].uniq.numpy(), ref.uniq)

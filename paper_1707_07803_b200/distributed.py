"""Multi-GPU sparse -> MPO conversion: nonzeros sharded over ranks, one
exchange step.

Each rank converts a contiguous shard of the COO entries locally
(convert.cu: split, key, radix sort, segment) and obtains its sorted
unique block keys.  The only collective is an all-gather of those keys
(NCCL over NVLink/NVSwitch on the GPU box; gloo in the CPU tests); every
rank then forms the global sorted unique key list with the same device
radix sort and maps its local block ids to global ones by binary search.
Because shards are contiguous ranges of the input order, concatenating the
per-rank (i1, j1, ti, values) reproduces the single-device / reference
arrays exactly (sparse.py:247 ``np.unique(..., return_inverse=True)``).

The per-rank primitives are injected (``ops``) so that the exchange logic
runs unchanged under gloo on CPU tensors in the tests.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from math import prod

import numpy as np

from . import _lib
from .partition import PartitionPlan

__all__ = ["ShardResult", "DeviceOps", "convert_sharded", "shard_range"]


@dataclass
class ShardResult:
    i1: object        # this rank's kept entries, input order
    j1: object
    ti: object        # GLOBAL block ids
    values: object
    uniq: object      # global sorted unique block keys (replicated)
    rank: int         # global nonzero block count (MPO interior rank)
    kept_offset: int  # position of this shard's first kept entry globally
    nkept_total: int


def shard_range(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous nnz shard [lo, hi) of rank ``rank``."""
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


class DeviceOps:
    """Per-rank primitives on the current CUDA device (C-ABI kernels);
    tensors are torch CUDA int64 / float64 tensors (plumbing only)."""

    def __init__(self, device=None):
        import torch
        self.torch = torch
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        self.ctx = _lib.context(self.device.index)

    def local(self, row1, col1, val, plan: PartitionPlan):
        torch = self.torch
        rf = _lib.as_i64(plan.row_factors)
        cf = _lib.as_i64(plan.col_factors)
        h = C.c_void_p()
        n = int(row1.numel())
        _lib.call("mpo_sparse_convert", self.ctx, C.c_void_p(row1.data_ptr()),
                  C.c_void_p(col1.data_ptr()), C.c_void_p(val.data_ptr()), n, 0, plan.d,
                  rf.ctypes.data_as(_lib._I64P), cf.ctypes.data_as(_lib._I64P), C.byref(h))
        try:
            nk, rk = C.c_int64(), C.c_int64()
            _lib.check(_lib.load().mpo_conv_info(h, C.byref(nk), C.byref(rk)))
            nk, rk = nk.value, rk.value
            i64 = dict(dtype=torch.int64, device=self.device)
            i1 = torch.empty(nk, **i64); j1 = torch.empty(nk, **i64); ti = torch.empty(nk, **i64)
            v = torch.empty(nk, dtype=torch.float64, device=self.device)
            u = torch.empty(rk, **i64)
            _lib.call("mpo_conv_copy", self.ctx, h, C.c_void_p(i1.data_ptr()),
                      C.c_void_p(j1.data_ptr()), C.c_void_p(ti.data_ptr()),
                      C.c_void_p(v.data_ptr()), C.c_void_p(u.data_ptr()), 0)
        finally:
            _lib.load().mpo_conv_free(h)
        return i1, j1, ti, v, u

    def unique(self, keys, max_key: int):
        out = self.torch.empty_like(keys)
        nu = C.c_int64()
        _lib.call("mpo_keys_unique", self.ctx, C.c_void_p(keys.data_ptr()), int(keys.numel()),
                  int(max_key), C.c_void_p(out.data_ptr()), C.byref(nu))
        return out[: nu.value]

    def lookup(self, table, q):
        out = self.torch.empty_like(q)
        _lib.call("mpo_keys_lookup", self.ctx, C.c_void_p(table.data_ptr()), int(table.numel()),
                  C.c_void_p(q.data_ptr()), int(q.numel()), C.c_void_p(out.data_ptr()))
        return out

    def remap(self, mapping, ti):
        _lib.call("mpo_remap_ids", self.ctx, C.c_void_p(mapping.data_ptr()),
                  C.c_void_p(ti.data_ptr()), int(ti.numel()))
        return ti


def convert_sharded(row1, col1, val, plan: PartitionPlan, ops, group=None) -> ShardResult:
    """Convert this rank's contiguous shard; one all-gather merges the block
    keys.  ``row1``/``col1``/``val`` are this rank's entries (1-based)."""
    import torch
    import torch.distributed as dist

    i1, j1, ti, values, uniq = ops.local(row1, col1, val, plan)
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    max_key = prod(plan.row_factors[1:]) * prod(plan.col_factors[1:]) - 1
    if world == 1:
        return ShardResult(i1, j1, ti, values, uniq, int(uniq.numel()), 0, int(ti.numel()))
    dev = uniq.device
    meta = torch.tensor([uniq.numel(), ti.numel()], dtype=torch.int64, device=dev)
    metas = [torch.empty_like(meta) for _ in range(world)]
    dist.all_gather(metas, meta, group=group)
    counts = [int(m[0]) for m in metas]
    kept = [int(m[1]) for m in metas]
    me = dist.get_rank(group)
    width = max(max(counts), 1)
    padded = torch.full((width,), -1, dtype=torch.int64, device=dev)
    padded[: uniq.numel()] = uniq
    bufs = [torch.empty_like(padded) for _ in range(world)]
    dist.all_gather(bufs, padded, group=group)
    allkeys = torch.cat([b[:c] for b, c in zip(bufs, counts)])
    merged = ops.unique(allkeys, max_key)
    mapping = ops.lookup(merged, uniq)
    ti = ops.remap(mapping, ti)
    return ShardResult(i1, j1, ti, values, merged, int(merged.numel()), sum(kept[:me]), sum(kept))

"""Multi-GPU sparse -> MPO conversion: nonzeros sharded over ranks, block
keys exchanged by key range (option (b)).

Reference: ``matrix_to_mpo`` (/root/reference/pkg/src/mposvd/sparse.py:207-258),
whose parity-critical step is ``np.unique(key, return_inverse=True)``
(sparse.py:247) over ALL nonzeros.  Here each rank owns a contiguous range
of the input entries and:

1. converts its shard locally (convert.cu: split, key, radix sort, segment)
   -> local sorted unique block keys ``u`` and local block ids ``ti``;
2. contributes 256 evenly spaced samples of ``u``; one all-gather of the
   samples gives every rank the same ``world - 1`` key splitters;
3. cuts ``u`` at the splitters (binary search) and sends each piece to the
   rank owning that key range (one variable-size all-to-all of keys);
4. merges what it received (sorted unique, O(blocks / world)), so rank r
   holds exactly the global unique keys of its key range, in global order;
   one all-gather of the per-range counts gives its global id offset;
5. answers, for every key it received, the global block id (binary search
   + offset) and returns the answers along the reverse all-to-all; the
   origin rank remaps its ``ti`` through them.

No rank ever handles the whole key set: per-rank work is O(nnz/world +
blocks/world + world * 256).  Because shards are contiguous ranges of the
input order and key ranges are contiguous ranges of the sorted key order,
concatenating the per-rank (i1, j1, ti, values) in rank order reproduces the
reference's arrays exactly, and concatenating the per-rank ``uniq`` shards
reproduces its ``uniq`` (sparse.py:247).

The algorithm is written once, as a per-rank generator that yields its
collective requests (``_rank_steps``); ``convert_sharded`` services them
with torch.distributed (NCCL over NVLink/NVSwitch on the GPU box, gloo in the
CPU tests) and ``convert_sharded_emulated`` runs ``world`` shards in lock
step on one device, servicing the same requests by list operations (the
single-GPU test of the exchange).  The per-rank primitives are injected
(``ops``): ``DeviceOps`` calls the C-ABI kernels.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass
from math import prod

from . import _lib
from .partition import PartitionPlan

__all__ = ["ShardResult", "Entries", "DeviceOps", "convert_sharded", "convert_sharded_emulated",
           "shard_range", "SAMPLES_PER_RANK"]

SAMPLES_PER_RANK = 256


@dataclass
class ShardResult:
    entries: object     # this rank's kept entries (input order): .i1, .j1, .values
    ti: object          # GLOBAL block ids
    uniq: object        # the global sorted unique block keys of this rank's key range
                        # (all of them when replicate=True)
    uniq_offset: int    # global block id of uniq[0]
    rank: int           # global nonzero block count (MPO interior rank)
    kept_offset: int    # position of this shard's first kept entry globally
    nkept_total: int

    # per-entry arrays: derived on first access on the device path (they are
    # the input's in-block offsets and values, sparse.py:241-242, 236)
    i1 = property(lambda self: self.entries.i1)
    j1 = property(lambda self: self.entries.j1)
    values = property(lambda self: self.entries.values)


class Entries:
    """Plain (i1, j1, values) holder (CPU stand-ins, tests)."""

    def __init__(self, i1, j1, values):
        self.i1, self.j1, self.values = i1, j1, values


class _DevView:
    """Zero-copy view of a buffer owned by a conversion handle (CUDA array
    interface); keeps the owner alive while torch tensors reference it."""

    def __init__(self, ptr, n, typestr, owner):
        self.owner = owner
        self.__cuda_array_interface__ = {"shape": (int(n),), "typestr": typestr,
                                         "data": (int(ptr), False), "version": 3,
                                         "strides": None}


class _ConvHandle:
    def __init__(self, h):
        self.h = h

    def __del__(self):
        try:
            if self.h is not None and self.h.value:
                _lib.load().mpo_conv_free(self.h)
        except Exception:  # pragma: no cover - interpreter shutdown
            pass
        self.h = None


class _LazyEntries:
    """i1, j1, values of a device conversion, fetched (and, without explicit
    zeros, derived from the input) only when first read."""

    def __init__(self, ops, handle, n):
        self._ops, self._h, self._n, self._t = ops, handle, n, None

    def _get(self):
        if self._t is None:
            ptrs = [C.c_void_p() for _ in range(3)]
            _lib.call("mpo_conv_ptrs", self._ops.ctx, self._h.h, C.byref(ptrs[0]),
                      C.byref(ptrs[1]), None, C.byref(ptrs[2]), None)
            self._t = (self._ops.view(ptrs[0], self._n, "<i8", self._h),
                       self._ops.view(ptrs[1], self._n, "<i8", self._h),
                       self._ops.view(ptrs[2], self._n, "<f8", self._h))
        return self._t

    i1 = property(lambda self: self._get()[0])
    j1 = property(lambda self: self._get()[1])
    values = property(lambda self: self._get()[2])


def shard_range(n: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous nnz shard [lo, hi) of rank ``rank``."""
    base, extra = divmod(n, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


class DeviceOps:
    """Per-rank primitives on a CUDA device (C-ABI kernels); tensors are torch
    CUDA int64 / float64 tensors (plumbing only)."""

    def __init__(self, device=None):
        import torch
        self.torch = torch
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None else device)
        self.ctx = _lib.context(self.device.index)

    def view(self, ptr, n, typestr, owner):
        torch = self.torch
        if n == 0 or not ptr.value:
            dt = {"<i8": torch.int64, "<f8": torch.float64}[typestr]
            return torch.empty(0, dtype=dt, device=self.device)
        return torch.as_tensor(_DevView(ptr.value, n, typestr, owner), device=self.device)

    def local(self, row1, col1, val, plan: PartitionPlan):
        """Device conversion of one shard; returns (entries, ti, uniq) with ti
        and uniq zero-copy views of the handle's buffers.  row1/col1/val must
        stay alive while the entries may still be read (derived from them)."""
        rf = _lib.as_i64(plan.row_factors)
        cf = _lib.as_i64(plan.col_factors)
        h = C.c_void_p()
        n = int(row1.numel())
        _lib.call("mpo_sparse_convert", self.ctx, C.c_void_p(row1.data_ptr()),
                  C.c_void_p(col1.data_ptr()), C.c_void_p(val.data_ptr()), n, 0, plan.d,
                  rf.ctypes.data_as(_lib._I64P), cf.ctypes.data_as(_lib._I64P), C.byref(h))
        owner = _ConvHandle(h)
        owner.inputs = (row1, col1, val)   # the lazily derived entries read them
        nk, rk = C.c_int64(), C.c_int64()
        _lib.check(_lib.load().mpo_conv_info(h, C.byref(nk), C.byref(rk)))
        pt, pu = C.c_void_p(), C.c_void_p()
        _lib.call("mpo_conv_ptrs", self.ctx, h, None, None, C.byref(pt), None, C.byref(pu))
        ti = self.view(pt, nk.value, "<i8", owner)
        u = self.view(pu, rk.value, "<i8", owner)
        return _LazyEntries(self, owner, nk.value), ti, u

    def unique(self, keys, max_key: int):
        out = self.torch.empty_like(keys)
        nu = C.c_int64()
        _lib.call("mpo_keys_unique", self.ctx, C.c_void_p(keys.data_ptr()), int(keys.numel()),
                  int(max_key), C.c_void_p(out.data_ptr()), C.byref(nu))
        return out[: nu.value]

    def search(self, table, q, offset: int = 0, exact: bool = False):
        """offset + lower_bound(table, q) (-1 where absent when exact)."""
        out = self.torch.empty_like(q)
        _lib.call("mpo_keys_search", self.ctx, C.c_void_p(table.data_ptr()), int(table.numel()),
                  C.c_void_p(q.data_ptr()), int(q.numel()), int(offset), int(bool(exact)),
                  C.c_void_p(out.data_ptr()))
        return out

    def remap(self, mapping, ti):
        _lib.call("mpo_remap_ids", self.ctx, C.c_void_p(mapping.data_ptr()),
                  C.c_void_p(ti.data_ptr()), int(ti.numel()))
        return ti


def _rank_steps(row1, col1, val, plan: PartitionPlan, ops, world: int, me: int,
                replicate: bool):
    """One rank's side of the sharded conversion.  Yields collective
    requests and receives their results:

    ("all_gather", t)              -> list of every rank's t (same shape)
    ("all_to_all", t, send, recv)  -> concatenation of the pieces sent to me
    ("all_gather_v", t, counts)    -> list of every rank's t (sizes counts)
    """
    import torch
    entries, ti, u = ops.local(row1, col1, val, plan)
    max_key = prod(plan.row_factors[1:]) * prod(plan.col_factors[1:]) - 1
    nloc = int(u.numel())
    dev = u.device
    # (2) samples -> common splitters
    s = SAMPLES_PER_RANK
    if nloc:
        pos = ((torch.arange(s, dtype=torch.float64, device=dev) + 0.5) * (nloc / s)).long()
        samples = u[pos.clamp_(max=nloc - 1)]
    else:
        samples = torch.full((s,), -1, dtype=torch.int64, device=dev)
    gathered = yield ("all_gather", samples)
    allsamp = torch.cat(gathered)
    allsamp = allsamp[allsamp >= 0]
    srt = ops.unique(allsamp.contiguous(), max_key) if allsamp.numel() else allsamp
    m = int(srt.numel())
    if m:
        pick = torch.tensor([(r * m) // world for r in range(1, world)], dtype=torch.int64,
                            device=dev)
        splitters = srt[pick].contiguous()
    else:
        splitters = torch.full((world - 1,), max_key + 1, dtype=torch.int64, device=dev)
    # (3) cut the local keys at the splitters, exchange counts then keys
    cuts = ops.search(u, splitters).cpu().tolist() if world > 1 else []
    bounds = [0] + cuts + [nloc]
    send = [bounds[r + 1] - bounds[r] for r in range(world)]
    meta = torch.tensor(send + [int(ti.numel())], dtype=torch.int64, device=dev)
    metas = yield ("all_gather", meta)
    metas = [x.cpu().tolist() for x in metas]
    recv = [metas[src][me] for src in range(world)]
    kept = [metas[src][world] for src in range(world)]
    got = yield ("all_to_all", u, send, recv)
    # (4) the global unique keys of my key range; global offset
    mine = ops.unique(got, max_key) if got.numel() else got
    cnt = torch.tensor([int(mine.numel())], dtype=torch.int64, device=dev)
    counts = [int(x.item()) for x in (yield ("all_gather", cnt))]
    offset = sum(counts[:me])
    # (5) global ids of the keys I received, back to their origin ranks
    ids = ops.search(mine, got, offset, exact=True) if got.numel() else got
    mapping = yield ("all_to_all", ids, recv, send)
    ti = ops.remap(mapping, ti) if ti.numel() else ti
    uniq, uoff = mine, offset
    if replicate:
        parts = yield ("all_gather_v", mine, counts)
        uniq, uoff = torch.cat(parts), 0
    return ShardResult(entries, ti, uniq, uoff, sum(counts), sum(kept[:me]), sum(kept))


def convert_sharded(row1, col1, val, plan: PartitionPlan, ops, group=None,
                    replicate: bool = False) -> ShardResult:
    """Convert this rank's contiguous shard (1-based ``row1``/``col1``,
    ``val``) with the key-range exchange over torch.distributed."""
    import torch
    import torch.distributed as dist
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    me = dist.get_rank(group) if dist.is_initialized() else 0
    if world == 1:
        entries, ti, u = ops.local(row1, col1, val, plan)
        return ShardResult(entries, ti, u, 0, int(u.numel()), 0, int(ti.numel()))
    gen = _rank_steps(row1, col1, val, plan, ops, world, me, replicate)
    res = None
    while True:
        try:
            req = gen.send(res)
        except StopIteration as fin:
            return fin.value
        kind, t = req[0], req[1]
        if kind == "all_gather":
            out = [torch.empty_like(t) for _ in range(world)]
            dist.all_gather(out, t.contiguous(), group=group)
            res = out
        elif kind == "all_to_all":
            send, recv = req[2], req[3]
            out = torch.empty(sum(recv), dtype=t.dtype, device=t.device)
            dist.all_to_all_single(out, t.contiguous(), output_split_sizes=recv,
                                   input_split_sizes=send, group=group)
            res = out
        elif kind == "all_gather_v":
            counts = req[2]
            width = max(max(counts), 1)
            padded = torch.zeros(width, dtype=t.dtype, device=t.device)
            padded[: t.numel()] = t
            out = [torch.empty_like(padded) for _ in range(world)]
            dist.all_gather(out, padded, group=group)
            res = [o[:c] for o, c in zip(out, counts)]
        else:  # pragma: no cover
            raise RuntimeError(f"unknown collective {kind}")


def convert_sharded_emulated(shards, plan: PartitionPlan, ops, replicate: bool = False):
    """Run ``len(shards)`` ranks' conversions in lock step on one device,
    servicing their collective requests with list operations (same per-rank
    code path as convert_sharded; the single-GPU test of the exchange).
    ``shards`` = [(row1, col1, val), ...] in rank order."""
    import torch
    world = len(shards)
    gens = [_rank_steps(r, c, v, plan, ops, world, me, replicate)
            for me, (r, c, v) in enumerate(shards)]
    results = [None] * world
    done = [None] * world
    while True:
        reqs = []
        for me, g in enumerate(gens):
            try:
                reqs.append(g.send(results[me]))
            except StopIteration as fin:
                done[me] = fin.value
                reqs.append(None)
        if all(r is None for r in reqs):
            return done
        assert all(r is not None for r in reqs), "ranks diverged"
        kind = reqs[0][0]
        if kind in ("all_gather", "all_gather_v"):
            ts = [r[1] for r in reqs]
            results = [list(ts) for _ in range(world)]
        elif kind == "all_to_all":
            pieces = []
            for r in reqs:
                t, send = r[1], r[2]
                offs = [0]
                for x in send:
                    offs.append(offs[-1] + x)
                pieces.append([t[offs[k]:offs[k + 1]] for k in range(world)])
            results = [torch.cat([pieces[src][dst] for src in range(world)])
                       for dst in range(world)]
        else:  # pragma: no cover
            raise RuntimeError(f"unknown collective {kind}")

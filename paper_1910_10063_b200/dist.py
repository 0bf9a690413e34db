"""Multi-GPU orchestration of the hot path: one process per GPU, fact rows
sharded with the reference's own partition (``chunk_spans``,
proj/src/parallel.cpp:31-43), dimension columns replicated, and the real
exchange steps as collectives:

* index build (config 4): per-GPU u32 histogram -> all-reduce SUM -> every
  rank runs the same deterministic sort (no broadcast needed);
* group-by (config 3): per-GPU count/sum partials -> reduce SUM to a root
  (the reference's fold of private arrays, parallel.cpp:155-157), shipped in
  the packed combine layout (8 B per tail key instead of 16) whenever a
  16-byte guard all-reduce proves the packed fields cannot overflow;
* selection (config 5): no row exchange -- a shard's offsets carry its first
  row as ``base`` (scalar.cpp:38), so the shard concatenation in rank order
  is parallel_select's order (parallel.cpp:102-129) -- and the per-category
  sums are combined EXACTLY: the 96-bit fixed-point limbs are reduced as
  int64 and converted to fp64 once, on the root;
* gather: no exchange; the output stays row-sharded.

Errors keep the reference's semantics across shards: the first out-of-domain
row of the WHOLE column (operators.cpp:32-41) is found by all-gathering each
shard's first violation (as a global row), and every rank raises the same
DomainViolation -- no rank is left blocked in a collective.

The per-shard compute is an *executor*: ``GpuExecutor`` calls the sm_100a
kernels through libskx; tests substitute a CPU executor (the oracle).  The
collectives are a *Collectives* object: ``SkxCollectives`` is libskx's own
NCCL communicator (skx_comm_init_rank, include/skx.h) on the executor's
stream -- the path bench.py runs on N GPUs; ``TorchCollectives`` is
torch.distributed (gloo on CPU for the world-size-2 tests, or NCCL);
``Single`` is the one-GPU no-op.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch
import torch.distributed as dist

from . import _native
from .errors import DomainViolation, Error
from .skewdx import chunk_spans

INT64_MAX = (1 << 63) - 1
SUM, MIN, MAX = _native.OP_SUM, _native.OP_MIN, _native.OP_MAX
# group-by combine layout: ids 1..GROUPBY_HOT travel as u64 pairs, the tail packed
GROUPBY_HOT = 1 << 16


@dataclass
class Shard:
    rank: int
    world: int
    begin: int
    end: int

    @property
    def rows(self) -> int:
        return self.end - self.begin


def shard_for(n_rows: int, rank: int | None = None, world: int | None = None) -> Shard:
    """This rank's contiguous span of the fact table (chunk_spans order)."""
    if world is None:
        world = dist.get_world_size() if dist.is_initialized() else 1
    if rank is None:
        rank = dist.get_rank() if dist.is_initialized() else 0
    b, e = chunk_spans(n_rows, world)[rank]
    return Shard(rank, world, b, e)


# ---------------------------------------------------------------------------
# collectives
# ---------------------------------------------------------------------------
class Single:
    """One rank: every collective is the identity."""
    world, rank = 1, 0

    def allreduce(self, t, op=SUM):
        return t

    def reduce(self, t, root=0, op=SUM):
        return t

    def allgather(self, t):
        return t.clone()

    def barrier(self):
        pass


_TORCH_OP = {SUM: "SUM", MIN: "MIN", MAX: "MAX"}
_SIGNED = {torch.uint32: torch.int32, torch.uint64: torch.int64, torch.uint16: torch.int16}


def _signed(t):
    # u32/u64 SUM wraps exactly like i32/i64 two's complement; MIN/MAX are only
    # used on non-negative int64 values
    return t.view(_SIGNED[t.dtype]) if t.dtype in _SIGNED else t


class TorchCollectives:
    """torch.distributed (gloo on CPU tensors, or NCCL on CUDA tensors).  With
    gloo, CUDA tensors are staged through host memory (the one-GPU dry run)."""

    def __init__(self):
        self.world, self.rank = dist.get_world_size(), dist.get_rank()
        self.gloo = dist.get_backend() != "nccl"

    def _host(self, t):
        return t.cpu() if (self.gloo and t.is_cuda) else t

    def allreduce(self, t, op=SUM):
        h = self._host(t)
        dist.all_reduce(_signed(h), op=getattr(dist.ReduceOp, _TORCH_OP[op]))
        if h is not t:
            t.copy_(h)
        return t

    def reduce(self, t, root=0, op=SUM):
        if not self.gloo:
            dist.reduce(_signed(t), dst=root, op=getattr(dist.ReduceOp, _TORCH_OP[op]))
            return t
        # gloo: an all-reduce leaves the root's result identical to a reduce
        return self.allreduce(t, op)

    def allgather(self, t):
        h = self._host(t)
        parts = [torch.empty_like(_signed(h)) for _ in range(self.world)]
        dist.all_gather(parts, _signed(h).contiguous())
        return torch.cat(parts).view(t.dtype).to(t.device)

    def barrier(self):
        dist.barrier()


_DT = {torch.uint32: _native.DT_U32, torch.int32: _native.DT_I32, torch.uint64: _native.DT_U64,
       torch.int64: _native.DT_I64, torch.float64: _native.DT_F64}


class SkxCollectives:
    """libskx's NCCL communicator (one device of a process-per-GPU job):
    collectives are enqueued on the current torch stream, i.e. in order with
    the kernels of the same step."""

    def __init__(self, device: int, world: int, rank: int, unique_id: bytes):
        self.lib = _native.load()
        self.world, self.rank, self.device = world, rank, device
        h = C.c_void_p()
        idb = C.create_string_buffer(bytes(unique_id), 128)
        st = self.lib.skx_comm_init_rank(device, world, rank, idb, C.byref(h))
        if st != _native.OK:
            raise Error(f"skx_comm_init_rank failed (status {st})")
        self.handle = h

    @staticmethod
    def from_process_group(device: int) -> "SkxCollectives":
        """Rank 0 creates the NCCL unique id; torch.distributed ships it."""
        lib = _native.load()
        obj = [None]
        if dist.get_rank() == 0:
            buf = C.create_string_buffer(128)
            if lib.skx_comm_unique_id(buf) != _native.OK:
                raise Error("skx_comm_unique_id failed")
            obj[0] = buf.raw
        dist.broadcast_object_list(obj, src=0)
        return SkxCollectives(device, dist.get_world_size(), dist.get_rank(), obj[0])

    def close(self):
        if getattr(self, "handle", None):
            self.lib.skx_comm_destroy(self.handle)
            self.handle = None

    def _check(self, st):
        if st != _native.OK:
            raise Error("NCCL: " + (self.lib.skx_comm_error(self.handle) or b"").decode())

    def _args(self, t):
        bufs = (C.c_void_p * 1)(t.data_ptr())
        strm = (C.c_void_p * 1)(torch.cuda.current_stream(self.device).cuda_stream)
        return bufs, strm

    def allreduce(self, t, op=SUM):
        b, s = self._args(t)
        self._check(self.lib.skx_allreduce(self.handle, b, t.numel(), _DT[t.dtype], op, s))
        return t

    def reduce(self, t, root=0, op=SUM):
        b, s = self._args(t)
        self._check(self.lib.skx_reduce(self.handle, b, t.numel(), _DT[t.dtype], op, root, s))
        return t

    def allgather(self, t):
        out = torch.empty(t.numel() * self.world, dtype=t.dtype, device=t.device)
        b, s = self._args(t)
        r = (C.c_void_p * 1)(out.data_ptr())
        self._check(self.lib.skx_allgather(self.handle, b, r, t.numel(), _DT[t.dtype], s))
        return out

    def barrier(self):
        dist.barrier()


def default_collectives(device: int | None = None):
    """Single for one rank; libskx NCCL when the process group is NCCL;
    torch.distributed otherwise (gloo)."""
    if not (dist.is_available() and dist.is_initialized()) or dist.get_world_size() == 1:
        return Single()
    if dist.get_backend() == "nccl":
        return SkxCollectives.from_process_group(
            torch.cuda.current_device() if device is None else device)
    return TorchCollectives()


# ---------------------------------------------------------------------------
# executor: per-shard compute on the local GPU (libskx), all asynchronous
# ---------------------------------------------------------------------------
class GpuExecutor:
    def __init__(self, ctx=None):
        from . import skewdx as sx
        self.sx = sx
        self.ctx = ctx or sx.context(torch.cuda.current_device())
        self.device = torch.device("cuda", self.ctx.device)

    def histogram_u32(self, fact, d, out=None):
        return self.sx.histogram_u32(fact, d, out, ctx=self.ctx, sync=False)

    def build_index(self, counts_u32, total):
        return self.sx.build_index(self.sx.FrequencyProfile(counts_u32, total), ctx=self.ctx,
                                   sync=False)

    def recode(self, fact, index, out=None):
        return self.sx.recode_fact(fact, index, out=out, ctx=self.ctx, sync=False)

    def permute(self, dim, index):
        return self.sx.permute_dimension(dim, index, ctx=self.ctx, sync=False)

    def gather(self, fact, dim, out=None):
        return self.sx.materialize(fact, dim, out=out, ctx=self.ctx, sync=False)

    def aggregate(self, fact, measure, d, counts=None, sums=None):
        return self.sx.aggregate_count_sum(fact, measure, d, ctx=self.ctx, sync=False,
                                           counts=counts, sums=sums)

    def groupby_pack(self, counts, sums, hot, buf=None, guard=None):
        d = counts.numel()
        buf = torch.empty(d + hot, dtype=torch.uint64, device=counts.device) if buf is None else buf
        guard = torch.empty(2, dtype=torch.uint64, device=counts.device) if guard is None else guard
        p = self.sx._ptr
        self.ctx.call("skx_groupby_pack", p(counts), p(sums), d, hot, p(buf), p(guard),
                      self.ctx.stream(), sync=False)
        return buf, guard

    def groupby_unpack(self, buf, d, hot, counts, sums):
        p = self.sx._ptr
        self.ctx.call("skx_groupby_unpack", p(buf), d, hot, p(counts), p(sums), self.ctx.stream(),
                      sync=False)

    def select_gather_sum(self, fact, bitmap, cols, n_categories, base, out):
        cat, price, supp, flag = cols
        return self.sx.select_gather_sum(fact, bitmap, cat, price, supp, flag, n_categories,
                                         base=base, ctx=self.ctx, sync=False, out=out)

    def sum_partials(self, n_categories, out=None):
        out = (torch.empty(2 + 3 * n_categories, dtype=torch.int64, device=self.device)
               if out is None else out)
        self.ctx.call("skx_select_sum_partials", n_categories, self.sx._ptr(out),
                      self.ctx.stream(), sync=False)
        return out

    def sums_from_partials(self, partials, n_categories, nranks, sums):
        self.ctx.call("skx_select_sums_from_partials", self.sx._ptr(partials), n_categories,
                      nranks, self.sx._ptr(sums), self.ctx.stream(), sync=False)

    def take_violation(self):
        """Waits for this shard's work; (local row, value) of its first
        out-of-domain row, or None.  Other deferred errors raise."""
        try:
            self.ctx.sync()
        except DomainViolation as e:
            return e.row(), e.value()
        return None

    @staticmethod
    def packed_ok(guard_sum) -> bool:
        g = guard_sum.cpu().view(torch.int64).numpy().view(np.uint64)
        return bool(g[0] < (1 << 24) and g[1] < (1 << 40))


# ---------------------------------------------------------------------------
# phase timing (CUDA events on the launching stream; None on CPU)
# ---------------------------------------------------------------------------
class PhaseTimer:
    """Records a CUDA event after each named phase of one step."""

    def __init__(self):
        self.events = [("start", torch.cuda.Event(enable_timing=True))]
        self.events[0][1].record()

    def mark(self, name):
        e = torch.cuda.Event(enable_timing=True)
        e.record()
        self.events.append((name, e))

    def phases_ms(self):
        torch.cuda.synchronize()
        out = {}
        for (_, a), (name, b) in zip(self.events, self.events[1:]):
            out[name] = out.get(name, 0.0) + a.elapsed_time(b)
        return out


def _mark(timer, name):
    if timer is not None:
        timer.mark(name)


# ---------------------------------------------------------------------------
# orchestration
# ---------------------------------------------------------------------------
def check_violations(ex, coll, shard: Shard, domain: int) -> None:
    """Raise, on EVERY rank, DomainViolation for the first out-of-domain row
    of the whole (sharded) column -- find_domain_violation's row,
    operators.cpp:32-41 -- after this shard's work completes."""
    v = ex.take_violation()
    if coll.world == 1:
        if v is not None:
            raise DomainViolation(shard.begin + v[0], v[1], domain)
        return
    mine = torch.tensor([shard.begin + v[0] if v else INT64_MAX, v[1] if v else 0],
                        dtype=torch.int64, device=ex.device)
    allv = coll.allgather(mine).view(-1, 2).cpu()
    k = int(torch.argmin(allv[:, 0]))
    row = int(allv[k, 0])
    if row != INT64_MAX:
        raise DomainViolation(row, int(allv[k, 1]), domain)


def rebuild(fact_shard, d: int, n_total: int, ex, coll=None, shard: Shard | None = None,
            counts=None, timer=None, check=True):
    """Distributed rebuild (permindex.cpp:86-88): local histogram, all-reduce,
    the identical deterministic sort on every rank.  Returns (index, counts)."""
    coll = coll or Single()
    shard = shard or Shard(coll.rank, coll.world, 0, int(fact_shard.numel()))
    counts = ex.histogram_u32(fact_shard, d, counts)
    _mark(timer, "histogram")
    if check:
        check_violations(ex, coll, shard, d)
    # u32 counters summed as wrapping integers: total rows <= 2^32-1 keeps
    # every count exact
    coll.allreduce(counts, SUM)
    _mark(timer, "allreduce")
    index = ex.build_index(counts, n_total)
    _mark(timer, "sort")
    return index, counts


def aggregate(fact_shard, measure_shard, d: int, ex, coll=None, shard: Shard | None = None,
              root: int = 0, packed: bool = True, hot: int = GROUPBY_HOT, counts=None,
              sums=None, timer=None, check=True, stats=None):
    """Distributed COUNT/SUM (operators.cpp:100-118 per shard; the fold of
    parallel.cpp:155-157 across shards) reduced to ``root``.  u64 sums wrap
    mod 2^64 like the reference's accumulators.  ``stats`` (a dict) receives
    the combine path taken and the bytes each rank sent."""
    coll = coll or Single()
    shard = shard or Shard(coll.rank, coll.world, 0, int(fact_shard.numel()))
    counts, sums = ex.aggregate(fact_shard, measure_shard, d, counts, sums)
    _mark(timer, "aggregate")
    if check:
        check_violations(ex, coll, shard, d)
    if coll.world == 1:
        return counts, sums
    if packed and d > hot:
        buf, guard = ex.groupby_pack(counts, sums, hot)
        coll.allreduce(guard, SUM)
        if ex.packed_ok(guard):
            coll.reduce(buf, root, SUM)
            if coll.rank == root:
                ex.groupby_unpack(buf, d, hot, counts, sums)
            _mark(timer, "reduce")
            if stats is not None:
                stats.update(path="packed", bytes=int(buf.numel()) * 8 + 16)
            return counts, sums
    coll.reduce(counts, root, SUM)
    coll.reduce(sums, root, SUM)
    _mark(timer, "reduce")
    if stats is not None:
        stats.update(path="pairs", bytes=int(counts.numel() + sums.numel()) * 8)
    return counts, sums


def select_gather_sum(fact_shard, bitmap, cols, n_categories: int, ex, coll=None,
                      shard: Shard | None = None, capacity: int | None = None, root: int = 0,
                      base: int | None = None, out=None, timer=None, check=True):
    """Config 5 on a shard: offsets (base = the shard's first row, so the
    rank-order concatenation is parallel_select's order), the four gathered
    columns, and per-category sums combined exactly across ranks (96-bit
    fixed-point limbs reduced as int64, converted once on ``root``; the fp64
    sums are reduced beside them for the device's fp64 fallback).
    Returns ex's output tuple (off, cat, price, supp, flag, sums, count)."""
    coll = coll or Single()
    shard = shard or Shard(coll.rank, coll.world, 0, int(fact_shard.numel()))
    base = shard.begin if base is None else base
    if out is None:
        m = max(int(fact_shard.numel() if capacity is None else capacity), 1)
        dev = fact_shard.device
        out = tuple(torch.empty(m, dtype=t, device=dev) for t in
                    (torch.uint32, torch.int32, torch.float32, torch.uint64, torch.uint16)) + (
            torch.empty(n_categories, dtype=torch.float64, device=dev),
            torch.zeros(1, dtype=torch.uint64, device=dev))
    out = ex.select_gather_sum(fact_shard, bitmap, cols, n_categories, base, out)
    _mark(timer, "select")
    if check:
        check_violations(ex, coll, shard, bitmap.size())
    if coll.world > 1:
        part = ex.sum_partials(n_categories)
        sums = out[5]
        coll.reduce(part, root, SUM)
        coll.reduce(sums, root, SUM)
        if coll.rank == root:
            ex.sums_from_partials(part, n_categories, coll.world, sums)
        _mark(timer, "reduce")
    return out


def gather(fact_shard, dim, ex, out=None):
    """Distributed materialize: no exchange, the output stays row-sharded."""
    return ex.gather(fact_shard, dim, out)


def concat_selection(local_offsets, coll, root: int = 0):
    """Shard selections concatenated in rank order on ``root`` (the order of
    parallel_select, parallel.cpp:122-128); other ranks get their own."""
    if coll.world == 1:
        return local_offsets
    n_local = torch.tensor([local_offsets.numel()], dtype=torch.int64,
                           device=local_offsets.device)
    sizes = coll.allgather(n_local).cpu()
    mx = int(sizes.max())
    padded = torch.zeros(max(mx, 1), dtype=torch.int64, device=local_offsets.device)
    padded[: local_offsets.numel()] = local_offsets.to(torch.int64)
    parts = coll.allgather(padded).view(coll.world, -1)
    if coll.rank != root:
        return local_offsets
    return torch.cat([parts[r, : int(sizes[r])] for r in range(coll.world)])

"""Multi-GPU orchestration of the hot path: one process per GPU, fact rows
sharded with the reference's own partition (``chunk_spans``,
proj/src/parallel.cpp:31-43), dimension columns replicated, and the two real
exchange steps done with torch.distributed collectives:

* index build (BASELINE config 4): per-GPU u32 histogram -> all-reduce ->
  every rank runs the same deterministic sort (no broadcast needed);
* group-by (BASELINE config 3): per-GPU u64 count/sum partials -> reduce to
  the root (the reference's fold of private arrays, parallel.cpp:155-157);
* gather / selection: no data exchange; a selection shard's offsets carry its
  first row as ``base`` (scalar.cpp:38), so concatenating shards in rank order
  is parallel_select's global order (parallel.cpp:122-128).

The per-shard compute is an *executor* object.  ``GpuExecutor`` calls the
sm_100a kernels through libskx; tests substitute a CPU executor (the oracle)
to exercise this host logic with world_size 2 over gloo on machines without
GPUs.  Collectives operate on the tensors the executor returns, so NCCL
(CUDA tensors) and gloo (CPU tensors) share one code path.
"""
from __future__ import annotations

from dataclasses import dataclass

import torch
import torch.distributed as dist

from .skewdx import chunk_spans


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


def _world() -> int:
    return dist.get_world_size() if dist.is_available() and dist.is_initialized() else 1


class GpuExecutor:
    """Per-shard compute on the local GPU (libskx)."""

    def __init__(self, ctx=None):
        from . import skewdx as sx
        self.sx = sx
        self.ctx = ctx

    def histogram_u32(self, fact, d):
        return self.sx.histogram_u32(fact, d, ctx=self.ctx)

    def build_index(self, counts_u32, total):
        return self.sx.build_index(self.sx.FrequencyProfile(counts_u32, total), ctx=self.ctx)

    def recode(self, fact, index):
        return self.sx.recode_fact(fact, index, ctx=self.ctx)

    def gather(self, fact, dim):
        return self.sx.materialize(fact, dim, ctx=self.ctx)

    def aggregate(self, fact, measure, d):
        return self.sx.aggregate_count_sum(fact, measure, d, ctx=self.ctx)

    def select(self, fact, bitmap, base):
        return self.sx.select(fact, bitmap, base=base, ctx=self.ctx)


def rebuild(fact_shard: torch.Tensor, d: int, n_total: int, ex) -> object:
    """Distributed rebuild (permindex.cpp:86-88): local histogram, all-reduce,
    identical deterministic sort on every rank."""
    counts = ex.histogram_u32(fact_shard, d)
    if _world() > 1:
        # u32 counters summed as i32: two's-complement wrap is identical, and
        # total rows <= 2^32-1 keeps every count exact.
        dist.all_reduce(counts.view(torch.int32), op=dist.ReduceOp.SUM)
    return ex.build_index(counts, n_total)


def aggregate(fact_shard, measure_shard, d: int, ex, root: int = 0):
    """Distributed COUNT/SUM: per-shard partials reduced to ``root`` (u64
    sums wrap mod 2^64 exactly like the reference's accumulators)."""
    counts, sums = ex.aggregate(fact_shard, measure_shard, d)
    if _world() > 1:
        dist.reduce(counts.view(torch.int64), dst=root, op=dist.ReduceOp.SUM)
        dist.reduce(sums.view(torch.int64), dst=root, op=dist.ReduceOp.SUM)
    return counts, sums


def select(fact_shard, bitmap, shard: Shard, ex, gather_to: int | None = 0):
    """Distributed selection: local offsets carry ``base = shard.begin``;
    optionally gathered to one rank and concatenated in rank order."""
    local = ex.select(fact_shard, bitmap, shard.begin)
    if _world() == 1 or gather_to is None:
        return local
    n_local = torch.tensor([local.numel()], dtype=torch.int64, device=local.device)
    sizes = [torch.zeros_like(n_local) for _ in range(_world())]
    dist.all_gather(sizes, n_local)
    mx = int(max(int(s.item()) for s in sizes))
    padded = torch.zeros(max(mx, 1), dtype=torch.int64, device=local.device)
    padded[: local.numel()] = local.to(torch.int64)
    parts = [torch.zeros_like(padded) for _ in range(_world())]
    dist.all_gather(parts, padded)
    if dist.get_rank() != gather_to:
        return local
    return torch.cat([p[: int(s.item())] for p, s in zip(parts, sizes)])


def gather(fact_shard, dim, ex):
    """Distributed materialize: no exchange, the output stays row-sharded."""
    return ex.gather(fact_shard, dim)

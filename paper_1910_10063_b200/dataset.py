"""Synthetic BASELINE workloads built on the device (the B200 counterpart of
the reference bench's dataset builder, proj/tools/benchcli/dataset.cpp:30-54).

A workload is carried in both layouts like ``BenchDataset``
(dataset.hpp:20-44): ``rand`` -- Zipf ranks scattered over ids by the seeded
random bijection (column.cpp:62-71) -- and ``freq`` -- the same rows recoded
through the permutation index built from them, with the dimension columns
permuted (dataset.cpp:30-43: rebuild, recode_fact, permute_dimension).

Each GPU materialises only its own shard of fact rows (``chunk_spans``,
parallel.cpp:31-43); the counter-based generator makes any row range
reproducible independently.  Dimension columns are replicated.
"""
from __future__ import annotations

import ctypes as C
import time
from dataclasses import dataclass, field

import numpy as np
import torch

from . import skewdx as sx

KIND_RAW, KIND_UNIFORM, KIND_LOGNORMAL = 0, 1, 2
GAMMA = 0x9E3779B97F4A7C15  # splitmix64 increment: fill_column kind 1 keys row i by seed + i*GAMMA
SEED = 42


@dataclass(frozen=True)
class Workload:
    """One BASELINE.json config: domain D, total fact rows N, Zipf s, seed."""
    name: str
    d: int
    n: int
    z: float
    seed: int


# BASELINE.json configs[0..4] at their stated sizes (bench.py and the
# BASELINE-scale parity tests build exactly these).
C1 = Workload("C1 FK-join gather (Q1 shape)", 1 << 22, 1 << 24, 1.0, SEED + 7)
C2 = Workload("C2 large FK-join gather", 1 << 27, 1 << 30, 1.0, SEED)
C3 = Workload("C3 group-by COUNT+SUM", 1 << 24, 1 << 30, 1.0, SEED + 1)
C4 = Workload("C4 index build at scale", 1 << 26, 1 << 30, 1.25, SEED + 9)
C5 = Workload("C5 multi-column FK join with selection", 1 << 25, 1 << 31, 1.0, SEED + 12)


def fill_column(kind: int, dtype: torch.dtype, n: int, seed: int, p0: float = 0.0,
                p1: float = 0.0, device="cuda", ctx=None) -> torch.Tensor:
    out = torch.empty(int(n), dtype=dtype, device=device)
    ctx = ctx or sx.context(out.device.index)
    w = out.element_size()
    ctx.call("skx_fill_column", int(kind), w, int(seed) & (2**64 - 1), int(n), float(p0),
             float(p1), C.c_void_p(out.data_ptr()), ctx.stream(), sync=False)
    return out


@dataclass
class Shard:
    rank: int
    world: int
    begin: int
    end: int

    @property
    def rows(self) -> int:
        return self.end - self.begin


def shard_of(n: int, rank: int = 0, world: int = 1) -> Shard:
    b, e = sx.chunk_spans(n, world)[rank]
    return Shard(rank, world, b, e)


@dataclass
class GatherDataset:
    """Q1 workload: fact FK shard in both layouts plus one value column."""
    d: int
    n: int
    z: float
    seed: int
    shard: Shard
    fact_rand: torch.Tensor
    fact_freq: torch.Tensor
    dim_rand: torch.Tensor
    dim_freq: torch.Tensor
    index: sx.PermutationIndex
    timings_ms: dict = field(default_factory=dict)

    def fact(self, layout: str) -> torch.Tensor:
        return self.fact_rand if layout == "rand" else self.fact_freq

    def dim(self, layout: str) -> torch.Tensor:
        return self.dim_rand if layout == "rand" else self.dim_freq


def _allreduce_u32(t: torch.Tensor) -> None:
    import torch.distributed as dist
    if dist.is_available() and dist.is_initialized() and dist.get_world_size() > 1:
        dist.all_reduce(t.view(torch.int32), op=dist.ReduceOp.SUM)  # u32 wrap == i32 wrap


def make_rand_fact(d: int, n: int, z: float, seed: int, shard: Shard, device="cuda"):
    """Zipf(z) draws over ranks, rank -> id by random_bijection(d, seed)."""
    cdf = torch.from_numpy(sx.zipf_cdf(d, z)).to(device)
    r2i = torch.from_numpy(sx.random_bijection(d, seed)).to(device)
    fact = sx.generate_zipf(cdf, shard.rows, seed, rank_to_id=r2i, row_begin=shard.begin,
                            sync=False)
    del cdf, r2i
    return fact


def build_index_sharded(fact_shard: torch.Tensor, d: int, n_total: int, ctx=None):
    """Index build at scale (BASELINE config 4): per-GPU u32 histogram of the
    local shard -> NCCL all-reduce -> the same deterministic sort on every GPU."""
    counts = sx.histogram_u32(fact_shard, d, ctx=ctx, sync=False)
    _allreduce_u32(counts)
    return sx.build_index(sx.FrequencyProfile(counts, n_total), ctx=ctx, sync=False)


def make_gather_dataset(d: int, n: int, z: float, seed: int, value_dtype=torch.int64,
                        shard: Shard | None = None, device="cuda") -> GatherDataset:
    shard = shard or shard_of(n)
    ctx = sx.context(torch.device(device).index or 0)
    t = {}
    t0 = time.perf_counter()
    fact_rand = make_rand_fact(d, n, z, seed, shard, device)
    torch.cuda.synchronize()
    t["generate_s"] = time.perf_counter() - t0
    # dimension value column: splitmix64(seed ^ (0xd1000000 + i)) (dataset.cpp:35-38)
    dim_rand = fill_column(KIND_RAW, value_dtype, d, seed, device=device)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
    ev[0].record()
    index = build_index_sharded(fact_rand, d, n, ctx)
    ev[1].record()
    fact_freq = sx.recode_fact(fact_rand, index, sync=False)
    ev[2].record()
    dim_freq = sx.permute_dimension(dim_rand, index, sync=False)
    ev[3].record()
    ctx.sync()
    t["index_build_ms"] = ev[0].elapsed_time(ev[1])
    t["recode_ms"] = ev[1].elapsed_time(ev[2])
    t["permute_ms"] = ev[2].elapsed_time(ev[3])
    return GatherDataset(d, n, z, seed, shard, fact_rand, fact_freq, dim_rand, dim_freq, index, t)


@dataclass
class GroupByDataset:
    """Q3 workload (BASELINE config 3): recoded FK shard + int64 quantity."""
    d: int
    n: int
    shard: Shard
    fact_freq: torch.Tensor
    qty: torch.Tensor


def make_groupby_dataset(d: int, n: int, z: float, seed: int, shard: Shard | None = None,
                         device="cuda") -> GroupByDataset:
    shard = shard or shard_of(n)
    ctx = sx.context(torch.device(device).index or 0)
    fact_rand = make_rand_fact(d, n, z, seed, shard, device)
    index = build_index_sharded(fact_rand, d, n, ctx)
    fact_freq = sx.recode_fact(fact_rand, index, sync=False)
    del fact_rand, index
    # quantity uniform 1..100 (int64), keyed by the GLOBAL row number, so any
    # sharding of the rows sees the same values
    qty = fill_column(KIND_UNIFORM, torch.int64, shard.rows, qty_seed(seed, shard.begin), 1, 100,
                      device=device)
    ctx.sync()
    return GroupByDataset(d, n, shard, fact_freq, qty)


def qty_seed(seed: int, row_begin: int) -> int:
    """fill_column kind-1 seed whose local row i is global row row_begin + i."""
    return (seed * 1000003 + row_begin * GAMMA) & (2**64 - 1)


@dataclass
class C1Dataset:
    """configs[0]: D=2^22 int32 price (uniform 1..10^6), 2^24 FKs, s=1.0."""
    g: GatherDataset
    price: torch.Tensor
    price_freq: torch.Tensor


def make_c1_dataset(shard: Shard | None = None, w: Workload = C1) -> C1Dataset:
    shard = shard or shard_of(w.n)
    g = make_gather_dataset(w.d, w.n, w.z, w.seed, torch.int32, shard)
    price = fill_column(KIND_UNIFORM, torch.int32, w.d, w.seed + 1, 1, 1000000)
    price_f = sx.permute_dimension(price, g.index, sync=False)
    return C1Dataset(g, price, price_f)


@dataclass
class IndexBuildDataset:
    """configs[3]: the original-layout FK shard and the two dimension columns
    (int32, float32) the index build permutes."""
    d: int
    n: int
    shard: Shard
    fact: torch.Tensor
    dim_i: torch.Tensor
    dim_f: torch.Tensor


def make_index_build_dataset(shard: Shard | None = None, w: Workload = C4) -> IndexBuildDataset:
    shard = shard or shard_of(w.n)
    fact = make_rand_fact(w.d, w.n, w.z, w.seed, shard)
    dim_i = fill_column(KIND_RAW, torch.int32, w.d, w.seed + 1)
    dim_f = fill_column(KIND_RAW, torch.int32, w.d, w.seed + 2).view(torch.float32)
    return IndexBuildDataset(w.d, w.n, shard, fact, dim_i, dim_f)


@dataclass
class SelectDataset:
    """configs[4]: recoded FK shard; category int32 (uniform 0..999), price
    float32 (lognormal mu=3 sigma=1), supplier int64, flag int16 -- all in the
    reordered (rank) layout -- and the bitmap of category < 100."""
    d: int
    n: int
    shard: Shard
    fact: torch.Tensor
    index: sx.PermutationIndex
    cat: torch.Tensor
    price: torch.Tensor
    supp: torch.Tensor
    flag: torch.Tensor
    bitmap: sx.Bitmap


def make_select_dataset(shard: Shard | None = None, w: Workload = C5) -> SelectDataset:
    shard = shard or shard_of(w.n)
    ctx = sx.context(torch.cuda.current_device())
    fact = make_rand_fact(w.d, w.n, w.z, w.seed, shard)
    index = build_index_sharded(fact, w.d, w.n, ctx)
    fact_f = sx.recode_fact(fact, index, sync=False)
    del fact
    cat = sx.permute_dimension(fill_column(KIND_UNIFORM, torch.int32, w.d, w.seed + 1, 0, 1000),
                               index, sync=False)
    price = sx.permute_dimension(fill_column(KIND_LOGNORMAL, torch.float32, w.d, w.seed + 2, 3.0,
                                             1.0), index, sync=False)
    supp = sx.permute_dimension(fill_column(KIND_RAW, torch.int64, w.d, w.seed + 3), index,
                                sync=False)
    flag = sx.permute_dimension(fill_column(KIND_RAW, torch.int16, w.d, w.seed + 4), index,
                                sync=False)
    bm = sx.build_bitmap_lt(cat, 100, sync=False)  # category < 100, already in rank space
    ctx.sync()
    return SelectDataset(w.d, w.n, shard, fact_f, index, cat, price, supp, flag, bm)


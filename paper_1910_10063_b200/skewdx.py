"""Host-side mirror of the reference operator API over libskx.so.

Same names, argument meaning and error behaviour as the reference's C++ API
(proj/include/skewdx/permindex.hpp:34-59, operators.hpp:57-122,
parallel.hpp:34-61), with columns held as CUDA tensors (resident in HBM)
instead of host ``std::vector``s:

=====================================  ======================================
reference (skewdx::)                   here
=====================================  ======================================
Column (std::vector<uint32_t>)         1-D ``torch.uint32`` CUDA tensor
count_frequencies(fact, D)             ``count_frequencies(fact, D)``
build_index(profile)                   ``build_index(profile)``
recode_fact / permute_dimension        ``recode_fact`` / ``permute_dimension``
rebuild(fact, D)                       ``rebuild(fact, D)``
materialize(fact, dim)                 ``materialize(fact, dim)``
select(fact, bitmap)                   ``select(fact, bitmap)``
aggregate_count / aggregate_sum        ``aggregate_count`` / ``aggregate_sum``
parallel_aggregate(fact, D, plan)      ``parallel_aggregate(fact, D, plan)``
heavy_hitter_count(fact, D, k)         ``heavy_hitter_count(fact, D, k)``
permute_bitmap(bitmap, index)          ``permute_bitmap(bitmap, index)``
=====================================  ======================================

Every call enqueues on the current torch stream and then synchronises on it
so that a DomainViolation / InvalidArgument is raised by the call that
caused it, as in the reference.  Pass ``sync=False`` to keep the call
asynchronous (errors then surface at the next ``Context.sync()``).
"""
from __future__ import annotations

import ctypes as C
import enum
import threading
from dataclasses import dataclass

import numpy as np
import torch

from . import _native
from .errors import DomainViolation, Error, InvalidArgument, NativeUnavailable

MAX_DOMAIN_CARDINALITY = 0xFFFFFFFE  # column.hpp:17

_WIDTH = {torch.uint16: 2, torch.int16: 2, torch.uint32: 4, torch.int32: 4, torch.float32: 4,
          torch.uint64: 8, torch.int64: 8, torch.float64: 8}


# ---------------------------------------------------------------------------
# Context
# ---------------------------------------------------------------------------
class Context:
    """One libskx context per (host thread, device); owns device scratch."""

    def __init__(self, device: int = 0):
        if not torch.cuda.is_available():
            raise NativeUnavailable("no CUDA device: libskx has no CPU fallback")
        self.lib = _native.load()
        self.device = int(device)
        h = C.c_void_p()
        with torch.cuda.device(self.device):
            st = self.lib.skx_ctx_create(self.device, C.byref(h))
        if st != 0:
            raise NativeUnavailable(f"skx_ctx_create(device={device}) failed with status {st}")
        self.handle = h

    def close(self):
        if getattr(self, "handle", None):
            self.lib.skx_ctx_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001
            pass

    def stream(self):
        return C.c_void_p(torch.cuda.current_stream(self.device).cuda_stream)

    def check(self, status: int) -> None:
        if status != _native.OK:
            info = _native.ErrorInfo()
            self.lib.skx_last_error(self.handle, C.byref(info))
            _native.raise_for(status, info)

    def sync(self, stream=None) -> None:
        """Wait for the stream and raise any deferred device-side error."""
        self.check(self.lib.skx_sync(self.handle, stream if stream is not None else self.stream()))

    def launches(self) -> int:
        return int(self.lib.skx_launch_count(self.handle))

    def set_gather_policy(self, policy: int) -> None:
        self.check(self.lib.skx_set_gather_policy(self.handle, policy))

    def gather_last_plan(self, stream=None) -> dict:
        """The last gather launch of this context (include/skx.h, policy bit
        8192): the path it took, its column's plan and the plan's sample."""
        info = (C.c_uint32 * 4)()
        self.check(self.lib.skx_gather_last_plan(
            self.handle, info, stream if stream is not None else self.stream()))
        return {"partitioned": bool(info[0]), "plan_partitioned": bool(info[3]),
                "sample_first_touch": int(info[1]), "sample_ascending_pairs": int(info[2]),
                "sample_rows": 65536}

    def call(self, name: str, *args, sync: bool = True):
        self.check(getattr(self.lib, name)(self.handle, *args))
        if sync:
            self.sync()


_tls = threading.local()


def context(device: int | None = None) -> Context:
    if device is None:
        device = torch.cuda.current_device()
    ctxs = getattr(_tls, "ctxs", None)
    if ctxs is None:
        ctxs = _tls.ctxs = {}
    if device not in ctxs:
        ctxs[device] = Context(device)
    return ctxs[device]


# ---------------------------------------------------------------------------
# helpers
# ---------------------------------------------------------------------------
def _ptr(t: torch.Tensor | None):
    return C.c_void_p(t.data_ptr()) if t is not None else None


def _col(fact: torch.Tensor, name: str = "fact") -> torch.Tensor:
    if not isinstance(fact, torch.Tensor) or not fact.is_cuda:
        raise InvalidArgument(f"{name} must be a CUDA tensor")
    if fact.dim() != 1:
        raise InvalidArgument(f"{name} must be 1-D")
    if fact.dtype == torch.int32:
        fact = fact.view(torch.uint32)
    if fact.dtype != torch.uint32:
        raise InvalidArgument(f"{name} must hold uint32 identifiers, got {fact.dtype}")
    return fact.contiguous()


def _values(dim: torch.Tensor, name: str = "dim") -> torch.Tensor:
    if not isinstance(dim, torch.Tensor) or not dim.is_cuda or dim.dim() != 1:
        raise InvalidArgument(f"{name} must be a 1-D CUDA tensor")
    if dim.dtype not in _WIDTH:
        raise InvalidArgument(f"{name}: unsupported dtype {dim.dtype}")
    return dim.contiguous()


def _ctx_for(t: torch.Tensor, ctx: Context | None) -> Context:
    return ctx if ctx is not None else context(t.device.index)


# ---------------------------------------------------------------------------
# permindex.hpp
# ---------------------------------------------------------------------------
@dataclass
class FrequencyProfile:
    """permindex.hpp:14-17: counts indexed by identifier - 1, and their total."""
    counts: torch.Tensor  # uint64[D]
    total: int


@dataclass
class PermutationIndex:
    """permindex.hpp:23-30: offsets (rank -> id) and ranks (id -> rank)."""
    offsets: torch.Tensor  # uint32[D]
    ranks: torch.Tensor  # uint32[D]

    def domain_cardinality(self) -> int:
        return int(self.offsets.numel())


def count_frequencies(fact, domain_cardinality: int, *, ctx=None, sync=True) -> FrequencyProfile:
    """permindex.cpp:18-30; raises DomainViolation naming the first bad row."""
    fact = _col(fact)
    ctx = _ctx_for(fact, ctx)
    d = int(domain_cardinality)
    counts = torch.empty(d, dtype=torch.uint64, device=fact.device)
    ctx.call("skx_count_frequencies", _ptr(fact), fact.numel(), d, _ptr(counts), ctx.stream(),
             sync=sync)
    return FrequencyProfile(counts, int(fact.numel()))


def histogram_u32(fact, domain_cardinality: int, counts=None, *, accumulate=False, ctx=None,
                  sync=True) -> torch.Tensor:
    """u32 per-shard histogram (the partial that is all-reduced across GPUs)."""
    fact = _col(fact)
    ctx = _ctx_for(fact, ctx)
    d = int(domain_cardinality)
    if counts is None:
        counts = torch.empty(d, dtype=torch.uint32, device=fact.device)
    ctx.call("skx_histogram_u32", _ptr(fact), fact.numel(), d, _ptr(counts), int(accumulate),
             ctx.stream(), sync=sync)
    return counts


def build_index(profile: FrequencyProfile, *, ctx=None, sync=True) -> PermutationIndex:
    """permindex.cpp:32-58: offsets sorted by (count desc, id asc); ranks = inverse."""
    counts = profile.counts
    if not counts.is_cuda:
        counts = counts.cuda()
    ctx = _ctx_for(counts, ctx)
    d = counts.numel()
    if d > MAX_DOMAIN_CARDINALITY:
        raise InvalidArgument("frequency profile exceeds the 32-bit identifier space")
    offsets = torch.empty(d, dtype=torch.uint32, device=counts.device)
    ranks = torch.empty(d, dtype=torch.uint32, device=counts.device)
    if counts.dtype in (torch.uint32, torch.int32):
        ctx.call("skx_build_index_u32", _ptr(counts.contiguous()), d, int(profile.total),
                 _ptr(offsets), _ptr(ranks), ctx.stream(), sync=sync)
    else:
        ctx.call("skx_build_index", _ptr(counts.contiguous()), d, int(profile.total),
                 _ptr(offsets), _ptr(ranks), ctx.stream(), sync=sync)
    return PermutationIndex(offsets, ranks)


def rebuild(fact, domain_cardinality: int, *, ctx=None, sync=True) -> PermutationIndex:
    """permindex.cpp:86-88: count_frequencies followed by build_index."""
    fact = _col(fact)
    ctx = _ctx_for(fact, ctx)
    d = int(domain_cardinality)
    offsets = torch.empty(d, dtype=torch.uint32, device=fact.device)
    ranks = torch.empty(d, dtype=torch.uint32, device=fact.device)
    ctx.call("skx_rebuild", _ptr(fact), fact.numel(), d, _ptr(offsets), _ptr(ranks), ctx.stream(),
             sync=sync)
    return PermutationIndex(offsets, ranks)


def recode_fact(fact, index: PermutationIndex, *, out=None, ctx=None, sync=True) -> torch.Tensor:
    """permindex.cpp:60-64: out[k] = ranks[fact[k]-1]."""
    fact = _col(fact)
    ctx = _ctx_for(fact, ctx)
    if out is None:
        out = torch.empty_like(fact)
    ctx.call("skx_recode_fact", _ptr(fact), fact.numel(), _ptr(index.ranks),
             index.domain_cardinality(), _ptr(out), ctx.stream(), sync=sync)
    return out


def permute_dimension(dim, index: PermutationIndex, *, ctx=None, sync=True) -> torch.Tensor:
    """permindex.cpp:66-73: out[r] = dim[offsets[r]-1]; length must match."""
    dim = _values(dim)
    ctx = _ctx_for(dim, ctx)
    w = _WIDTH[dim.dtype]
    out = torch.empty_like(dim)
    ctx.call(f"skx_permute_dimension_u{8 * w}", _ptr(dim), dim.numel(), _ptr(index.offsets),
             index.domain_cardinality(), _ptr(out), ctx.stream(), sync=sync)
    return out


# ---------------------------------------------------------------------------
# operators.hpp
# ---------------------------------------------------------------------------
class Bitmap:
    """operators.hpp:17-36: packed little-endian predicate bits over 1..D."""

    def __init__(self, size: int, words: torch.Tensor | None = None, device=None):
        self._size = int(size)
        nw = (self._size + 63) // 64
        if words is None:
            words = torch.zeros(nw, dtype=torch.uint64, device=device or "cuda")
        if words.numel() != nw:
            raise InvalidArgument("bitmap word count does not match its size")
        self.words = words

    def size(self) -> int:
        return self._size

    def count(self) -> int:
        w = self.words.cpu().numpy().view(np.uint8)
        return int(np.unpackbits(w).sum())

    @staticmethod
    def from_numpy(words: np.ndarray, size: int, device="cuda") -> "Bitmap":
        return Bitmap(size, torch.from_numpy(np.ascontiguousarray(words, np.uint64)).to(device))


def build_bitmap_lt(dim_values, threshold: int, *, ctx=None, sync=True) -> Bitmap:
    """build_bitmap(dim, v < threshold) (operators.hpp:38-45) for an int32 column."""
    dim = _values(dim_values)
    if dim.dtype not in (torch.int32, torch.uint32):
        raise InvalidArgument("build_bitmap_lt needs a 32-bit integer column")
    ctx = _ctx_for(dim, ctx)
    bm = Bitmap(dim.numel(), device=dim.device)
    ctx.call("skx_build_bitmap_lt_i32", _ptr(dim), dim.numel(), int(threshold), _ptr(bm.words),
             ctx.stream(), sync=sync)
    return bm


def permute_bitmap(bitmap: Bitmap, index: PermutationIndex, *, ctx=None, sync=True) -> Bitmap:
    """operators.cpp:21-30: out bit r = input bit of the id holding rank r+1."""
    ctx = _ctx_for(bitmap.words, ctx)
    out = Bitmap(bitmap.size(), device=bitmap.words.device)
    ctx.call("skx_permute_bitmap", _ptr(bitmap.words), bitmap.size(), _ptr(index.offsets),
             index.domain_cardinality(), _ptr(out.words), ctx.stream(), sync=sync)
    return out


def materialize(fact, dim, *, out=None, ctx=None, sync=True) -> torch.Tensor:
    """Q1, operators.cpp:60-66: out[k] = dim[fact[k]-1] (any 2/4/8-byte dtype)."""
    fact = _col(fact)
    dim = _values(dim)
    ctx = _ctx_for(fact, ctx)
    if out is None:
        out = torch.empty(fact.numel(), dtype=dim.dtype, device=fact.device)
    w = _WIDTH[dim.dtype]
    ctx.call(f"skx_gather_u{8 * w}", _ptr(fact), fact.numel(), _ptr(dim), dim.numel(), _ptr(out),
             ctx.stream(), sync=sync)
    return out


def materialize_split(fact, dim, threshold: int, *, out=None, ctx=None, sync=True) -> torch.Tensor:
    """operators.cpp:68-85: the same result as materialize, computed in two
    passes split on the rank threshold t (ids <= t first, then the misses)."""
    fact = _col(fact)
    dim = _values(dim)
    ctx = _ctx_for(fact, ctx)
    w = _WIDTH[dim.dtype]
    if w not in (4, 8):
        raise InvalidArgument("materialize_split: 32- or 64-bit values")
    if out is None:
        out = torch.empty(fact.numel(), dtype=dim.dtype, device=fact.device)
    ctx.call(f"skx_gather_split_u{8 * w}", _ptr(fact), fact.numel(), _ptr(dim), dim.numel(),
             int(threshold), _ptr(out), ctx.stream(), sync=sync)
    return out


def select(fact, bitmap: Bitmap, *, base: int = 0, ctx=None) -> torch.Tensor:
    """Q2, operators.cpp:87-98: ascending 0-based row offsets whose bit is set."""
    fact = _col(fact)
    ctx = _ctx_for(fact, ctx)
    n = fact.numel()
    if n > 0xFFFFFFFF:
        raise InvalidArgument("select: fact row offsets exceed 32 bits")
    out = torch.empty(max(n, 1), dtype=torch.uint32, device=fact.device)
    cnt = torch.zeros(1, dtype=torch.uint64, device=fact.device)
    ctx.call("skx_select_offsets", _ptr(fact), n, _ptr(bitmap.words), bitmap.size(), int(base),
             _ptr(out), _ptr(cnt), ctx.stream(), sync=True)
    return out[: int(cnt.item())]


def aggregate_count(fact, domain_cardinality: int, *, hot_threshold: int = 0, ctx=None,
                    sync=True) -> torch.Tensor:
    """Q3, operators.cpp:100-105: counts[i] = occurrences of id i+1 (uint64)."""
    fact = _col(fact)
    ctx = _ctx_for(fact, ctx)
    d = int(domain_cardinality)
    counts = torch.empty(d, dtype=torch.uint64, device=fact.device)
    ctx.call("skx_aggregate", _ptr(fact), None, 0, fact.numel(), d, int(hot_threshold),
             _ptr(counts), None, ctx.stream(), sync=sync)
    return counts


def aggregate_count_sum(fact, measure, domain_cardinality: int, *, hot_threshold: int = 0,
                        ctx=None, sync=True, counts=None, sums=None):
    """COUNT and SUM(measure) per key in one pass (BASELINE config 3).

    measure: uint32/int32 (the reference's Column) or uint64/int64 (int64 qty).
    Returns (counts, sums) as uint64 tensors; integer sums wrap mod 2^64 as in
    the reference's std::uint64_t accumulators.
    """
    fact = _col(fact)
    measure = _values(measure, "measure")
    if measure.numel() != fact.numel():
        raise InvalidArgument("aggregate_sum: measure length does not match fact length")
    mw = _WIDTH[measure.dtype]
    if mw not in (4, 8) or measure.dtype.is_floating_point:
        raise InvalidArgument("aggregate: measure must be a 32- or 64-bit integer column")
    ctx = _ctx_for(fact, ctx)
    d = int(domain_cardinality)
    if counts is None:
        counts = torch.empty(d, dtype=torch.uint64, device=fact.device)
    if sums is None:
        sums = torch.empty(d, dtype=torch.uint64, device=fact.device)
    ctx.call("skx_aggregate", _ptr(fact), _ptr(measure), mw, fact.numel(), d, int(hot_threshold),
             _ptr(counts), _ptr(sums), ctx.stream(), sync=sync)
    return counts, sums


def aggregate_sum(fact, measure, domain_cardinality: int, **kw) -> torch.Tensor:
    """Q3 over a measure column, operators.cpp:107-118."""
    return aggregate_count_sum(fact, measure, domain_cardinality, **kw)[1]


@dataclass
class HeavyHitters:
    """operators.hpp:87-93: (id, count) by count desc then id asc; clamped flag."""
    top: list
    clamped: bool = False


def heavy_hitter_count(fact, domain_cardinality: int, k: int, *, ctx=None) -> HeavyHitters:
    """Q3a, operators.cpp:184-203: counts of ids 1..k of a recoded column."""
    if k == 0:
        raise InvalidArgument("heavy_hitter_count: k must be at least 1")
    fact = _col(fact)
    ctx = _ctx_for(fact, ctx)
    d = int(domain_cardinality)
    cutoff = min(k, d)
    counts = torch.empty(max(cutoff, 1), dtype=torch.uint64, device=fact.device)
    ctx.call("skx_heavy_hitter_count", _ptr(fact), fact.numel(), d, int(k), _ptr(counts),
             ctx.stream(), sync=True)
    c = counts[:cutoff].cpu().numpy()
    # order_heavy_hitters (operators.cpp:169-182): count desc, then id asc
    top = sorted(((i + 1, int(c[i])) for i in range(cutoff)), key=lambda t: (-t[1], t[0]))
    return HeavyHitters(top, k > d)


# ---------------------------------------------------------------------------
# parallel.hpp
# ---------------------------------------------------------------------------
class AggStrategy(enum.IntEnum):
    independent = 0
    shared_atomic = 1
    hybrid = 2


@dataclass
class ParallelPlan:
    """parallel.hpp:23-30.  On the GPU every strategy runs the same smem-hot +
    global-tail kernel; hot_threshold sizes the shared-memory region."""
    threads: int = 1
    strategy: AggStrategy = AggStrategy.independent
    hot_threshold: int = 8192
    pin_threads: bool = False


def chunk_spans(n: int, threads: int):
    """parallel.cpp:31-43: contiguous near-equal spans; first n%T get +1."""
    if threads == 0:
        raise InvalidArgument("thread count must be at least 1")
    base, extra = divmod(int(n), int(threads))
    spans, b = [], 0
    for t in range(threads):
        ln = base + (1 if t < extra else 0)
        spans.append((b, b + ln))
        b += ln
    return spans


def parallel_materialize(fact, dim, plan: ParallelPlan | None = None, **kw):
    """parallel.cpp:87-100 -- one GPU already runs the whole column in parallel."""
    return materialize(fact, dim, **kw)


def parallel_select(fact, bitmap: Bitmap, plan: ParallelPlan | None = None, **kw):
    """parallel.cpp:102-129 -- ascending order, identical to select."""
    return select(fact, bitmap, **kw)


def parallel_aggregate(fact, domain_cardinality: int, plan: ParallelPlan | None = None, **kw):
    """parallel.cpp:131-216 (COUNT).  Validates the hybrid threshold like the
    reference (:135-138); results are identical for every strategy."""
    plan = plan or ParallelPlan()
    if plan.threads == 0:
        raise InvalidArgument("thread count must be at least 1")
    if plan.strategy == AggStrategy.hybrid and not (1 <= plan.hot_threshold <= domain_cardinality):
        raise InvalidArgument("hybrid hot threshold must lie in 1..D")
    hot = plan.hot_threshold if plan.strategy == AggStrategy.hybrid else 0
    return aggregate_count(fact, domain_cardinality, hot_threshold=hot, **kw)


# ---------------------------------------------------------------------------
# column.hpp generator (parallel, counter-based)
# ---------------------------------------------------------------------------
def zipf_cdf(domain_cardinality: int, z: float) -> np.ndarray:
    """zipf_frequencies + partial_sum, cdf[-1] = 1.0 (column.cpp:44-60,77-79), host."""
    lib = _native.load()
    d = int(domain_cardinality)
    out = np.empty(d, np.float64)
    if lib.skx_zipf_cdf_host(d, float(z), out.ctypes.data_as(C.c_void_p)) != 0:
        raise InvalidArgument("zipf spec: invalid domain cardinality or exponent")
    return out


def random_bijection(n: int, seed: int) -> np.ndarray:
    """column.cpp:62-71 (mt19937_64 Fisher-Yates), host, bit-identical."""
    lib = _native.load()
    out = np.empty(int(n), np.uint32)
    lib.skx_random_bijection_host(int(n), int(seed) & (2**64 - 1), out.ctypes.data_as(C.c_void_p))
    return out


def generate_zipf(cdf: torch.Tensor, n: int, seed: int, *, rank_to_id: torch.Tensor | None = None,
                  row_begin: int = 0, out: torch.Tensor | None = None, ctx=None,
                  sync=True) -> torch.Tensor:
    """Rows [row_begin, row_begin+n) of the counter-based Zipf FK column."""
    if not cdf.is_cuda or cdf.dtype != torch.float64:
        raise InvalidArgument("cdf must be a float64 CUDA tensor")
    ctx = _ctx_for(cdf, ctx)
    if out is None:
        out = torch.empty(int(n), dtype=torch.uint32, device=cdf.device)
    ctx.call("skx_generate_zipf", _ptr(cdf), cdf.numel(), _ptr(rank_to_id),
             int(seed) & (2**64 - 1), int(row_begin), int(n), _ptr(out), ctx.stream(), sync=sync)
    return out


def select_gather_sum(fact, bitmap: Bitmap, cat, price, supp, flag, n_categories: int, *,
                      base: int = 0, capacity: int | None = None, ctx=None, sync=True,
                      out=None):
    """BASELINE config 5 fused: selected offsets, the 4 gathered columns and
    per-category fp64 SUM(price).

    ``capacity`` sizes the output columns (default: every row).  When more
    rows are selected than fit, the call is repeated with exactly-sized
    outputs, so the result is always complete.  ``out`` = (off, cat, price,
    supp, flag, sums, count) preallocated device tensors (then ``sync=False``
    keeps the call asynchronous and the caller reads ``count``)."""
    fact = _col(fact)
    ctx = _ctx_for(fact, ctx)
    n = fact.numel()
    dev = fact.device
    if out is None:
        m = max(int(n if capacity is None else capacity), 1)
        out = (torch.empty(m, dtype=torch.uint32, device=dev),
               torch.empty(m, dtype=torch.int32, device=dev),
               torch.empty(m, dtype=torch.float32, device=dev),
               torch.empty(m, dtype=torch.uint64, device=dev),
               torch.empty(m, dtype=torch.uint16, device=dev),
               torch.empty(int(n_categories), dtype=torch.float64, device=dev),
               torch.zeros(1, dtype=torch.uint64, device=dev))
    o_off, o_cat, o_pr, o_su, o_fl, sums, cnt = out
    cap = o_off.numel()
    ctx.call("skx_select_gather_sum", _ptr(fact), n, _ptr(bitmap.words), bitmap.size(),
             _ptr(cat), _ptr(price), _ptr(supp), _ptr(flag), int(base), int(n_categories), cap,
             _ptr(o_off), _ptr(o_cat), _ptr(o_pr), _ptr(o_su), _ptr(o_fl), _ptr(sums), _ptr(cnt),
             ctx.stream(), sync=sync)
    if not sync:
        return out
    c = int(cnt.item())
    if c > cap:  # too small: once more with exactly-sized outputs
        return select_gather_sum(fact, bitmap, cat, price, supp, flag, n_categories, base=base,
                                 capacity=c, ctx=ctx)
    return o_off[:c], o_cat[:c], o_pr[:c], o_su[:c], o_fl[:c], sums


# ---------------------------------------------------------------------------
# Cache model (cachemodel.hpp)
# ---------------------------------------------------------------------------
class Layout(enum.IntEnum):
    """column.hpp Layout: rand = ranks scattered by random_bijection, freq = in place."""
    rand = 0
    freq = 1


@dataclass
class CacheGeometry:
    """cachemodel.hpp:14-22."""
    lines: int = 1
    line_bytes: int = 64
    element_bytes: int = 4

    def elements_per_line(self) -> int:
        return self.line_bytes // self.element_bytes

    def validate(self):
        if self.lines == 0:
            raise InvalidArgument("cache geometry: line count must be at least 1")
        if self.element_bytes == 0 or self.line_bytes == 0 or self.line_bytes % self.element_bytes:
            raise InvalidArgument("cache geometry: line bytes must be a multiple of element bytes")


@dataclass
class LruStats:
    """cachemodel.hpp:46-66."""
    accesses: int = 0
    hits: int = 0
    distinct_lines: int = 0

    def hit_rate(self) -> float:
        return 0.0 if self.accesses == 0 else self.hits / self.accesses

    def steady_hit_rate(self, cache_lines: int) -> float:
        fill = min(self.distinct_lines, cache_lines)
        denom = self.accesses - fill
        return 0.0 if denom == 0 else self.hits / denom


def line_frequencies(value_freqs: torch.Tensor, layout: Layout, geometry: CacheGeometry,
                     seed: int, *, ctx=None, sync=True) -> torch.Tensor:
    """cachemodel.cpp:22-45 on the device: per-line access frequencies of a
    float64 per-rank frequency vector (bit-identical to the reference)."""
    geometry.validate()
    if not value_freqs.is_cuda or value_freqs.dtype != torch.float64:
        raise InvalidArgument("value_freqs must be a float64 CUDA tensor")
    d = value_freqs.numel()
    if d == 0:
        raise InvalidArgument("line_frequencies: empty frequency vector")
    ctx = _ctx_for(value_freqs, ctx)
    per = geometry.elements_per_line()
    out = torch.empty((d + per - 1) // per, dtype=torch.float64, device=value_freqs.device)
    r2i = None
    if Layout(layout) == Layout.rand:
        r2i = torch.from_numpy(random_bijection(d, seed)).to(value_freqs.device)
    ctx.call("skx_line_frequencies", _ptr(value_freqs.contiguous()), d, _ptr(r2i), per, _ptr(out),
             ctx.stream(), sync=sync)
    return out


def estimate_hit_rate(line_freqs: torch.Tensor, cache_lines: int, *, ctx=None) -> float:
    """cachemodel.cpp:76-123 on the device (the reference to rounding)."""
    if cache_lines == 0:
        raise InvalidArgument("estimate_hit_rate: cache must have at least 1 line")
    if not line_freqs.is_cuda or line_freqs.dtype != torch.float64:
        raise InvalidArgument("line_freqs must be a float64 CUDA tensor")
    ctx = _ctx_for(line_freqs, ctx)
    res = torch.empty(1, dtype=torch.float64, device=line_freqs.device)
    ctx.call("skx_estimate_hit_rate", _ptr(line_freqs.contiguous()), line_freqs.numel(),
             int(cache_lines), _ptr(res), ctx.stream(), sync=True)
    return float(res.item())


def trace_from_column(fact: torch.Tensor, geometry: CacheGeometry, *, ctx=None,
                      sync=True) -> torch.Tensor:
    """cachemodel.cpp:175-186 on the device: 0-based line ids of a 1-based FK column."""
    geometry.validate()
    fact = _col(fact)
    ctx = _ctx_for(fact, ctx)
    out = torch.empty(fact.numel(), dtype=torch.uint32, device=fact.device)
    ctx.call("skx_trace_from_column", _ptr(fact), fact.numel(), geometry.elements_per_line(),
             _ptr(out), ctx.stream(), sync=sync)
    return out


def simulate_lru(trace, cache_lines: int) -> LruStats:
    """cachemodel.cpp:125-173: exact sequential LRU over a trace (host)."""
    if cache_lines == 0:
        raise InvalidArgument("simulate_lru: cache must have at least 1 line")
    t = trace.cpu().numpy() if isinstance(trace, torch.Tensor) else np.asarray(trace)
    t = np.ascontiguousarray(t, dtype=np.uint32)
    st = np.zeros(3, np.uint64)
    lib = _native.load()
    if lib.skx_simulate_lru_host(t.ctypes.data_as(C.c_void_p), len(t), int(cache_lines),
                                 st.ctypes.data_as(C.c_void_p)) != 0:
        raise InvalidArgument("simulate_lru: invalid arguments")
    return LruStats(int(st[0]), int(st[1]), int(st[2]))


__all__ = [
    "Layout", "CacheGeometry", "LruStats", "line_frequencies", "estimate_hit_rate",
    "trace_from_column", "simulate_lru",
    "Context", "context", "FrequencyProfile", "PermutationIndex", "count_frequencies",
    "histogram_u32", "build_index", "rebuild", "recode_fact", "permute_dimension", "Bitmap",
    "build_bitmap_lt", "permute_bitmap", "materialize", "select", "aggregate_count",
    "aggregate_count_sum", "aggregate_sum", "HeavyHitters", "heavy_hitter_count", "AggStrategy",
    "ParallelPlan", "chunk_spans", "parallel_materialize", "parallel_select", "parallel_aggregate",
    "zipf_cdf", "random_bijection", "generate_zipf", "select_gather_sum", "DomainViolation",
    "InvalidArgument", "Error",
]

"""ctypes bindings for the parity checkers (TEST INFRASTRUCTURE ONLY).

Two checkers live here:

* ``Oracle`` -- the C restatement in ``skx_oracle.c`` (``liboracle.so``), each
  function citing the reference file:line it follows;
* ``Reference`` -- the unmodified reference library compiled from
  ``/root/reference/proj/src`` into ``oracle/_ref/libskewdx_ref.so`` with our
  ``ref_capi.cpp`` bridge.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU-baseline
leg may import this module.  The product package ``paper_1910_10063_b200``
never does.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "liboracle.so")
REF_SO = os.path.join(HERE, "_ref", "libskewdx_ref.so")

OK, INVALID, DOMAIN = 0, 1, 2


class OracleError(Exception):
    def __init__(self, status, row=None, value=None):
        super().__init__(f"status {status} row={row} value={value}")
        self.status, self.row, self.value = status, row, value


def build(ref: bool = True) -> None:
    """Build liboracle.so (and the reference .so when its sources exist)."""
    targets = ["oracle"]
    if ref and os.path.isdir("/root/reference/proj/src"):
        targets.append("ref")
        if os.path.exists(os.path.join(HERE, "..", "paper_1910_10063_b200", "libskewdx_b200.so")):
            targets.append("refsuite")
    subprocess.check_call(["make", "-s", "-C", HERE, *targets])


def _p(a):
    return a.ctypes.data_as(C.c_void_p) if a is not None else None


def _u32(a):
    return np.ascontiguousarray(a, dtype=np.uint32)


def _u64(a):
    return np.ascontiguousarray(a, dtype=np.uint64)


class _Err:
    def __init__(self):
        self.row = C.c_uint64(0)
        self.value = C.c_uint32(0)

    def args(self):
        return C.byref(self.row), C.byref(self.value)

    def check(self, st):
        if st == DOMAIN:
            raise OracleError(st, self.row.value, self.value.value)
        if st != OK:
            raise OracleError(st)


class Oracle:
    """C restatement of the reference hot path (skx_oracle.c)."""

    def __init__(self, path: str = ORACLE_SO):
        if not os.path.exists(path):
            build(ref=False)
        L = self.L = C.CDLL(path)
        vp, u64, u32, dbl = C.c_void_p, C.c_uint64, C.c_uint32, C.c_double
        L.orc_splitmix64.restype = u64
        L.orc_splitmix64.argtypes = [u64]
        L.orc_zipf_frequencies.argtypes = [u32, dbl, vp]
        L.orc_zipf_cdf.argtypes = [u32, dbl, vp]
        L.orc_random_bijection.argtypes = [u32, u64, vp]
        L.orc_generate_fact_column_rand.argtypes = [u32, u64, dbl, u64, vp, vp]
        L.orc_generate_zipf_counter.argtypes = [vp, u32, vp, u64, u64, u64, vp]
        L.orc_generate_zipf_counter_mt.argtypes = [vp, u32, vp, u64, u64, vp, u32]
        L.orc_find_domain_violation.restype = u64
        L.orc_find_domain_violation.argtypes = [vp, u64, u64]
        L.orc_count_frequencies.argtypes = [vp, u64, u32, vp, vp, vp]
        L.orc_build_index.argtypes = [vp, u32, u64, vp, vp]
        for w in ("u16", "u32", "u64"):
            getattr(L, f"orc_gather_{w}").argtypes = [vp, u64, vp, u64, vp, vp, vp]
            getattr(L, f"orc_permute_dimension_{w}").argtypes = [vp, u64, vp, u32, vp]
        L.orc_recode_fact.argtypes = [vp, u64, vp, u32, vp, vp, vp]
        L.orc_aggregate_count_sum_u64.argtypes = [vp, vp, u64, u32, vp, vp, vp, vp]
        L.orc_aggregate_count_sum_u32.argtypes = [vp, vp, u64, u32, vp, vp, vp, vp]
        L.orc_select_offsets.argtypes = [vp, u64, vp, u64, u32, vp, vp, vp, vp]
        L.orc_permute_bitmap.argtypes = [vp, u64, vp, u32, vp]
        L.orc_select_gather_sum.argtypes = [vp, u64, vp, u32, vp, vp, vp, vp, u32, u32,
                                            vp, vp, vp, vp, vp, vp, vp, vp, vp]
        L.orc_chunk_spans.argtypes = [u64, u32, vp, vp]
        L.orc_parallel_gather_u64.argtypes = [vp, u64, vp, u64, vp, u32, vp, vp]
        L.orc_rolling_checksum_u32.restype = u64
        L.orc_rolling_checksum_u32.argtypes = [vp, u64]
        L.orc_unordered_checksum_u64.restype = u64
        L.orc_unordered_checksum_u64.argtypes = [vp, u64]
        L.orc_line_frequencies.argtypes = [vp, u32, C.c_int, u64, u32, vp]
        L.orc_estimate_hit_rate.argtypes = [vp, u64, u64, vp]
        L.orc_simulate_lru.argtypes = [vp, u64, u64, vp, vp, vp]
        L.orc_trace_from_column.argtypes = [vp, u64, u32, vp, vp, vp]
        # multi-threaded forms (skx_oracle_mt.c) for BASELINE-scale parity
        L.orc_find_domain_violation_mt.restype = u64
        L.orc_find_domain_violation_mt.argtypes = [vp, u64, u64, u32]
        L.orc_count_frequencies_mt.argtypes = [vp, u64, u32, vp, u32, vp, vp]
        L.orc_build_index_radix.argtypes = [vp, u32, u64, vp, vp]
        L.orc_gather_mt.argtypes = [C.c_int, vp, u64, vp, u64, vp, u32, vp, vp]
        L.orc_aggregate_count_sum_mt.argtypes = [vp, vp, u64, u32, vp, vp, u32, vp, vp]
        L.orc_select_gather_sum_mt.argtypes = [vp, u64, vp, u32, vp, vp, vp, vp, u32, u32,
                                               vp, vp, vp, vp, vp, vp, vp, u64, u32, vp, vp]
        L.orc_build_bitmap_lt_i32.argtypes = [vp, u64, C.c_int32, vp]
        L.orc_fill_column.argtypes = [C.c_int, C.c_int, u64, u64, dbl, dbl, vp, u32]
        self.threads = os.cpu_count() or 1

    # -- generator ------------------------------------------------------------
    def splitmix64(self, x: int) -> int:
        return self.L.orc_splitmix64(x)

    def zipf_frequencies(self, d, z):
        out = np.empty(d, np.float64)
        if self.L.orc_zipf_frequencies(d, z, _p(out)):
            raise OracleError(INVALID)
        return out

    def zipf_cdf(self, d, z):
        out = np.empty(d, np.float64)
        if self.L.orc_zipf_cdf(d, z, _p(out)):
            raise OracleError(INVALID)
        return out

    def random_bijection(self, n, seed):
        out = np.empty(n, np.uint32)
        self.L.orc_random_bijection(n, seed, _p(out))
        return out

    def generate_fact_column_rand(self, d, n, z, seed, with_counts=False):
        vals = np.empty(n, np.uint32)
        cnt = np.empty(d, np.uint64) if with_counts else None
        if self.L.orc_generate_fact_column_rand(d, n, z, seed, _p(vals), _p(cnt)):
            raise OracleError(INVALID)
        return (vals, cnt) if with_counts else vals

    def generate_zipf_counter(self, cdf, rank_to_id, seed, row_begin, n):
        cdf = np.ascontiguousarray(cdf, np.float64)
        r2i = None if rank_to_id is None else _u32(rank_to_id)
        out = np.empty(n, np.uint32)
        self.L.orc_generate_zipf_counter(_p(cdf), len(cdf), _p(r2i), seed, row_begin, n, _p(out))
        return out

    def generate_zipf_counter_mt(self, cdf, rank_to_id, seed, n, threads):
        cdf = np.ascontiguousarray(cdf, np.float64)
        r2i = None if rank_to_id is None else _u32(rank_to_id)
        out = np.empty(n, np.uint32)
        self.L.orc_generate_zipf_counter_mt(_p(cdf), len(cdf), _p(r2i), seed, n, _p(out), threads)
        return out

    # -- index ----------------------------------------------------------------
    def find_domain_violation(self, fact, d):
        fact = _u32(fact)
        r = self.L.orc_find_domain_violation(_p(fact), len(fact), d)
        return None if r == 2**64 - 1 else r

    def count_frequencies(self, fact, d):
        fact = _u32(fact)
        out = np.empty(d, np.uint64)
        e = _Err()
        e.check(self.L.orc_count_frequencies(_p(fact), len(fact), d, _p(out), *e.args()))
        return out

    def build_index(self, counts, total=None):
        counts = _u64(counts)
        d = len(counts)
        total = int(counts.sum(dtype=np.uint64)) if total is None else total
        off = np.empty(d, np.uint32)
        rk = np.empty(d, np.uint32)
        st = self.L.orc_build_index(_p(counts), d, total, _p(off), _p(rk))
        if st:
            raise OracleError(st)
        return off, rk

    def rebuild(self, fact, d):
        return self.build_index(self.count_frequencies(fact, d))

    def recode_fact(self, fact, ranks):
        return self.gather(fact, _u32(ranks))

    def permute_dimension(self, dim, offsets):
        dim = np.ascontiguousarray(dim)
        offsets = _u32(offsets)
        w = {2: "u16", 4: "u32", 8: "u64"}[dim.dtype.itemsize]
        out = np.empty_like(dim)
        st = getattr(self.L, f"orc_permute_dimension_{w}")(_p(dim), len(dim), _p(offsets),
                                                          len(offsets), _p(out))
        if st:
            raise OracleError(st)
        return out

    # -- operators ------------------------------------------------------------
    def gather(self, fact, dim):
        fact = _u32(fact)
        dim = np.ascontiguousarray(dim)
        w = {2: "u16", 4: "u32", 8: "u64"}[dim.dtype.itemsize]
        out = np.empty(len(fact), dim.dtype)
        e = _Err()
        e.check(getattr(self.L, f"orc_gather_{w}")(_p(fact), len(fact), _p(dim), len(dim),
                                                   _p(out), *e.args()))
        return out

    materialize = gather

    def aggregate_count_sum(self, fact, measure, d):
        fact = _u32(fact)
        counts = np.empty(d, np.uint64)
        sums = np.empty(d, np.uint64)
        e = _Err()
        if measure is None or np.asarray(measure).dtype.itemsize == 8:
            m = None if measure is None else _u64(measure)
            fn = self.L.orc_aggregate_count_sum_u64
        else:
            m = _u32(measure)
            fn = self.L.orc_aggregate_count_sum_u32
        e.check(fn(_p(fact), _p(m), len(fact), d, _p(counts), _p(sums), *e.args()))
        return counts, sums

    def select_offsets(self, fact, words, bits, base=0):
        fact = _u32(fact)
        words = _u64(words)
        out = np.empty(max(len(fact), 1), np.uint32)
        cnt = C.c_uint64(0)
        e = _Err()
        e.check(self.L.orc_select_offsets(_p(fact), len(fact), _p(words), bits, base, _p(out),
                                          C.byref(cnt), *e.args()))
        return out[: cnt.value].copy()

    def permute_bitmap(self, words, bits, offsets):
        words = _u64(words)
        offsets = _u32(offsets)
        out = np.empty((bits + 63) // 64, np.uint64)
        st = self.L.orc_permute_bitmap(_p(words), bits, _p(offsets), len(offsets), _p(out))
        if st:
            raise OracleError(st)
        return out

    def select_gather_sum(self, fact, words, cat, price, supp, flag, n_categories, base=0):
        fact = _u32(fact)
        words = _u64(words)
        cat = np.ascontiguousarray(cat, np.int32)
        price = np.ascontiguousarray(price, np.float32)
        supp = _u64(supp)
        flag = np.ascontiguousarray(flag, np.uint16)
        n = len(fact)
        m = max(n, 1)
        o_off = np.empty(m, np.uint32)
        o_cat = np.empty(m, np.int32)
        o_pr = np.empty(m, np.float32)
        o_su = np.empty(m, np.uint64)
        o_fl = np.empty(m, np.uint16)
        sums = np.empty(n_categories, np.float64)
        cnt = C.c_uint64(0)
        e = _Err()
        e.check(self.L.orc_select_gather_sum(_p(fact), n, _p(words), len(cat), _p(cat), _p(price),
                                             _p(supp), _p(flag), base, n_categories, _p(o_off),
                                             _p(o_cat), _p(o_pr), _p(o_su), _p(o_fl), _p(sums),
                                             C.byref(cnt), *e.args()))
        c = cnt.value
        return (o_off[:c].copy(), o_cat[:c].copy(), o_pr[:c].copy(), o_su[:c].copy(),
                o_fl[:c].copy(), sums)

    def chunk_spans(self, n, threads):
        b = np.empty(threads, np.uint64)
        e = np.empty(threads, np.uint64)
        if self.L.orc_chunk_spans(n, threads, _p(b), _p(e)):
            raise OracleError(INVALID)
        return [(int(x), int(y)) for x, y in zip(b, e)]

    def parallel_gather_u64(self, fact, dim, out, threads):
        e = _Err()
        e.check(self.L.orc_parallel_gather_u64(_p(fact), len(fact), _p(dim), len(dim), _p(out),
                                               threads, *e.args()))
        return out

    # -- multi-threaded forms (skx_oracle_mt.c): BASELINE-scale parity --------
    def find_domain_violation_mt(self, fact, d):
        fact = _u32(fact)
        r = self.L.orc_find_domain_violation_mt(_p(fact), len(fact), d, self.threads)
        return None if r == 2**64 - 1 else r

    def count_frequencies_mt(self, fact, d):
        fact = _u32(fact)
        out = np.empty(d, np.uint64)
        e = _Err()
        e.check(self.L.orc_count_frequencies_mt(_p(fact), len(fact), d, _p(out), self.threads,
                                                *e.args()))
        return out

    def build_index_radix(self, counts, total=None):
        counts = _u64(counts)
        d = len(counts)
        total = int(counts.sum(dtype=np.uint64)) if total is None else total
        off = np.empty(d, np.uint32)
        rk = np.empty(d, np.uint32)
        st = self.L.orc_build_index_radix(_p(counts), d, total, _p(off), _p(rk))
        if st:
            raise OracleError(st)
        return off, rk

    def gather_mt(self, fact, dim, out=None):
        fact = _u32(fact)
        dim = np.ascontiguousarray(dim)
        out = np.empty(len(fact), dim.dtype) if out is None else out
        e = _Err()
        e.check(self.L.orc_gather_mt(dim.dtype.itemsize, _p(fact), len(fact), _p(dim), len(dim),
                                     _p(out), self.threads, *e.args()))
        return out

    def aggregate_count_sum_mt(self, fact, measure, d):
        fact = _u32(fact)
        m = None if measure is None else _u64(measure)
        counts = np.empty(d, np.uint64)
        sums = np.empty(d, np.uint64)
        e = _Err()
        e.check(self.L.orc_aggregate_count_sum_mt(_p(fact), _p(m), len(fact), d, _p(counts),
                                                  _p(sums), self.threads, *e.args()))
        return counts, sums

    def select_gather_sum_mt(self, fact, words, cat, price, supp, flag, n_categories, base=0,
                             capacity=None):
        fact = _u32(fact)
        words = _u64(words)
        cat = np.ascontiguousarray(cat, np.int32)
        price = np.ascontiguousarray(price, np.float32)
        supp = _u64(supp)
        flag = np.ascontiguousarray(flag, np.uint16)
        n = len(fact)
        m = max(n if capacity is None else capacity, 1)
        outs = [np.empty(m, t) for t in (np.uint32, np.int32, np.float32, np.uint64, np.uint16)]
        sums = np.empty(n_categories, np.float64)
        cnt = C.c_uint64(0)
        e = _Err()
        st = self.L.orc_select_gather_sum_mt(_p(fact), n, _p(words), len(cat), _p(cat), _p(price),
                                             _p(supp), _p(flag), base, n_categories,
                                             *[_p(o) for o in outs], _p(sums), C.byref(cnt), m,
                                             self.threads, *e.args())
        if st == INVALID and cnt.value > m:  # more rows selected than `capacity`: exact size
            return self.select_gather_sum_mt(fact, words, cat, price, supp, flag, n_categories,
                                             base, capacity=cnt.value)
        e.check(st)
        c = cnt.value
        return tuple(o[:c] for o in outs) + (sums,)

    def build_bitmap_lt_i32(self, dim, threshold):
        dim = np.ascontiguousarray(dim, np.int32)
        w = np.empty((len(dim) + 63) // 64, np.uint64)
        self.L.orc_build_bitmap_lt_i32(_p(dim), len(dim), threshold, _p(w))
        return w

    def fill_column(self, kind, dtype, n, seed, p0=0.0, p1=0.0):
        out = np.empty(n, dtype)
        if self.L.orc_fill_column(kind, out.dtype.itemsize, seed & (2**64 - 1), n, float(p0),
                                  float(p1), _p(out), self.threads):
            raise OracleError(INVALID)
        return out

    def rolling_checksum(self, v):
        v = _u32(v)
        return self.L.orc_rolling_checksum_u32(_p(v), len(v))

    def unordered_checksum(self, v):
        v = _u64(v)
        return self.L.orc_unordered_checksum_u64(_p(v), len(v))

    # -- cache model (cachemodel.cpp) ---------------------------------------------
    def line_frequencies(self, value_freqs, layout, line_bytes, element_bytes, seed):
        vf = np.ascontiguousarray(value_freqs, dtype=np.float64)
        per = line_bytes // element_bytes
        out = np.empty((len(vf) + per - 1) // per, np.float64)
        if self.L.orc_line_frequencies(_p(vf), len(vf), 0 if layout == "freq" else 1, seed, per,
                                       _p(out)):
            raise OracleError(1)
        return out

    def estimate_hit_rate(self, line_freqs, cache_lines):
        lf = np.ascontiguousarray(line_freqs, dtype=np.float64)
        r = C.c_double(0.0)
        if self.L.orc_estimate_hit_rate(_p(lf), len(lf), cache_lines, C.byref(r)):
            raise OracleError(1)
        return r.value

    def simulate_lru(self, trace, cache_lines):
        t = _u32(trace)
        a, h, dd = C.c_uint64(), C.c_uint64(), C.c_uint64()
        if self.L.orc_simulate_lru(_p(t), len(t), cache_lines, C.byref(a), C.byref(h), C.byref(dd)):
            raise OracleError(1)
        return a.value, h.value, dd.value

    def trace_from_column(self, fact, line_bytes, element_bytes):
        fact = _u32(fact)
        out = np.empty(len(fact), np.uint32)
        e = _Err()
        e.check(self.L.orc_trace_from_column(_p(fact), len(fact), line_bytes // element_bytes,
                                             _p(out), *e.args()))
        return out


class Reference:
    """The unmodified reference library (oracle/_ref/libskewdx_ref.so)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            build(ref=True)
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        L = self.L = C.CDLL(path)
        vp, u64, u32, dbl, ci = C.c_void_p, C.c_uint64, C.c_uint32, C.c_double, C.c_int
        L.ref_hardware_concurrency.restype = C.c_uint
        L.ref_zipf_frequencies.argtypes = [u32, dbl, vp]
        L.ref_random_bijection.argtypes = [u32, u64, vp]
        L.ref_generate_fact_column.argtypes = [u32, u64, dbl, u64, ci, vp, vp]
        L.ref_count_frequencies.argtypes = [vp, u64, u32, vp, vp, vp, vp]
        L.ref_build_index.argtypes = [vp, u32, u64, vp, vp]
        L.ref_rebuild.argtypes = [vp, u64, u32, vp, vp, vp, vp]
        L.ref_recode_fact.argtypes = [vp, u64, vp, vp, u32, vp, vp, vp]
        L.ref_permute_dimension.argtypes = [vp, u64, vp, vp, u32, vp]
        L.ref_materialize.argtypes = [vp, u64, vp, u64, vp, vp, vp]
        L.ref_parallel_materialize.argtypes = [vp, u64, vp, u64, vp, C.c_uint, vp, vp]
        L.ref_select.argtypes = [vp, u64, vp, u64, vp, vp, C.c_uint, vp, vp]
        L.ref_permute_bitmap.argtypes = [vp, u64, vp, vp, u32, vp]
        L.ref_aggregate_count.argtypes = [vp, u64, u32, vp, vp, vp]
        L.ref_aggregate_sum.argtypes = [vp, vp, u64, u64, u32, vp, vp, vp]
        L.ref_parallel_aggregate.argtypes = [vp, u64, u32, C.c_uint, ci, u32, vp, vp, vp, vp]
        L.ref_heavy_hitter_count.argtypes = [vp, u64, u32, u32, vp, vp, vp, vp]
        L.ref_time_index_build.argtypes = [vp, u64, u32, vp, vp, vp]
        L.ref_time_parallel_materialize.restype = dbl
        L.ref_time_parallel_materialize.argtypes = [vp, u64, vp, u64, C.c_uint, ci]
        L.ref_time_gather_kernel.restype = dbl
        L.ref_time_gather_kernel.argtypes = [vp, u64, vp, vp, C.c_uint, ci]
        L.ref_line_frequencies.argtypes = [vp, u32, ci, u64, u32, u32, vp]
        L.ref_estimate_hit_rate.argtypes = [vp, u64, u64, vp]
        L.ref_simulate_lru.argtypes = [vp, u64, u64, vp]
        L.ref_trace_from_column.argtypes = [vp, u64, u32, u32, vp, vp, vp]
        L.ref_time_parallel_select.restype = dbl
        L.ref_time_parallel_select.argtypes = [vp, u64, vp, u64, C.c_uint, ci, vp]
        L.ref_time_aggregate_sum.restype = dbl
        L.ref_time_aggregate_sum.argtypes = [vp, vp, u64, u32, ci]
        L.ref_time_parallel_aggregate.restype = dbl
        L.ref_time_parallel_aggregate.argtypes = [vp, u64, u32, C.c_uint, ci, u32, ci]
        L.ref_time_rebuild.restype = dbl
        L.ref_time_rebuild.argtypes = [vp, u64, u32, ci]
        L.ref_active_kernels_name.restype = C.c_char_p

    def hardware_concurrency(self):
        return self.L.ref_hardware_concurrency()

    def zipf_frequencies(self, d, z):
        out = np.empty(d, np.float64)
        if self.L.ref_zipf_frequencies(d, z, _p(out)):
            raise OracleError(INVALID)
        return out

    def random_bijection(self, n, seed):
        out = np.empty(n, np.uint32)
        self.L.ref_random_bijection(n, seed, _p(out))
        return out

    def generate_fact_column(self, d, n, z, seed, layout="rand", with_counts=False):
        vals = np.empty(n, np.uint32)
        cnt = np.empty(d, np.uint64)
        st = self.L.ref_generate_fact_column(d, n, z, seed, 1 if layout == "freq" else 0,
                                             _p(vals), _p(cnt))
        if st:
            raise OracleError(st)
        return (vals, cnt) if with_counts else vals

    def count_frequencies(self, fact, d):
        fact = _u32(fact)
        out = np.empty(d, np.uint64)
        tot = C.c_uint64(0)
        e = _Err()
        e.check(self.L.ref_count_frequencies(_p(fact), len(fact), d, _p(out), C.byref(tot),
                                             *e.args()))
        return out

    def build_index(self, counts, total=None):
        counts = _u64(counts)
        d = len(counts)
        total = int(counts.sum(dtype=np.uint64)) if total is None else total
        off = np.empty(d, np.uint32)
        rk = np.empty(d, np.uint32)
        st = self.L.ref_build_index(_p(counts), d, total, _p(off), _p(rk))
        if st:
            raise OracleError(st)
        return off, rk

    def rebuild(self, fact, d):
        fact = _u32(fact)
        off = np.empty(d, np.uint32)
        rk = np.empty(d, np.uint32)
        e = _Err()
        e.check(self.L.ref_rebuild(_p(fact), len(fact), d, _p(off), _p(rk), *e.args()))
        return off, rk

    def recode_fact(self, fact, offsets, ranks):
        fact, offsets, ranks = _u32(fact), _u32(offsets), _u32(ranks)
        out = np.empty(len(fact), np.uint32)
        e = _Err()
        e.check(self.L.ref_recode_fact(_p(fact), len(fact), _p(offsets), _p(ranks), len(offsets),
                                       _p(out), *e.args()))
        return out

    def permute_dimension(self, dim, offsets, ranks):
        dim, offsets, ranks = _u32(dim), _u32(offsets), _u32(ranks)
        out = np.empty(len(dim), np.uint32)
        st = self.L.ref_permute_dimension(_p(dim), len(dim), _p(offsets), _p(ranks),
                                          len(offsets), _p(out))
        if st:
            raise OracleError(st)
        return out

    def materialize(self, fact, dim, threads=1):
        fact, dim = _u32(fact), _u32(dim)
        out = np.empty(len(fact), np.uint32)
        e = _Err()
        if threads <= 1:
            st = self.L.ref_materialize(_p(fact), len(fact), _p(dim), len(dim), _p(out),
                                        *e.args())
        else:
            st = self.L.ref_parallel_materialize(_p(fact), len(fact), _p(dim), len(dim),
                                                 _p(out), threads, *e.args())
        e.check(st)
        return out

    def select(self, fact, words, bits, threads=1):
        fact, words = _u32(fact), _u64(words)
        out = np.empty(max(len(fact), 1), np.uint32)
        cnt = C.c_uint64(0)
        e = _Err()
        e.check(self.L.ref_select(_p(fact), len(fact), _p(words), bits, _p(out), C.byref(cnt),
                                  threads, *e.args()))
        return out[: cnt.value].copy()

    def permute_bitmap(self, words, bits, offsets, ranks):
        words, offsets, ranks = _u64(words), _u32(offsets), _u32(ranks)
        out = np.empty((bits + 63) // 64, np.uint64)
        st = self.L.ref_permute_bitmap(_p(words), bits, _p(offsets), _p(ranks), len(offsets),
                                       _p(out))
        if st:
            raise OracleError(st)
        return out

    def aggregate_count(self, fact, d):
        fact = _u32(fact)
        out = np.empty(d, np.uint64)
        e = _Err()
        e.check(self.L.ref_aggregate_count(_p(fact), len(fact), d, _p(out), *e.args()))
        return out

    def aggregate_sum(self, fact, measure, d):
        fact, measure = _u32(fact), _u32(measure)
        out = np.empty(d, np.uint64)
        e = _Err()
        e.check(self.L.ref_aggregate_sum(_p(fact), _p(measure), len(fact), len(measure), d,
                                         _p(out), *e.args()))
        return out

    def parallel_aggregate(self, fact, d, threads, strategy, hot_threshold=8192):
        fact = _u32(fact)
        out = np.empty(d, np.uint64)
        shared = C.c_uint64(0)
        e = _Err()
        e.check(self.L.ref_parallel_aggregate(_p(fact), len(fact), d, threads, strategy,
                                              hot_threshold, _p(out), C.byref(shared),
                                              *e.args()))
        return out, shared.value

    def heavy_hitter_count(self, fact, d, k):
        fact = _u32(fact)
        m = min(k, d)
        ids = np.empty(m, np.uint32)
        cnt = np.empty(m, np.uint64)
        ln = C.c_uint64(0)
        cl = C.c_int(0)
        st = self.L.ref_heavy_hitter_count(_p(fact), len(fact), d, k, _p(ids), _p(cnt),
                                           C.byref(ln), C.byref(cl))
        if st:
            raise OracleError(st)
        return ids[: ln.value], cnt[: ln.value], bool(cl.value)

    def line_frequencies(self, value_freqs, layout, line_bytes, element_bytes, seed):
        vf = np.ascontiguousarray(value_freqs, dtype=np.float64)
        per = line_bytes // element_bytes
        out = np.empty((len(vf) + per - 1) // per, np.float64)
        if self.L.ref_line_frequencies(_p(vf), len(vf), 1 if layout == "freq" else 0, seed,
                                       line_bytes, element_bytes, _p(out)):
            raise OracleError(1)
        return out

    def estimate_hit_rate(self, line_freqs, cache_lines):
        lf = np.ascontiguousarray(line_freqs, dtype=np.float64)
        r = C.c_double(0.0)
        if self.L.ref_estimate_hit_rate(_p(lf), len(lf), cache_lines, C.byref(r)):
            raise OracleError(1)
        return r.value

    def simulate_lru(self, trace, cache_lines):
        t = _u32(trace)
        st = np.zeros(3, np.uint64)
        if self.L.ref_simulate_lru(_p(t), len(t), cache_lines, _p(st)):
            raise OracleError(1)
        return int(st[0]), int(st[1]), int(st[2])

    def trace_from_column(self, fact, line_bytes, element_bytes):
        fact = _u32(fact)
        out = np.empty(len(fact), np.uint32)
        e = _Err()
        e.check(self.L.ref_trace_from_column(_p(fact), len(fact), line_bytes, element_bytes,
                                             _p(out), *e.args()))
        return out

    def active_kernels_name(self):
        return self.L.ref_active_kernels_name().decode()

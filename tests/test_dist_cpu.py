"""World-size-2 tests of the multi-GPU host logic (paper_1910_10063_b200/dist.py)
over gloo on CPU, with the oracle as the per-shard executor: the sharded
results after the collectives must equal the single-process oracle on the
whole column (the same contract the NCCL path has on B200s), the group-by's
packed combine must be bit-identical to the plain one (and fall back when its
guard fails), the config-5 category sums must combine exactly, and a domain
violation in one shard must raise the same DomainViolation (global row) on
every rank instead of leaving a rank blocked in a collective."""
import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle.oracle import Oracle, OracleError


class _Bitmap:
    def __init__(self, words, bits):
        self.words, self.bits = words, bits

    def size(self):
        return self.bits


class OracleExecutor:
    """CPU stand-in for dist.GpuExecutor (TEST ONLY): same method contract on
    CPU tensors, computed by the oracle (and, for the combine layouts, by
    numpy restatements of the combine kernels in csrc/combine.cu and
    csrc/select.cu)."""

    device = torch.device("cpu")

    def __init__(self):
        self.o = Oracle()
        self.pending = None
        self.last_sel = None

    def _guard(self, fn):
        try:
            return fn()
        except OracleError as e:
            if e.status != 2:
                raise
            self.pending = (e.row, e.value)
            return None

    def histogram_u32(self, fact, d, out=None):
        c = self._guard(lambda: self.o.count_frequencies(fact.numpy(), d))
        c = np.zeros(d, np.uint64) if c is None else c
        t = torch.from_numpy(c.astype(np.uint32))
        if out is not None:
            out.copy_(t)
            return out
        return t

    def build_index(self, counts_u32, total):
        off, rk = self.o.build_index(counts_u32.numpy().astype(np.uint64), total)
        return (torch.from_numpy(off), torch.from_numpy(rk))

    def recode(self, fact, index, out=None):
        return torch.from_numpy(self.o.recode_fact(fact.numpy(), index[1].numpy()))

    def gather(self, fact, dim, out=None):
        return torch.from_numpy(self.o.gather(fact.numpy(), dim.numpy()))

    def aggregate(self, fact, measure, d, counts=None, sums=None):
        r = self._guard(lambda: self.o.aggregate_count_sum(fact.numpy(),
                                                          measure.numpy().view(np.uint64), d))
        c, s = r if r is not None else (np.zeros(d, np.uint64), np.zeros(d, np.uint64))
        return torch.from_numpy(c), torch.from_numpy(s)

    # restatement of k_groupby_pack / k_groupby_unpack (csrc/combine.cu)
    def groupby_pack(self, counts, sums, hot):
        c = counts.numpy().view(np.uint64)
        s = sums.numpy().view(np.uint64)
        tail_c, tail_s = c[hot:], s[hot:]
        packed = (tail_c << np.uint64(40)) | (tail_s & np.uint64((1 << 40) - 1))
        buf = np.concatenate([c[:hot], s[:hot], packed])
        guard = np.array([tail_c.max(initial=0), tail_s.max(initial=0)], np.uint64)
        return torch.from_numpy(buf), torch.from_numpy(guard)

    def groupby_unpack(self, buf, d, hot, counts, sums):
        b = buf.numpy().view(np.uint64)
        w = b[2 * hot:]
        counts.copy_(torch.from_numpy(np.concatenate([b[:hot], w >> np.uint64(40)])))
        sums.copy_(torch.from_numpy(np.concatenate([b[hot:2 * hot], w & np.uint64((1 << 40) - 1)])))

    @staticmethod
    def packed_ok(guard_sum):
        g = guard_sum.numpy().view(np.uint64)
        return bool(g[0] < (1 << 24) and g[1] < (1 << 40))

    def select_gather_sum(self, fact, bitmap, cols, ncat, base, out):
        cat, price, supp, flag = (c.numpy() for c in cols)
        r = self._guard(lambda: self.o.select_gather_sum(
            fact.numpy(), bitmap.words, cat, price, supp.view(np.uint64), flag.view(np.uint16),
            ncat, base=base))
        if r is None:
            r = tuple(np.zeros(0, t) for t in (np.uint32, np.int32, np.float32, np.uint64,
                                              np.uint16)) + (np.zeros(ncat),)
        # the device's fixed-point partial (k_pack_records scale, emit_row's
        # rounding to 2^-S, 96-bit two's complement words)
        p = price.astype(np.float64)
        sel = ((bitmap.words[np.arange(len(p)) >> 6] >> (np.arange(len(p)) & 63).astype(np.uint64))
               & np.uint64(1)).astype(bool)
        p = p[sel]  # the device's scale comes from the selected keys' prices
        fin = p[np.isfinite(p) & (p != 0)]
        S = 0
        fixed = bool(np.isfinite(p).all()) and ncat <= 4096
        if fixed and fin.size:
            e = np.frexp(np.abs(fin))[1]
            fixed = int(e.max() - e.min()) <= 30
            S = 62 - int(e.max())
        tot = [0] * ncat
        if fixed:
            v = np.rint(np.ldexp(r[2].astype(np.float64), S)).astype(np.int64)
            for c, x in zip(r[1].tolist(), v.tolist()):
                if 0 <= c < ncat:
                    tot[c] += x
        self.last_sel = (fixed, S, tot)
        return tuple(torch.from_numpy(np.ascontiguousarray(a)) for a in r) + (
            torch.tensor([len(r[0])], dtype=torch.int64),)

    def sum_partials(self, ncat):
        fixed, S, tot = self.last_sel
        out = [1 if fixed else 0, S if fixed else 0]
        for t in tot:
            w = t % (1 << 96)
            hi = w >> 64
            out += [w & 0xFFFFFFFF, (w >> 32) & 0xFFFFFFFF, hi - (1 << 32) if hi >= 1 << 31 else hi]
        return torch.tensor(out, dtype=torch.int64)

    def sums_from_partials(self, part, ncat, nranks, sums):
        p = part.tolist()
        if p[0] != nranks or p[1] % nranks:
            return
        S = p[1] // nranks
        for c in range(ncat):
            t = p[2 + 3 * c] + (p[3 + 3 * c] << 32) + (p[4 + 3 * c] << 64)
            sums[c] = math.ldexp(float(t), -S)

    def take_violation(self):
        v, self.pending = self.pending, None
        return v


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _data(o, d, n):
    cdf = o.zipf_cdf(d, 1.1)
    return o.generate_zipf_counter(cdf, o.random_bijection(d, 5), 5, 0, n)


def _worker(rank, world, port, d, n, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1910_10063_b200 import dist as sdist
    from paper_1910_10063_b200.errors import DomainViolation
    o = Oracle()
    ex = OracleExecutor()
    coll = sdist.default_collectives()
    assert isinstance(coll, sdist.TorchCollectives)
    shard = sdist.shard_for(n)
    full = _data(o, d, n)
    fact = torch.from_numpy(full[shard.begin:shard.end].copy())
    res = {}
    # index build: local histogram + all-reduce + identical sort
    (off, rk), _ = sdist.rebuild(fact, d, n, ex, coll, shard)
    rec = ex.recode(fact, (off, rk))
    # group-by on the recoded shard: packed combine, forced pairs, guard failure
    meas = torch.from_numpy((np.arange(shard.begin, shard.end, dtype=np.int64) % 97) + 1)
    st1, st2, st3 = {}, {}, {}
    c1, s1 = sdist.aggregate(rec, meas, d, ex, coll, shard, hot=64, stats=st1)
    c2, s2 = sdist.aggregate(rec, meas, d, ex, coll, shard, packed=False, stats=st2)
    big = meas.clone()
    big[-1] = 1 << 41  # a tail key's sum cannot be packed
    c3, s3 = sdist.aggregate(rec, big, d, ex, coll, shard, hot=64, stats=st3)
    res.update(c1=c1.numpy(), s1=s1.numpy(), c2=c2.numpy(), s2=s2.numpy(), c3=c3.numpy(),
               s3=s3.numpy(), paths=np.array([st1["path"], st2["path"], st3["path"]]))
    # config 5 on the recoded shard: offsets with base, exact category sums
    rng = np.random.default_rng(7)
    cat = torch.from_numpy(rng.integers(0, 50, size=d, dtype=np.int32))
    price = torch.from_numpy(np.exp(3 + rng.standard_normal(d)).astype(np.float32))
    supp = torch.from_numpy(rng.integers(0, 2**62, size=d, dtype=np.int64))
    flag = torch.from_numpy(rng.integers(0, 2**15, size=d, dtype=np.int16))
    words = o.build_bitmap_lt_i32(cat.numpy(), 20)
    bm = _Bitmap(words, d)
    out = sdist.select_gather_sum(rec, bm, (cat, price, supp, flag), 50, ex, coll, shard)
    res.update(sel_off=sdist.concat_selection(out[0], coll).numpy(), sums=out[5].numpy())
    # a domain violation in rank 1's shard: every rank raises it, global row
    bad = fact.clone()
    if rank == 1:
        bad[10] = d + 3
        bad[20] = 0
    for fn in (lambda: sdist.rebuild(bad, d, n, ex, coll, shard),
               lambda: sdist.aggregate(bad, meas, d, ex, coll, shard)):
        try:
            fn()
            res.setdefault("raised", []).append(-1)
        except DomainViolation as e:
            res.setdefault("raised", []).append(e.row())
            res.setdefault("values", []).append(e.value())
    res["raised"] = np.array(res["raised"])
    res["values"] = np.array(res.get("values", []))
    np.savez(os.path.join(out_dir, f"r{rank}.npz"), off=off.numpy(), rk=rk.numpy(),
             rec=rec.numpy(), **res)
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_sharded_path_equals_whole_column(tmp_path, world):
    d, n = 3001, 200003
    mp.spawn(_worker, args=(world, _free_port(), d, n, str(tmp_path)), nprocs=world, join=True)
    o = Oracle()
    fact = _data(o, d, n)
    off, rk = o.rebuild(fact, d)
    r = [np.load(tmp_path / f"r{k}.npz") for k in range(world)]
    for k in range(world):
        assert np.array_equal(r[k]["off"], off) and np.array_equal(r[k]["rk"], rk)
    rec = np.concatenate([r[k]["rec"] for k in range(world)])
    assert np.array_equal(rec, o.recode_fact(fact, rk))
    meas = (np.arange(n, dtype=np.int64) % 97) + 1
    c, s = o.aggregate_count_sum(rec, meas.view(np.uint64), d)
    r0 = r[0]
    assert list(r0["paths"]) == ["packed", "pairs", "pairs"]
    for ck, sk in (("c1", "s1"), ("c2", "s2")):
        assert np.array_equal(r0[ck], c) and np.array_equal(r0[sk], s)
    big = meas.copy()
    for k in range(world):  # each shard's last row carries 2^41
        big[o.chunk_spans(n, world)[k][1] - 1] = 1 << 41
    c3, s3 = o.aggregate_count_sum(rec, big.view(np.uint64), d)
    assert np.array_equal(r0["c3"], c3) and np.array_equal(r0["s3"], s3)
    # selection: rank-order concatenation == the whole-column selection
    rng = np.random.default_rng(7)
    cat = rng.integers(0, 50, size=d, dtype=np.int32)
    price = np.exp(3 + rng.standard_normal(d)).astype(np.float32)
    supp = rng.integers(0, 2**62, size=d, dtype=np.int64).view(np.uint64)
    flag = rng.integers(0, 2**15, size=d, dtype=np.int16).view(np.uint16)
    words = o.build_bitmap_lt_i32(cat, 20)
    exp = o.select_gather_sum(rec, words, cat, price, supp, flag, 50)
    assert np.array_equal(r0["sel_off"].astype(np.uint32), exp[0])
    assert np.allclose(r0["sums"], exp[5], rtol=1e-12, atol=0)
    # exact combine: the root's sums are the correctly rounded exact sums
    S = 62 - int(np.frexp(np.abs(price[cat < 20].astype(np.float64)))[1].max())
    v = np.rint(np.ldexp(exp[2].astype(np.float64), S)).astype(np.int64)
    tot = [0] * 50
    for cc, x in zip(exp[1].tolist(), v.tolist()):
        tot[cc] += x
    assert r0["sums"].tolist() == [math.ldexp(float(t), -S) for t in tot]
    # violation in rank 1's shard: global row = shard begin + 10, on every rank
    b1 = o.chunk_spans(n, world)[1][0]
    for k in range(world):
        assert r[k]["raised"].tolist() == [b1 + 10, b1 + 10]
        assert r[k]["values"].tolist() == [d + 3, d + 3]


def test_shard_for_matches_chunk_spans():
    from paper_1910_10063_b200 import dist as sdist
    o = Oracle()
    for n, w in [(0, 2), (7, 3), (1 << 20, 8), (1000003, 4)]:
        spans = o.chunk_spans(n, w)
        for r in range(w):
            s = sdist.shard_for(n, r, w)
            assert (s.begin, s.end) == spans[r]


def _worker_small(rank, world, port, n, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1910_10063_b200 import dist as sdist
    from paper_1910_10063_b200.errors import DomainViolation
    o = Oracle()
    ex = OracleExecutor()
    coll = sdist.default_collectives()
    d = 7
    full = (np.arange(n, dtype=np.uint32) * 5) % d + 1
    shard = sdist.shard_for(n)
    fact = torch.from_numpy(full[shard.begin:shard.end].copy())
    (off, rk), _ = sdist.rebuild(fact, d, n, ex, coll, shard)
    meas = torch.ones(shard.rows, dtype=torch.int64)
    c, s = sdist.aggregate(fact, meas, d, ex, coll, shard, hot=2)
    # violations in two shards: the smaller global row wins on every rank
    bad = fact.clone()
    if shard.rows and rank in (1, world - 1):
        bad[0] = 0 if rank == 1 else d + 1
    try:
        sdist.rebuild(bad, d, n, ex, coll, shard)
        raised = -1
    except DomainViolation as e:
        raised = e.row()
    np.savez(os.path.join(out_dir, f"s{rank}.npz"), off=off.numpy(), c=c.numpy(), s=s.numpy(),
             raised=np.array([raised]), rows=np.array([shard.rows]))
    dist.destroy_process_group()


@pytest.mark.parametrize("world,n", [(4, 3), (3, 10)])
def test_uneven_and_empty_shards(tmp_path, world, n):
    """chunk_spans shards of unequal length, including empty ones (n < world):
    the index and the reduced counts equal the whole-column results, and with
    violations in two shards every rank raises the smaller global row."""
    mp.spawn(_worker_small, args=(world, _free_port(), n, str(tmp_path)), nprocs=world, join=True)
    o = Oracle()
    d = 7
    full = (np.arange(n, dtype=np.uint32) * 5) % d + 1
    off, _ = o.rebuild(full, d)
    c, s = o.aggregate_count_sum(full, np.ones(n, np.uint64), d)
    r = [np.load(tmp_path / f"s{k}.npz") for k in range(world)]
    spans = o.chunk_spans(n, world)
    bad_rows = [spans[k][0] for k in (1, world - 1) if spans[k][1] > spans[k][0]]
    for k in range(world):
        assert np.array_equal(r[k]["off"], off)
        assert int(r[k]["raised"][0]) == (min(bad_rows) if bad_rows else -1)
    assert np.array_equal(r[0]["c"], c) and np.array_equal(r[0]["s"], s)
    assert sum(int(x["rows"][0]) for x in r) == n

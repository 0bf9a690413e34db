"""GPU parity: the sm_100a kernels (through the C-ABI in libskx.so) against
the pinned oracle and the reference's golden fixtures.  Bit-exact for every
integer / index / byte result; fp64 category sums within 1e-6 relative."""
import numpy as np
import pytest
import torch

from conftest import words_from_bits

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sx():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_1910_10063_b200 import skewdx
    skewdx.context(0)
    return skewdx


def cu(a, dtype=None):
    t = torch.from_numpy(np.ascontiguousarray(a))
    if dtype is not None:
        t = t.view(dtype)
    return t.cuda()


def np_(t):
    return t.cpu().numpy()


# ---------------------------------------------------------------- golden ---
def test_golden_cases_full_path(sx, ref_cases):
    for i in range(len(ref_cases)):
        c = ref_cases.case(i)
        d = c["d"]
        fact = cu(c["fact"])
        prof = sx.count_frequencies(fact, d)
        assert np.array_equal(np_(prof.counts), c["counts"]), i
        idx = sx.build_index(prof)
        assert np.array_equal(np_(idx.offsets), c["offsets"]), i
        assert np.array_equal(np_(idx.ranks), c["ranks"]), i
        idx2 = sx.rebuild(fact, d)
        assert np.array_equal(np_(idx2.offsets), c["offsets"]), i
        assert np.array_equal(np_(idx2.ranks), c["ranks"]), i
        rec = sx.recode_fact(fact, idx)
        assert np.array_equal(np_(rec), c["recoded"]), i
        dim = cu(c["dim"])
        dperm = sx.permute_dimension(dim, idx)
        assert np.array_equal(np_(dperm), c["dim_perm"]), i
        assert np.array_equal(np_(sx.materialize(fact, dim)), c["mat_rand"]), i
        assert np.array_equal(np_(sx.materialize(rec, dperm)), c["mat_freq"]), i
        counts, sums = sx.aggregate_count_sum(rec, cu(c["measure"]), d)
        assert np.array_equal(np_(counts), c["counts_freq"]), i
        assert np.array_equal(np_(sums), c["sums"]), i
        assert np.array_equal(np_(sx.aggregate_count(rec, d)), c["counts_freq"]), i
        bm = sx.Bitmap.from_numpy(c["words"], d)
        bmp = sx.permute_bitmap(bm, idx)
        assert np.array_equal(np_(bmp.words), c["words_perm"]), i
        assert np.array_equal(np_(sx.select(fact, bm)), c["sel_rand"]), i
        assert np.array_equal(np_(sx.select(rec, bmp)), c["sel_freq"]), i
        hh = sx.heavy_hitter_count(rec, d, 13)
        assert [t[0] for t in hh.top] == c["hh_ids"].tolist(), i
        assert [t[1] for t in hh.top] == c["hh_counts"].tolist(), i


# ------------------------------------------------------------------- KATs ---
def test_kat(sx, kat):
    from paper_1910_10063_b200 import DomainViolation, InvalidArgument
    for c in kat["count_frequencies"]:
        p = sx.count_frequencies(cu(np.array(c["fact"], np.uint32)), c["d"])
        assert np_(p.counts).tolist() == c["counts"] and p.total == c["total"]
    for c in kat["count_frequencies_violation"]:
        with pytest.raises(DomainViolation) as e:
            sx.count_frequencies(cu(np.array(c["fact"], np.uint32)), c["d"])
        assert e.value.row() == c["row"] and e.value.value() == c["value"]
    pf = kat["popularity_fixture"]
    fact = np.concatenate([np.full(cnt, i, np.uint32) for i, cnt in pf["by_count"]])
    np.random.default_rng(99).shuffle(fact)
    idx = sx.rebuild(cu(fact), pf["d"])
    assert np_(idx.offsets).tolist() == pf["offsets"] and np_(idx.ranks).tolist() == pf["ranks"]
    assert np_(sx.recode_fact(cu(np.array(pf["recode_in"], np.uint32)), idx)).tolist() == pf["recode_out"]
    assert np_(sx.permute_dimension(cu(np.array(pf["dim"], np.uint32)), idx)).tolist() == pf["permuted_dim"]
    for c in kat["build_index"]:
        idx = sx.build_index(sx.FrequencyProfile(cu(np.array(c["counts"], np.uint64)), c["total"]))
        assert np_(idx.offsets).tolist() == c["offsets"] and np_(idx.ranks).tolist() == c["ranks"]
    for c in kat["build_index_invalid"]:
        with pytest.raises(InvalidArgument):
            sx.build_index(sx.FrequencyProfile(cu(np.array(c["counts"], np.uint64)), c["total"]))
    c = kat["permute_length_mismatch"]
    idx = sx.rebuild(cu(np.array(c["fact"], np.uint32)), c["d"])
    with pytest.raises(InvalidArgument):
        sx.permute_dimension(cu(np.array(c["dim"], np.uint32)), idx)
    c = kat["aggregate_count"]
    assert np_(sx.aggregate_count(cu(np.array(c["fact"], np.uint32)), c["d"])).tolist() == c["counts"]
    c = kat["aggregate_sum"]
    assert np_(sx.aggregate_sum(cu(np.array(c["fact"], np.uint32)),
                                cu(np.array(c["measure"], np.uint32)), c["d"])).tolist() == c["sums"]
    with pytest.raises(InvalidArgument):
        sx.aggregate_sum(cu(np.array(c["fact"], np.uint32)), cu(np.array([1], np.uint32)), c["d"])
    for c in kat["select"]:
        bm = sx.Bitmap.from_numpy(words_from_bits(c["bits"], c["d"]), c["d"])
        assert np_(sx.select(cu(np.array(c["fact"], np.uint32)), bm)).tolist() == c["offsets"]
    c = kat["select_violation"]
    with pytest.raises(DomainViolation) as e:
        sx.select(cu(np.array(c["fact"], np.uint32)),
                  sx.Bitmap.from_numpy(words_from_bits(c["bits"], c["d"]), c["d"]))
    assert e.value.row() == c["row"] and e.value.value() == c["value"]
    c = kat["build_bitmap"]
    bm = sx.build_bitmap_lt(cu(np.array(c["values"], np.int32)), c["threshold"])
    assert np_(bm.words).tolist() == words_from_bits(c["set"], len(c["values"])).tolist()
    for c in kat["heavy_hitters"]:
        hh = sx.heavy_hitter_count(cu(np.array(c["fact"], np.uint32)), c["d"], c["k"])
        assert [list(t) for t in hh.top] == c["top"] and hh.clamped == c["clamped"]
    g = kat["gather_edges"]
    dim = cu(np.arange(10, 10 + g["d"], dtype=np.uint32))
    assert sx.materialize(cu(np.array([], np.uint32)), dim).numel() == 0
    for bad in (g["bad_high"], g["bad_zero"]):
        with pytest.raises(DomainViolation):
            sx.materialize(cu(np.array(bad, np.uint32)), dim)


# ------------------------------------------------------- oracle, seeded ---
@pytest.mark.parametrize("dtype,npdt", [(torch.uint16, np.uint16), (torch.uint32, np.uint32),
                                        (torch.uint64, np.uint64), (torch.float32, np.float32),
                                        (torch.int64, np.int64)])
def test_gather_widths_ragged_and_unaligned(sx, oracle, dtype, npdt):
    rng = np.random.default_rng(11)
    d = 5003
    dim_np = rng.integers(0, 2**63, size=d, dtype=np.uint64).astype(npdt) if npdt != np.float32 \
        else rng.standard_normal(d).astype(np.float32)
    dim = cu(dim_np)
    for n in [0, 1, 3, 4, 5, 7, 8, 9, 63, 64, 1000, 4097, 100003]:
        fact_np = rng.integers(1, d + 1, size=n + 3, dtype=np.uint32)
        full = cu(fact_np)
        for off in range(4):  # misaligned starts exercise the scalar head path
            f = full[off: off + n]
            out = sx.materialize(f, dim)
            exp = dim_np[fact_np[off: off + n].astype(np.int64) - 1]
            assert np.array_equal(np_(out).view(np.uint8), exp.view(np.uint8)), (n, off)
            # misaligned output buffer too
            big = torch.empty(n + 1, dtype=dtype, device="cuda")
            sx.materialize(f, dim, out=big[1:])
            assert np.array_equal(np_(big[1:]).view(np.uint8), exp.view(np.uint8)), (n, off)


def test_domain_violation_first_row(sx):
    from paper_1910_10063_b200 import DomainViolation
    d = 1000
    fact = np.random.default_rng(1).integers(1, d + 1, size=1 << 20, dtype=np.uint32)
    fact[777777] = d + 5
    fact[900001] = 0
    with pytest.raises(DomainViolation) as e:
        sx.materialize(cu(fact), cu(np.arange(d, dtype=np.uint32)))
    assert e.value.row() == 777777 and e.value.value() == d + 5
    fact[123] = 0
    for op in (lambda f: sx.count_frequencies(f, d), lambda f: sx.aggregate_count(f, d),
               lambda f: sx.rebuild(f, d),
               lambda f: sx.select(f, sx.Bitmap(d)),
               lambda f: sx.aggregate_count_sum(f, torch.ones(f.numel(), dtype=torch.int64,
                                                              device="cuda"), d)):
        with pytest.raises(DomainViolation) as e:
            op(cu(fact))
        assert e.value.row() == 123 and e.value.value() == 0
    # context is clean again afterwards
    assert sx.count_frequencies(cu(np.array([1, 2], np.uint32)), 2).counts.sum().item() == 2


def test_counter_generator_matches_oracle(sx, oracle):
    for d, z, n, begin in [(1, 0.0, 100, 0), (1000, 1.0, 100000, 0), (1 << 16, 1.25, 1 << 20, 12345)]:
        cdf_np = sx.zipf_cdf(d, z)
        assert np.array_equal(cdf_np, oracle.zipf_cdf(d, z))
        r2i = sx.random_bijection(d, 42)
        out = sx.generate_zipf(cu(cdf_np), n, 42, rank_to_id=cu(r2i), row_begin=begin)
        exp = oracle.generate_zipf_counter(cdf_np, r2i, 42, begin, n)
        assert np.array_equal(np_(out), exp)


@pytest.mark.parametrize("d,n,z", [(1, 1000, 0.0), (4096, 1 << 20, 0.0), (1 << 16, 1 << 21, 1.25),
                                   (1 << 20, 1 << 21, 1.0), (70001, 3 << 19, 2.0),
                                   (1 << 22, 1 << 22, 0.5)])
def test_index_build_vs_oracle(sx, oracle, d, n, z):
    cdf = sx.zipf_cdf(d, z)
    r2i = sx.random_bijection(d, 7)
    fact = sx.generate_zipf(cu(cdf), n, 7, rank_to_id=cu(r2i))
    f_np = np_(fact)
    counts = oracle.count_frequencies(f_np, d)
    assert np.array_equal(np_(sx.count_frequencies(fact, d).counts), counts)
    assert np.array_equal(np_(sx.histogram_u32(fact, d)).astype(np.uint64), counts)
    off, rk = oracle.build_index(counts, n)
    idx = sx.rebuild(fact, d)
    assert np.array_equal(np_(idx.offsets), off)
    assert np.array_equal(np_(idx.ranks), rk)
    rec = sx.recode_fact(fact, idx)
    assert np.array_equal(np_(rec), oracle.recode_fact(f_np, rk))


def test_build_index_wide_counts(sx, oracle):
    """u64 counts above 2^32 take the 64-bit key path."""
    rng = np.random.default_rng(3)
    counts = rng.integers(0, 2**40, size=10000, dtype=np.uint64)
    counts[rng.integers(0, 10000, size=3000)] = 0
    counts[:50] = 7  # ties
    total = int(counts.sum())
    idx = sx.build_index(sx.FrequencyProfile(cu(counts), total))
    off, rk = oracle.build_index(counts, total)
    assert np.array_equal(np_(idx.offsets), off) and np.array_equal(np_(idx.ranks), rk)


@pytest.mark.parametrize("hot", [0, 1, 7, 1000])
def test_aggregate_vs_oracle(sx, oracle, hot):
    d, n = 1 << 18, (1 << 22) + 3
    cdf = sx.zipf_cdf(d, 1.0)
    fact = sx.generate_zipf(cu(cdf), n, 99)  # rank space: hot ids are small
    f_np = np_(fact)
    meas = np.random.default_rng(2).integers(1, 101, size=n, dtype=np.int64)
    c_exp, s_exp = oracle.aggregate_count_sum(f_np, meas.view(np.uint64), d)
    c, s = sx.aggregate_count_sum(fact, cu(meas), d, hot_threshold=hot)
    assert np.array_equal(np_(c), c_exp) and np.array_equal(np_(s), s_exp)
    c, s = sx.aggregate_count_sum(fact[1:], cu(meas)[1:], d, hot_threshold=hot)  # unaligned
    c_exp, s_exp = oracle.aggregate_count_sum(f_np[1:], meas[1:].view(np.uint64), d)
    assert np.array_equal(np_(c), c_exp) and np.array_equal(np_(s), s_exp)
    c = sx.parallel_aggregate(fact, d, sx.ParallelPlan(threads=8, strategy=sx.AggStrategy.hybrid,
                                                       hot_threshold=max(hot, 1)))
    assert np.array_equal(np_(c), oracle.aggregate_count_sum(f_np, None, d)[0])


def test_select_gather_sum_vs_oracle(sx, oracle):
    d, n = 1 << 15, (1 << 21) + 17
    rng = np.random.default_rng(4)
    cat = rng.integers(0, 1000, size=d, dtype=np.int32)
    price = np.exp(3 + rng.standard_normal(d)).astype(np.float32)
    supp = rng.integers(0, 2**63, size=d, dtype=np.uint64)
    flag = rng.integers(0, 2**16, size=d, dtype=np.uint16)
    cdf = sx.zipf_cdf(d, 1.0)
    r2i = sx.random_bijection(d, 5)
    fact = sx.generate_zipf(cu(cdf), n, 5, rank_to_id=cu(r2i))
    bm = sx.build_bitmap_lt(cu(cat), 100)
    got = sx.select_gather_sum(fact, bm, cu(cat), cu(price), cu(supp), cu(flag), 1000, base=3)
    exp = oracle.select_gather_sum(np_(fact), np_(bm.words), cat, price, supp, flag, 1000, base=3)
    for g, e in zip(got[:5], exp[:5]):
        assert np.array_equal(np_(g), e)
    s, se = np_(got[5]), exp[5]
    assert np.allclose(s, se, rtol=1e-6, atol=0)  # fp64 sums, order differs
    # selection alone equals the oracle's select, also in the reordered space
    assert np.array_equal(np_(sx.select(fact, bm)), oracle.select_offsets(np_(fact), np_(bm.words), d))


@pytest.mark.parametrize("case", ["neg", "wide", "nan", "zero", "many_cats", "unaligned",
                                  "ragged", "dense", "mixed_density", "unaligned_dims"])
def test_select_gather_sum_paths(sx, oracle, case):
    """Fixed-point category sums (default) and the on-device fp64 fallback
    (non-finite price, exponent span > 2^30, > 4096 categories), signed
    prices, unaligned and ragged FK columns, and selections dense enough that
    slices overflow pass 1's compacted entries (re-derived in pass 2)."""
    d = 1 << 14
    n = (1 << 20) + (4093 if case == "ragged" else 0)
    rng = np.random.default_rng(11)
    ncat = 5000 if case == "many_cats" else 1000
    cat = rng.integers(0, ncat, size=d, dtype=np.int32)
    price = np.exp(3 + rng.standard_normal(d)).astype(np.float32)
    if case == "neg":
        price *= np.where(rng.random(d) < 0.5, -1, 1).astype(np.float32)
    elif case == "wide":
        price = np.exp2(rng.uniform(-20, 20, size=d)).astype(np.float32)
    elif case == "nan":
        price[np.flatnonzero(cat < 100)[3]] = np.nan
    elif case == "zero":
        price[:] = 0
    supp = rng.integers(0, 2**63, size=d, dtype=np.uint64)
    flag = rng.integers(0, 2**16, size=d, dtype=np.uint16)
    fact = sx.generate_zipf(cu(sx.zipf_cdf(d, 1.0)), n + 1, 7)
    fact = fact[1:] if case == "unaligned" else fact[:n]
    thr = {"many_cats": 700, "dense": 1000, "mixed_density": 250}.get(case, 100)
    bm = sx.build_bitmap_lt(cu(cat), thr)
    dcols = [cu(cat), cu(price), cu(supp), cu(flag)]
    if case == "unaligned_dims":  # dimension columns off their 16-byte alignment (scalar packing)
        dcols = [torch.cat([c[:1], c])[1:] for c in dcols]
    got = sx.select_gather_sum(fact, bm, *dcols, ncat, base=5)
    exp = oracle.select_gather_sum(np_(fact), np_(bm.words), cat, price, supp, flag, ncat, base=5)
    for g, e in zip(got[:5], exp[:5]):  # bit-exact (NaN payloads included)
        assert np.array_equal(np_(g).view(np.uint8), np.ascontiguousarray(e).view(np.uint8))
    s, se = np_(got[5]), exp[5]
    assert np.allclose(s, se, rtol=1e-6, atol=0, equal_nan=True)
    if case == "nan":
        assert np.isnan(s).sum() == 1


@pytest.mark.parametrize("thr", [100, 1000, 3])
def test_select_many_tiles(sx, oracle, thr):
    """2^25 + 12345 rows (thousands of slice groups per CTA, a ragged last
    slice), sparse / all-selected / nearly empty selections, and a capacity
    below the selected count (rows past it are counted, not written; the
    category sums still cover every selected row)."""
    d, n = 1 << 20, (1 << 25) + 12345
    rng = np.random.default_rng(thr)
    cat = rng.integers(0, 1000, size=d, dtype=np.int32)
    price = np.exp(3 + rng.standard_normal(d)).astype(np.float32)
    supp = rng.integers(0, 2**63, size=d, dtype=np.uint64)
    flag = rng.integers(0, 2**16, size=d, dtype=np.uint16)
    fact = sx.generate_zipf(cu(sx.zipf_cdf(d, 1.0)), n, 17)
    bm = sx.build_bitmap_lt(cu(cat), thr)
    f_np = np_(fact)
    exp_off = oracle.select_offsets(f_np, np_(bm.words), d, base=9)
    assert np.array_equal(np_(sx.select(fact, bm, base=9)), exp_off)
    got = sx.select_gather_sum(fact, bm, cu(cat), cu(price), cu(supp), cu(flag), 1000, base=9)
    exp = oracle.select_gather_sum(f_np, np_(bm.words), cat, price, supp, flag, 1000, base=9)
    for g, e in zip(got[:5], exp[:5]):
        assert np.array_equal(np_(g), e)
    assert np.allclose(np_(got[5]), exp[5], rtol=1e-6, atol=0)
    if thr == 100:  # truncated output: the first `cap` rows written, the count exact
        cap = len(exp_off) // 3
        out = (torch.empty(cap, dtype=torch.uint32, device="cuda"),
               torch.empty(cap, dtype=torch.int32, device="cuda"),
               torch.empty(cap, dtype=torch.float32, device="cuda"),
               torch.empty(cap, dtype=torch.uint64, device="cuda"),
               torch.empty(cap, dtype=torch.uint16, device="cuda"),
               torch.empty(1000, dtype=torch.float64, device="cuda"),
               torch.zeros(1, dtype=torch.uint64, device="cuda"))
        sx.select_gather_sum(fact, bm, cu(cat), cu(price), cu(supp), cu(flag), 1000, base=9,
                             out=out, sync=False)
        sx.context(0).sync()
        assert int(out[6].item()) == len(exp_off)
        for g, e in zip(out[:5], exp[:5]):
            assert np.array_equal(np_(g), e[:cap])
        assert np.allclose(np_(out[5]), exp[5], rtol=1e-6, atol=0)  # sums cover every row


@pytest.mark.parametrize("z", [1.0, 0.0])
def test_recode_large_rank_table(sx, z):
    """recode_fact for a rank table beyond half of L2 (D = 2^24 + 3, >= 4 rows
    per id): the hottest ids' ranks come from each CTA's shared-memory table,
    the rest from the rank table -- against numpy on an unaligned FK column
    (scalar head and tail rows), then the first out-of-domain row."""
    from paper_1910_10063_b200 import DomainViolation
    d = (1 << 24) + 3
    n = 4 * d + 1001
    fact = sx.generate_zipf(cu(sx.zipf_cdf(d, z)), n + 1, 29,
                            rank_to_id=cu(sx.random_bijection(d, 29)))[1:]
    idx = sx.rebuild(fact, d)
    out = torch.empty(n + 1, dtype=torch.uint32, device="cuda")[1:]  # same 16-byte phase
    got = np_(sx.recode_fact(fact, idx, out=out))
    exp = np_(idx.ranks)[np_(fact).astype(np.int64) - 1]
    assert np.array_equal(got, exp)
    bad = fact.clone()
    bad[n - 2] = d + 7
    bad[12345] = 0
    with pytest.raises(DomainViolation) as e:
        sx.recode_fact(bad, idx, out=out)
    assert e.value.row() == 12345 and e.value.value() == 0


def test_reorder_invariants_at_scale(sx):
    """Size-independent properties at 2^26 rows: gather equality across
    layouts, rank-space counts map back through offsets, multiset of counts
    preserved, bijection."""
    d, n = 1 << 22, 1 << 26
    cdf = cu(sx.zipf_cdf(d, 1.0))
    r2i = cu(sx.random_bijection(d, 42))
    fact = sx.generate_zipf(cdf, n, 42, rank_to_id=r2i)
    idx = sx.rebuild(fact, d)
    off = idx.offsets.to(torch.int64)
    rk = idx.ranks.to(torch.int64)
    assert torch.equal(rk[off - 1], torch.arange(1, d + 1, device="cuda"))
    rec = sx.recode_fact(fact, idx)
    dim = torch.randint(0, 2**62, (d,), dtype=torch.int64, device="cuda")
    dperm = sx.permute_dimension(dim, idx)
    assert torch.equal(sx.materialize(fact, dim), sx.materialize(rec, dperm))
    c_rand = sx.aggregate_count(fact, d).to(torch.int64)
    c_freq = sx.aggregate_count(rec, d).to(torch.int64)
    assert torch.equal(c_freq, c_rand[off - 1])
    assert bool((c_freq[:-1] >= c_freq[1:]).all())  # frequency-sorted
    assert int(c_freq.sum()) == n


def test_aggregate_packed_tail_exactness(sx):
    """The packed tail accumulator (count << 40 | sum) must stay exact through
    sum-field carries, count-field wraps and wide (>= 2^32) measures."""
    n = (1 << 24) + 1000
    fact = torch.full((n,), 2, dtype=torch.int32, device="cuda").view(torch.uint32)
    meas = torch.full((n,), 2**32 - 1, dtype=torch.int64, device="cuda")
    c, s = sx.aggregate_count_sum(fact, meas, 3, hot_threshold=1)  # id 2 is a tail key
    assert int(c[1].item()) == n
    assert int(s[1].view(torch.int64).item()) & (2**64 - 1) == (n * (2**32 - 1)) % 2**64
    rng = np.random.default_rng(8)
    m = rng.integers(0, 2**63, size=200000, dtype=np.int64)
    m[::3] = rng.integers(0, 100, size=len(m[::3]))
    f = rng.integers(1, 50, size=200000, dtype=np.uint32)
    c, s = sx.aggregate_count_sum(cu(f), cu(m), 49, hot_threshold=5)
    ce = np.bincount(f.astype(np.int64) - 1, minlength=49).astype(np.uint64)
    se = np.zeros(49, np.uint64)
    np.add.at(se, f.astype(np.int64) - 1, m.view(np.uint64))
    assert np.array_equal(np_(c), ce) and np.array_equal(np_(s), se)


@pytest.mark.parametrize("bucketed", [0, 1, 2])
@pytest.mark.parametrize("case", ["zipf", "uniform", "one_bucket"])
def test_histogram_bucketed_large_domain(sx, oracle, case, bucketed):
    """Domains whose counters exceed half of L2: packed 16-bit cold counters
    (mode 0, default), per-tile key-range staging (1; 'one_bucket' overflows a
    bucket and exercises its fallback) and direct counters (2)."""
    # u64 counters of D=2^26 (count_frequencies, 512 MiB) exceed 3x L2: mode 0 packs
    # them; the u32 ones (histogram_u32, 256 MiB) take the direct path
    d, n = 1 << 26, (1 << 22) + 5
    rng = np.random.default_rng(17)
    if case == "zipf":
        cdf = sx.zipf_cdf(d, 1.1)
        f = np.ascontiguousarray(np_(sx.generate_zipf(cu(cdf), n, 3, rank_to_id=cu(sx.random_bijection(d, 3)))))
    elif case == "uniform":
        f = rng.integers(1, d + 1, size=n, dtype=np.uint32)
    else:
        f = rng.integers(1, 32769, size=n, dtype=np.uint32)
    exp = oracle.count_frequencies(f, d)
    ctx = sx.context(0)
    ctx.check(ctx.lib.skx_set_histogram_mode(ctx.handle, bucketed))
    assert np.array_equal(np_(sx.count_frequencies(cu(f), d).counts), exp)
    assert np.array_equal(np_(sx.histogram_u32(cu(f), d)).astype(np.uint64), exp)
    idx = sx.rebuild(cu(f), d)
    ctx.check(ctx.lib.skx_set_histogram_mode(ctx.handle, 0))
    off, rk = oracle.build_index(exp, n)
    assert np.array_equal(np_(idx.offsets), off) and np.array_equal(np_(idx.ranks), rk)


@pytest.mark.parametrize("mode", [0, 1, 2])
@pytest.mark.parametrize("z", [0.0, 0.8])
def test_aggregate_large_domain_modes(sx, oracle, mode, z):
    """Tail pairs larger than half of L2: packed tail (default), the staged
    per-bucket path (uniform data overflows the buckets -> fallback) and the
    direct pair reductions."""
    d, n = 1 << 23, (1 << 22) + 3
    fact = sx.generate_zipf(cu(sx.zipf_cdf(d, z)), n, 21)  # rank space
    meas = np.random.default_rng(9).integers(1, 101, size=n, dtype=np.int64)
    ctx = sx.context(0)
    ctx.check(ctx.lib.skx_set_aggregate_mode(ctx.handle, mode))
    try:
        c, s = sx.aggregate_count_sum(fact, cu(meas), d)
    finally:
        ctx.check(ctx.lib.skx_set_aggregate_mode(ctx.handle, 0))
    ce, se = oracle.aggregate_count_sum(np_(fact), meas.view(np.uint64), d)
    assert np.array_equal(np_(c), ce) and np.array_equal(np_(s), se)


@pytest.mark.parametrize("case", ["big_measure", "count_wrap", "sum_carry", "mixed",
                                  "far_count_wrap", "far_sum_carry", "far_ok", "hot_lo_wrap",
                                  "hot_wide"])
def test_aggregate_packed_tail_fallback(sx, oracle, case):
    """The packed mode must detect every overflow on the device and redo the
    call exactly: measures >= 2^16, a cold key with >= 2^24 rows (count field
    wraps), a cold key whose sum reaches 2^40 -- and hot keys whose 32-bit
    sum-lo bins wrap within a CTA or take measures >= 2^32 (carried to the
    global sums)."""
    d, hot = 1000, 16
    rng = np.random.default_rng(5)
    if case.startswith("far"):
        # domains > 2^22 keep ids >= 2^18 in 4-byte accumulators (count 11 bits, sum 21 bits)
        d = (1 << 22) + 4099
        n = 200_003
        fact = rng.integers(1, d + 1, size=n, dtype=np.uint32)
        meas = rng.integers(1, 101, size=n, dtype=np.int64)
        if case == "far_count_wrap":
            fact[:5000] = 3_000_000  # 5000 rows > 2047 on one far key
        elif case == "far_sum_carry":
            fact[:100] = 3_000_001
            meas[:100] = 60000  # sum 6e6 >= 2^21 on one far key
    elif case == "big_measure":
        n = 100_003
        fact = rng.integers(1, d + 1, size=n, dtype=np.uint32)
        meas = rng.integers(0, 2**63, size=n, dtype=np.int64)
    elif case == "count_wrap":
        n = (1 << 24) + 77
        fact = np.full(n, 500, np.uint32)
        fact[::3] = rng.integers(1, d + 1, size=len(fact[::3]), dtype=np.uint32)
        fact[: (1 << 24) + 5] = 500
        meas = np.ones(n, np.int64)
    elif case == "sum_carry":
        n = (1 << 25) + 2
        fact = np.full(n, 700, np.uint32)
        meas = np.full(n, 65535, np.int64)
    elif case == "hot_lo_wrap":  # ~28 K rows per CTA of ~2^31 each on hot keys: bins wrap
        n = (1 << 22) + 9
        fact = rng.integers(1, 4, size=n, dtype=np.uint32)
        meas = rng.integers(2**30, 2**31, size=n, dtype=np.int64)
    elif case == "hot_wide":
        n = 300_007
        fact = rng.integers(1, d + 1, size=n, dtype=np.uint32)
        meas = rng.integers(1, 101, size=n, dtype=np.int64)
        meas[fact <= hot] = rng.integers(2**32, 2**40, size=int((fact <= hot).sum()))
    else:
        n = 1 << 20
        fact = rng.integers(1, d + 1, size=n, dtype=np.uint32)
        meas = rng.integers(1, 101, size=n, dtype=np.int64)
        meas[12345] = 1 << 40  # one cold row that cannot be packed
    c, s = sx.aggregate_count_sum(cu(fact), cu(meas), d, hot_threshold=hot)
    ce, se = oracle.aggregate_count_sum(fact, meas.view(np.uint64), d)
    assert np.array_equal(np_(c), ce) and np.array_equal(np_(s), se)
    # u32 measure (the reference's own Column type) through the same path
    if case in ("count_wrap", "mixed"):
        m32 = meas.astype(np.uint32)
        c, s = sx.aggregate_count_sum(cu(fact), cu(m32), d, hot_threshold=hot)
        ce, se = oracle.aggregate_count_sum(fact, m32, d)
        assert np.array_equal(np_(c), ce) and np.array_equal(np_(s), se)


@pytest.mark.parametrize("case", ["wrap_and_carry", "wide", "threshold"])
def test_aggregate_warm_bins_exact(sx, oracle, case):
    """Packed mode's 4-byte warm bins (ids past the 1024 hottest, count << 22 |
    sum in one shared word): a warm key with tens of thousands of rows per CTA
    (the count field wraps, the sum field carries) and measures >= 2^22 (sent
    to the exact global pair) stay exact; a caller's hot threshold bounds the
    warm range."""
    d = 70000
    rng = np.random.default_rng(31)
    n = (1 << 22) + 13
    fact = rng.integers(1, d + 1, size=n, dtype=np.uint32)
    fact[: n // 2] = 2000  # a warm key: ~14 K rows per CTA
    meas = rng.integers(150, 250, size=n, dtype=np.int64)
    hot = 0
    if case == "wide":
        meas[::7] = rng.integers(1 << 22, 1 << 40, size=len(meas[::7]))
        meas[::7] = np.where(fact[::7] < 50000, meas[::7], 5)  # wide only on hot / warm keys
    elif case == "threshold":
        hot = 1500
        fact[n // 2: n // 2 + 100000] = 1400
    c, s = sx.aggregate_count_sum(cu(fact), cu(meas), d, hot_threshold=hot)
    ce, se = oracle.aggregate_count_sum(fact, meas.view(np.uint64), d)
    assert np.array_equal(np_(c), ce) and np.array_equal(np_(s), se)


def test_cache_model_vs_reference_fixtures(sx):
    """Cache model on the device (csrc/cachemodel.cu) against the reference's
    outputs: line_frequencies and trace_from_column bit-exact,
    estimate_hit_rate to rounding (parallel prefix sums)."""
    import json
    import os
    z = np.load(os.path.join(os.path.dirname(__file__), "golden", "ref_cachemodel.npz"))
    meta = json.loads(bytes(z["meta"]).decode())
    for i, m in enumerate(meta):
        geom = sx.CacheGeometry(1, m["line_bytes"], m["element_bytes"])
        layout = sx.Layout.freq if m["layout"] == "freq" else sx.Layout.rand
        lf = sx.line_frequencies(cu(z[f"c{i}_value_freqs"]), layout, geom, m["seed"])
        assert np.array_equal(np_(lf), z[f"c{i}_line_freqs"]), i
        for s, exp in zip(m["caches"], m["estimate"]):
            got = sx.estimate_hit_rate(lf, s)
            assert got == pytest.approx(exp, rel=1e-9, abs=1e-15), (i, s)
        tr = sx.trace_from_column(cu(z[f"c{i}_fact"]), geom)
        assert np.array_equal(np_(tr), z[f"c{i}_trace"]), i
    from paper_1910_10063_b200 import DomainViolation
    with pytest.raises(DomainViolation) as e:  # cachemodel.cpp:180: id 0 at row 1
        sx.trace_from_column(cu(np.array([3, 0, 1], np.uint32)), sx.CacheGeometry(1, 64, 4))
    assert e.value.row() == 1 and e.value.value() == 0


@pytest.mark.parametrize("layout", ["freq", "rand"])
def test_cache_model_at_scale_vs_oracle(sx, oracle, layout):
    """2^22 keys, Zipf(1.0), B200 L2-like geometry: the device model equals
    the oracle (bit-exact lines, estimate to rounding)."""
    d = 1 << 22
    vf = oracle.zipf_frequencies(d, 1.0)
    lf_o = oracle.line_frequencies(vf, layout, 128, 8, 42)
    geom = sx.CacheGeometry(1, 128, 8)
    lf = sx.line_frequencies(cu(vf), sx.Layout[layout], geom, 42)
    assert np.array_equal(np_(lf), lf_o)
    for s in (1 << 10, 1 << 14, 1 << 17):
        assert sx.estimate_hit_rate(lf, s) == pytest.approx(oracle.estimate_hit_rate(lf_o, s),
                                                            rel=1e-9)


def test_histogram_c16_wrap_fallback(sx, oracle):
    """Packed 16-bit cold counters: fill every CTA's hash table with distinct
    keys first, then send > 2^16 rows of one key down the cold path -- the
    wrap must be caught on the device and the call redone exactly."""
    d = 1 << 27  # u32 counters of 512 MiB: beyond 3x L2, the packed path is on
    n = 1 << 26
    fact = np.full(n, d, np.uint32)  # the heavy key, cold once the tables are full
    fill = 2 * 444 * 4096  # two CTA iterations of distinct keys for every CTA
    # the fill keys share the heavy key's key-range pass (the last one), so
    # they are what the tables hold when the heavy key arrives
    fact[:fill] = np.arange(d - fill, d, dtype=np.uint32)
    exp = oracle.count_frequencies(fact, d)
    got = np_(sx.count_frequencies(cu(fact), d).counts)
    assert np.array_equal(got, exp)
    assert np.array_equal(np_(sx.histogram_u32(cu(fact), d)).astype(np.uint64), exp)


def test_histogram_c16_key_range_passes(sx, oracle):
    """Packed cold counters at D = 2^27 run as key-range passes (3 slices of
    the domain): a skewed original-layout column, ids spread over every pass,
    plus the first and last id of the domain."""
    d, n = 1 << 27, (1 << 24) + 5
    r2i = sx.random_bijection(d, 17)
    fact = sx.generate_zipf(cu(sx.zipf_cdf(d, 1.0)), n, 17, rank_to_id=cu(r2i))
    f_np = np_(fact).copy()
    f_np[:3] = [1, d, d // 3]
    exp = oracle.count_frequencies(f_np, d)
    assert np.array_equal(np_(sx.histogram_u32(cu(f_np), d)).astype(np.uint64), exp)
    f_np[n - 2] = d + 1  # violation reported once, by the first pass
    from paper_1910_10063_b200 import DomainViolation
    with pytest.raises(DomainViolation) as e:
        sx.count_frequencies(cu(f_np), d)
    assert e.value.row() == n - 2 and e.value.value() == d + 1


@pytest.mark.parametrize("d,n,hot", [((1 << 22) + 1, 1000, 0), ((1 << 22) + 1, (1 << 20) + 7, 0),
                                     ((1 << 23) + 17, (1 << 21) + 3, 5000), (3, 1, 0),
                                     ((1 << 24), 1 << 22, 0)])
def test_aggregate_tier_edges(sx, oracle, d, n, hot):
    """Domain sizes at and around the far-tier switch (D > 2^22), tiny inputs,
    an explicit hot threshold together with the far tier, both measure widths."""
    rng = np.random.default_rng(d ^ n)
    fact = sx.generate_zipf(cu(sx.zipf_cdf(d, 0.9)), n, 13)  # rank space, skewed
    for dt in (np.int64, np.uint32):
        meas = rng.integers(0, 3000, size=n).astype(dt)
        c, s = sx.aggregate_count_sum(fact, cu(meas), d, hot_threshold=hot)
        ce, se = oracle.aggregate_count_sum(np_(fact), meas.view(np.uint64) if dt == np.int64 else meas, d)
        assert np.array_equal(np_(c), ce) and np.array_equal(np_(s), se)
    c = sx.aggregate_count(fact, d, hot_threshold=hot)
    assert np.array_equal(np_(c), oracle.aggregate_count_sum(np_(fact), None, d)[0])


@pytest.mark.parametrize("n", [1, 255, 256, 257, 4097, 8191, 8192, 8193, 3 * 8192 + 5])
def test_select_tiny_and_slice_edges(sx, oracle, n):
    """Row counts around the 256-row slice and 4-row vector boundaries."""
    d = 1000
    rng = np.random.default_rng(n)
    fact = rng.integers(1, d + 1, size=n, dtype=np.uint32)
    bm = sx.build_bitmap_lt(cu(rng.integers(0, 1000, size=d, dtype=np.int32)), 300)
    got = np_(sx.select(cu(fact), bm))
    assert np.array_equal(got, oracle.select_offsets(fact, np_(bm.words), d))


@pytest.mark.parametrize("off", [0, 4, 8])
def test_select_fast_path_alignment_and_tail(sx, oracle, off):
    """Pass 1's fast path: 32-byte aligned (one 256-bit load per lane), 16-byte
    aligned (two 128-bit loads), a partial last slice, a mixed-density bitmap,
    and the first out-of-domain row inside the last slice."""
    from paper_1910_10063_b200 import DomainViolation
    d, n = 1 << 14, (1 << 18) + 77
    rng = np.random.default_rng(off)
    buf = cu(rng.integers(1, d + 1, size=n + off, dtype=np.uint32))
    fact = buf[off:]
    cat = rng.integers(0, 1000, size=d, dtype=np.int32)
    cat[:64] = 0  # the hottest-looking ids always selected: dense and sparse slices mix
    f_np = np_(fact)
    f_np[: 1 << 12] = rng.integers(1, 65, size=1 << 12, dtype=np.uint32)
    fact.copy_(cu(f_np))
    bm = sx.build_bitmap_lt(cu(cat), 100)
    got = np_(sx.select(fact, bm, base=5))
    assert np.array_equal(got, oracle.select_offsets(f_np, np_(bm.words), d, base=5))
    bad = f_np.copy()
    bad[n - 3] = d + 1
    bad[n - 1] = 0
    with pytest.raises(DomainViolation) as e:
        sx.select(cu(bad), bm)
    assert e.value.row() == n - 3 and e.value.value() == d + 1


@pytest.mark.parametrize("case", ["boundary", "all_big", "no_big", "one_big"])
def test_build_index_small_count_pass(sx, oracle, case):
    """The counting pass places ids with count < 255 directly and sorts only
    the ids with count >= 255: counts around the 254/255 boundary with ties,
    every count big, no big count at all (total >= 256), a single big id."""
    rng = np.random.default_rng(5)
    d = 50000
    if case == "boundary":
        counts = rng.choice(np.array([0, 1, 2, 253, 254, 255, 256, 511, 70000], np.uint64), size=d)
    elif case == "all_big":
        counts = rng.integers(255, 1 << 20, size=d, dtype=np.uint64)
        counts[::7] = 300  # ties
    elif case == "no_big":
        counts = rng.integers(0, 255, size=d, dtype=np.uint64)
    else:
        counts = rng.integers(0, 3, size=d, dtype=np.uint64)
        counts[d // 2] = 1 << 24
    total = int(counts.sum())
    idx = sx.build_index(sx.FrequencyProfile(cu(counts), total))
    off, rk = oracle.build_index(counts, total)
    assert np.array_equal(np_(idx.offsets), off) and np.array_equal(np_(idx.ranks), rk)
    idx32 = sx.build_index(sx.FrequencyProfile(cu(counts.astype(np.uint32)), total))
    assert np.array_equal(np_(idx32.offsets), off)


@pytest.mark.parametrize("policy", [129, 2177, 4225, 1, 0, 129 | 8192])
def test_gather_output_store_policies(sx, policy):
    """Every output-store variant of the gather (128-bit .cs stores, 8 KB
    shared-memory-staged cp.async.bulk stores, 256-bit stores, plain) writes
    the same bytes, for ragged sizes, partial CTA chunks and misaligned heads."""
    ctx = sx.context(0)
    rng = np.random.default_rng(policy)
    d = 70001
    dim_np = rng.integers(0, 2**63, size=d, dtype=np.uint64)
    dim = cu(dim_np)
    try:
        ctx.set_gather_policy(policy)
        for n in [1, 5, 1023, 1024 * 9 + 3, 1 << 20, (1 << 22) + 777, 40_000_003]:
            fact_np = rng.integers(1, d + 1, size=n + 1, dtype=np.uint32)
            full = cu(fact_np)
            for off in (0, 1):
                out = sx.materialize(full[off: off + n], dim)
                exp = dim_np[fact_np[off: off + n].astype(np.int64) - 1]
                assert np.array_equal(np_(out).view(np.uint64), exp), (policy, n, off)
    finally:
        ctx.set_gather_policy(129 | 8192)


@pytest.mark.parametrize("npdt", [np.uint32, np.uint64])
def test_gather_partitioned(sx, oracle, npdt):
    """The partitioned gather (policy bit 8192): cold rows radix-partitioned by
    key range, their values fetched slice by slice and merged back at the slots
    each chunk recorded.  Same bytes as the one-pass kernel (policy 129) and
    numpy with the path forced on (bit 16384) and under the plan's own gate,
    for Zipf, uniform and hot-only ids, ragged sizes with partial last chunks,
    misaligned heads, one and ~30 partitions, and the first bad row."""
    from paper_1910_10063_b200 import DomainViolation
    ctx = sx.context(0)
    rng = np.random.default_rng(11)
    w = np.dtype(npdt).itemsize
    hot = (32 << 20) // w                      # the direct prefix (SKX_PG_HOT_MB)
    try:
        for d in [2 * hot + 1, (1 << 30) // w + 12345]:   # 1 and ~30 partitions
            dim_np = rng.integers(0, np.iinfo(npdt).max, size=d, dtype=npdt)
            dim = cu(dim_np)
            cdf = oracle.zipf_cdf(d, 0.9)
            cases = [("zipf", oracle.generate_zipf_counter(cdf, None, 7, 0, (1 << 22) + 8192 * 3 + 5)),
                     ("uniform", rng.integers(1, d + 1, size=(1 << 23) + 3, dtype=np.uint32)),
                     ("hot_only", rng.integers(1, hot // 2, size=(1 << 22) + 1, dtype=np.uint32))]
            del cdf
            for name, fact_np in cases:
                n = fact_np.size - 1
                full = cu(fact_np)
                for pol in (129 | 8192 | 16384, 129 | 8192):
                    ctx.set_gather_policy(pol)
                    for off in (0, 1, 3):
                        exp = dim_np[fact_np[off: off + n].astype(np.int64) - 1]
                        # under the gate: the first launch plans beside the one-pass
                        # kernel, the second follows the landed plan
                        for rep in range(1 if pol & 16384 else 2):
                            out = sx.materialize(full[off: off + n], dim)
                            assert np.array_equal(np_(out).view(npdt), exp), (d, name, off, pol, rep)
                            plan = ctx.gather_last_plan()
                            if pol & 16384:
                                # a fresh (aligned) output behind a misaligned FK head cannot
                                # take 16-byte stores: those launches stay one-pass
                                assert plan["partitioned"] == (off == 0), (d, name, off)
                            else:
                                assert plan["partitioned"] == (rep == 1 and plan["plan_partitioned"])
                                if name == "hot_only":
                                    assert not plan["plan_partitioned"]
                                    assert plan["sample_first_touch"] == 0
                ctx.set_gather_policy(129)
                one = sx.materialize(full[1: 1 + n], dim)
                assert np.array_equal(np_(one).view(npdt),
                                      dim_np[fact_np[1: 1 + n].astype(np.int64) - 1])
            # first bad row, path forced on and under the gate
            for pol in (129 | 8192 | 16384, 129 | 8192):
                ctx.set_gather_policy(pol)
                for name, hi in (("cold", d), ("hot", hot // 2)):
                    fact_np = rng.integers(1, hi + 1, size=(1 << 22) + 7, dtype=np.uint32)
                    fact_np[3_000_001] = d + 9
                    fact_np[3_500_000] = 0
                    with pytest.raises(DomainViolation) as e:
                        sx.materialize(cu(fact_np), dim)
                    assert e.value.row() == 3_000_001 and e.value.value() == d + 9, (name, pol)
            del dim, dim_np
            torch.cuda.empty_cache()
    finally:
        ctx.set_gather_policy(129 | 8192)


@pytest.mark.parametrize("npdt", [np.uint32, np.uint64])
def test_gather_plan_gate(sx, oracle, npdt):
    """The plan's decisions (made beside a column's first launch, followed from
    the second) on the access patterns the index produces: uniform
    ids over a 1 GiB dimension with enough rows per line -> partitioned; a
    strongly skewed scattered column (recode at s=1.25), in-order walks
    (permute over count ties: ascending ids with small random gaps) and too
    few rows per dimension line -> one pass.
    The result is checked against numpy either way."""
    ctx = sx.context(0)
    rng = np.random.default_rng(5)
    w = np.dtype(npdt).itemsize
    d = (256 << 20) // w
    dim_np = rng.integers(0, np.iinfo(npdt).max, size=d, dtype=npdt)
    dim = cu(dim_np)
    n = 1 << 24                      # 8 rows per 128-byte line of the 256 MiB dimension
    cdf = oracle.zipf_cdf(d, 1.25)
    perm = oracle.random_bijection(d, 3)
    walk = (np.arange(n, dtype=np.uint64) * 3 % d + 1).astype(np.uint32)
    cases = [("uniform", rng.integers(1, d + 1, size=n, dtype=np.uint32), True),
             ("zipf1.25_scattered", oracle.generate_zipf_counter(cdf, perm, 9, 0, n), False),
             ("in_order", walk, False),
             ("tie_runs", (np.cumsum(rng.integers(1, 10, size=n)) % d + 1).astype(np.uint32), False),
             ("few_rows", rng.integers(1, d + 1, size=1 << 22, dtype=np.uint32), False)]
    for name, fact_np, want in cases:
        fact = cu(fact_np)
        ctx.set_gather_policy(129 | 8192)   # drops cached plans (the allocator reuses addresses)
        exp = dim_np[fact_np.astype(np.int64) - 1]
        before = ctx.launches()
        out = sx.materialize(fact, dim)
        assert ctx.launches() - before == 2, name          # one-pass kernel + plan kernel
        assert np.array_equal(np_(out).view(npdt), exp), name
        plan = ctx.gather_last_plan()
        assert not plan["partitioned"] and plan["plan_partitioned"] == want, (name, plan)
        # the same column again follows the landed plan: the four partitioned
        # kernels or the one-pass kernel alone, no plan kernel; same bytes
        before = ctx.launches()
        out2 = sx.materialize(fact, dim)
        assert ctx.launches() - before == (4 if want else 1), (name, ctx.launches() - before)
        assert np.array_equal(np_(out2).view(npdt), exp), name
        plan2 = ctx.gather_last_plan()
        assert plan2["partitioned"] == want and plan2["plan_partitioned"] == want, (name, plan2)
        assert plan2["sample_first_touch"] == plan["sample_first_touch"]
        # a rewritten column under a stale "partitioned" plan still gathers exactly
        if want:
            fact.view(torch.int32).copy_(cu(np.minimum(fact_np, 1000)).view(torch.int32))
            out3 = sx.materialize(fact, dim)
            assert np.array_equal(np_(out3).view(npdt), dim_np[np.minimum(fact_np, 1000).astype(np.int64) - 1])


@pytest.mark.parametrize("dtype,npdt", [(torch.uint32, np.uint32), (torch.int64, np.int64)])
def test_materialize_split_two_pass(sx, oracle, dtype, npdt):
    """materialize_split (operators.cpp:68-85): the two-pass device kernel
    (hot ids <= t gathered in pass 1, misses patched in pass 2) equals the
    one-pass gather for every threshold, ragged sizes; bad thresholds and
    out-of-domain rows raise like the reference."""
    from paper_1910_10063_b200 import DomainViolation, InvalidArgument
    rng = np.random.default_rng(5)
    d = 30011
    dim_np = rng.integers(0, 2**62, size=d, dtype=np.uint64).astype(npdt)
    dim = cu(dim_np)
    cdf = oracle.zipf_cdf(d, 1.0)
    for n in [1, 31, 33, 100003, (1 << 22) + 5]:
        fact_np = oracle.generate_zipf_counter(cdf, None, 3, 0, n)
        f = cu(fact_np)
        exp = oracle.gather(fact_np, dim_np)
        for t in [1, 7, 1000, d // 2, d]:
            got = sx.materialize_split(f, dim, t)
            assert np.array_equal(np_(got).view(npdt), exp), (n, t)
    f = cu(np.array([1, 2, 3], np.uint32))
    for t in (0, d + 1):
        with pytest.raises(InvalidArgument):
            sx.materialize_split(f, dim, t)
    bad = np.ones(5000, np.uint32)
    bad[4000], bad[4500] = d + 1, 0
    with pytest.raises(DomainViolation) as e:
        sx.materialize_split(cu(bad), dim, 10)
    assert e.value.row() == 4000 and e.value.value() == d + 1


def test_scratch_reserve_and_graph_capture(sx, oracle):
    """Scratch arenas are per stream and grow stream-ordered; skx_reserve grows
    them up front, which is what lets a scratch-using operator (the index
    build's sort) be captured in a CUDA Graph and replayed."""
    import ctypes as C
    ctx = sx.context(0)
    d, n = 1 << 16, 1 << 20
    rng = np.random.default_rng(8)
    fact_np = rng.integers(1, d + 1, size=n, dtype=np.uint32)
    fact = cu(fact_np)
    counts = sx.histogram_u32(fact, d)
    off = torch.empty(d, dtype=torch.uint32, device="cuda")
    rk = torch.empty_like(off)
    s = torch.cuda.Stream()
    sp = C.c_void_p(s.cuda_stream)

    def build():
        ctx.check(ctx.lib.skx_build_index_u32(ctx.handle, C.c_void_p(counts.data_ptr()), d, n,
                                              C.c_void_p(off.data_ptr()), C.c_void_p(rk.data_ptr()),
                                              sp))
    # a fresh stream has no arenas: growing one inside a capture is refused
    g = torch.cuda.CUDAGraph()
    import warnings
    with warnings.catch_warnings():
        warnings.simplefilter("ignore")  # the refused capture leaves an empty graph
        with pytest.raises(Exception):
            with torch.cuda.graph(g, stream=s):
                build()
    # reserve on that stream, then capture and replay
    ctx.check(ctx.lib.skx_reserve(ctx.handle, -1, 64 << 20, sp))
    got = (C.c_uint64 * 4)()
    ctx.check(ctx.lib.skx_scratch_bytes(ctx.handle, sp, got))
    assert min(got) >= 64 << 20
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        build()
    off.zero_()
    g.replay()
    torch.cuda.synchronize()
    ctx.sync(sp)
    eo, er = oracle.build_index(oracle.count_frequencies(fact_np, d), n)
    assert np.array_equal(np_(off), eo) and np.array_equal(np_(rk), er)


def test_gather_plan_in_graph_capture_and_two_streams(sx):
    """The gather's plan cache stays out of captured graphs (a captured launch
    over a partition-eligible column is the one-pass kernel alone: no plan
    kernel, no copy, no event), a forced partitioned launch captures once its
    scratch is reserved, and two streams of one context plan and follow their
    own columns independently."""
    import ctypes as C
    ctx = sx.context(0)
    rng = np.random.default_rng(21)
    d = (96 << 20) // 8                      # 96 MiB int64 dimension: eligible (> 2 x 32 MB)
    n = 1 << 23
    dim_np = rng.integers(0, 2**62, size=d, dtype=np.int64)
    dim = cu(dim_np)
    fact_np = rng.integers(1, d + 1, size=n, dtype=np.uint32)
    fact = cu(fact_np)
    exp = dim_np[fact_np.astype(np.int64) - 1]
    out = torch.empty(n, dtype=torch.int64, device="cuda")
    s = torch.cuda.Stream()
    sp = C.c_void_p(s.cuda_stream)

    def gather(stream_ptr, f=fact, o=out):
        ctx.check(ctx.lib.skx_gather_u64(ctx.handle, C.c_void_p(f.data_ptr()), f.numel(),
                                         C.c_void_p(dim.data_ptr()), d, C.c_void_p(o.data_ptr()),
                                         stream_ptr))
    try:
        ctx.set_gather_policy(129 | 8192)
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        before = ctx.launches()
        with torch.cuda.graph(g, stream=s):
            gather(sp)
        assert ctx.launches() - before == 1              # the one-pass kernel, nothing else
        out.zero_()
        g.replay()
        torch.cuda.synchronize()
        assert np.array_equal(np_(out), exp)
        # forced path: the records' scratch must exist before the capture
        ctx.set_gather_policy(129 | 8192 | 16384)
        ctx.check(ctx.lib.skx_reserve(ctx.handle, 1, 256 + (n // 8192 + 1) * 64 + n * 16 + 4096, sp))
        g2 = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g2, stream=s):
            gather(sp)
        for _ in range(2):
            out.zero_()
            g2.replay()
            torch.cuda.synchronize()
            assert np.array_equal(np_(out), exp)
        # two streams, two columns: uniform ids (partitioned from the second launch on) and
        # hot-only ids (one pass), interleaved
        ctx.set_gather_policy(129 | 8192)
        s2 = torch.cuda.Stream()
        sp2 = C.c_void_p(s2.cuda_stream)
        hot_np = rng.integers(1, 1000, size=n, dtype=np.uint32)
        hot = cu(hot_np)
        out2 = torch.empty_like(out)
        exp2 = dim_np[hot_np.astype(np.int64) - 1]
        torch.cuda.synchronize()
        for rep in range(3):
            out.zero_()
            out2.zero_()
            torch.cuda.synchronize()
            gather(sp)
            gather(sp2, hot, out2)
            p2 = ctx.gather_last_plan(sp2)
            torch.cuda.synchronize()
            assert np.array_equal(np_(out), exp) and np.array_equal(np_(out2), exp2), rep
            assert not p2["partitioned"] and not p2["plan_partitioned"]
        gather(sp)
        p1 = ctx.gather_last_plan(sp)
        assert p1["partitioned"] and p1["plan_partitioned"]
        ctx.sync(sp)
        ctx.sync(sp2)
    finally:
        ctx.set_gather_policy(129 | 8192)

"""Pins the CPU oracle (oracle/skx_oracle.c) before it is trusted as the
checker: against the reference's own known-answer vectors (golden/kat.json)
and against outputs of the unmodified reference library (golden/ref_cases.npz,
and live when oracle/_ref is built)."""
import numpy as np
import pytest

from conftest import words_from_bits
from oracle.oracle import DOMAIN, INVALID, OracleError


def test_kat_count_frequencies(oracle, kat):
    for c in kat["count_frequencies"]:
        assert oracle.count_frequencies(np.array(c["fact"], np.uint32), c["d"]).tolist() == c["counts"]
    for c in kat["count_frequencies_violation"]:
        with pytest.raises(OracleError) as e:
            oracle.count_frequencies(np.array(c["fact"], np.uint32), c["d"])
        assert (e.value.status, e.value.row, e.value.value) == (DOMAIN, c["row"], c["value"])


def _popularity(kat):
    pf = kat["popularity_fixture"]
    fact = np.concatenate([np.full(cnt, i, np.uint32) for i, cnt in pf["by_count"]])
    np.random.default_rng(99).shuffle(fact)
    return pf, fact


def test_kat_index(oracle, kat):
    pf, fact = _popularity(kat)
    off, rk = oracle.rebuild(fact, pf["d"])
    assert off.tolist() == pf["offsets"] and rk.tolist() == pf["ranks"]
    assert oracle.recode_fact(np.array(pf["recode_in"], np.uint32), rk).tolist() == pf["recode_out"]
    assert oracle.permute_dimension(np.array(pf["dim"], np.uint32), off).tolist() == pf["permuted_dim"]
    for c in kat["build_index"]:
        o, r = oracle.build_index(np.array(c["counts"], np.uint64), c["total"])
        assert o.tolist() == c["offsets"] and r.tolist() == c["ranks"]
    for c in kat["build_index_invalid"]:
        with pytest.raises(OracleError) as e:
            oracle.build_index(np.array(c["counts"], np.uint64), c["total"])
        assert e.value.status == INVALID
    c = kat["permute_length_mismatch"]
    off, _ = oracle.rebuild(np.array(c["fact"], np.uint32), c["d"])
    with pytest.raises(OracleError):
        oracle.permute_dimension(np.array(c["dim"], np.uint32), off)


def test_kat_operators(oracle, kat):
    c = kat["aggregate_count"]
    cnt, _ = oracle.aggregate_count_sum(np.array(c["fact"], np.uint32), None, c["d"])
    assert cnt.tolist() == c["counts"]
    c = kat["aggregate_sum"]
    _, s = oracle.aggregate_count_sum(np.array(c["fact"], np.uint32),
                                      np.array(c["measure"], np.uint32), c["d"])
    assert s.tolist() == c["sums"]
    for c in kat["select"]:
        w = words_from_bits(c["bits"], c["d"])
        assert oracle.select_offsets(np.array(c["fact"], np.uint32), w, c["d"]).tolist() == c["offsets"]
    c = kat["select_violation"]
    with pytest.raises(OracleError) as e:
        oracle.select_offsets(np.array(c["fact"], np.uint32), words_from_bits(c["bits"], c["d"]), c["d"])
    assert (e.value.row, e.value.value) == (c["row"], c["value"])
    g = kat["gather_edges"]
    dim = np.arange(10, 10 + g["d"], dtype=np.uint32)
    assert oracle.gather(np.array(g["empty"], np.uint32), dim).size == 0
    for bad in (g["bad_high"], g["bad_zero"]):
        with pytest.raises(OracleError):
            oracle.gather(np.array(bad, np.uint32), dim)


def test_kat_generator(oracle, kat):
    for c in kat["zipf_frequencies"]:
        p = oracle.zipf_frequencies(c["d"], c["z"]) * c["p_times"]
        assert np.allclose(p, c["scaled"], rtol=1e-12)


def test_kat_chunk_spans(oracle, kat):
    from paper_1910_10063_b200.skewdx import chunk_spans
    for n, t in kat["chunk_spans"]["cases"]:
        spans = oracle.chunk_spans(n, t)
        assert spans == chunk_spans(n, t)
        assert spans[0][0] == 0 and spans[-1][1] == n
        assert all(a[1] == b[0] for a, b in zip(spans, spans[1:]))
        lens = [e - b for b, e in spans]
        assert max(lens) - min(lens) <= 1


def test_oracle_matches_reference_fixtures(oracle, ref_cases):
    """Every array the reference produced is reproduced by the restatement."""
    for i in range(len(ref_cases)):
        c = ref_cases.case(i)
        d, seed = c["d"], c["seed"]
        fact = oracle.generate_fact_column_rand(d, c["n"], c["z"], seed)
        assert np.array_equal(fact, c["fact"]), i
        assert np.array_equal(oracle.count_frequencies(fact, d), c["counts"]), i
        off, rk = oracle.rebuild(fact, d)
        assert np.array_equal(off, c["offsets"]) and np.array_equal(rk, c["ranks"]), i
        rec = oracle.recode_fact(fact, rk)
        assert np.array_equal(rec, c["recoded"]), i
        assert np.array_equal(oracle.permute_dimension(c["dim"], off), c["dim_perm"]), i
        assert np.array_equal(oracle.gather(fact, c["dim"]), c["mat_rand"]), i
        assert np.array_equal(oracle.gather(rec, c["dim_perm"]), c["mat_freq"]), i
        cnt, s = oracle.aggregate_count_sum(rec, c["measure"], d)
        assert np.array_equal(cnt, c["counts_freq"]) and np.array_equal(s, c["sums"]), i
        assert np.array_equal(oracle.permute_bitmap(c["words"], d, off), c["words_perm"]), i
        assert np.array_equal(oracle.select_offsets(fact, c["words"], d), c["sel_rand"]), i
        assert np.array_equal(oracle.select_offsets(rec, c["words_perm"], d), c["sel_freq"]), i
        # the reorder invariants the reference tests rely on
        assert np.array_equal(c["mat_rand"], c["mat_freq"])
        assert np.array_equal(c["sel_rand"], c["sel_freq"])
        assert np.array_equal(c["counts_freq"], c["counts"][c["offsets"].astype(np.int64) - 1])


def test_oracle_matches_reference_live(oracle, reference):
    rng = np.random.default_rng(5)
    for _ in range(6):
        d = int(rng.integers(1, 3000))
        n = int(rng.integers(1, 20000))
        z = float(rng.integers(0, 250)) / 100
        seed = int(rng.integers(0, 2**63))
        f = reference.generate_fact_column(d, n, z, seed)
        assert np.array_equal(f, oracle.generate_fact_column_rand(d, n, z, seed))
        assert np.array_equal(reference.random_bijection(d, seed), oracle.random_bijection(d, seed))
        assert np.array_equal(reference.zipf_frequencies(d, z), oracle.zipf_frequencies(d, z))
        o1, r1 = reference.rebuild(f, d)
        o2, r2 = oracle.rebuild(f, d)
        assert np.array_equal(o1, o2) and np.array_equal(r1, r2)
        pc, shared = reference.parallel_aggregate(f, d, 4, 2, max(1, d // 3))
        assert np.array_equal(pc, oracle.count_frequencies(f, d))


def test_counter_generator_is_zipf(oracle):
    """The counter-based draw uses the reference's CDF and upper_bound; its
    empirical distribution follows Zipf (rank 1 share within 5 sigma)."""
    d, n = 1000, 200000
    cdf = oracle.zipf_cdf(d, 1.0)
    ranks = oracle.generate_zipf_counter(cdf, None, 42, 0, n)
    assert ranks.min() >= 1 and ranks.max() <= d
    p1 = oracle.zipf_frequencies(d, 1.0)[0]
    c1 = int((ranks == 1).sum())
    assert abs(c1 - n * p1) < 5 * np.sqrt(n * p1 * (1 - p1))
    # position-addressable: a shard equals the slice of the whole
    part = oracle.generate_zipf_counter(cdf, None, 42, 777, 1000)
    assert np.array_equal(part, ranks[777:1777])


# ---- the multi-threaded checker forms (skx_oracle_mt.c) used at BASELINE scale
# are pinned against the single-threaded restatement (and through it the KATs
# and reference fixtures above) on seeded inputs, including ragged spans,
# ties, zero counts and domain violations.
def test_mt_forms_equal_single_thread(oracle, kat, ref_cases):
    rng = np.random.default_rng(2024)
    for d, n, z in [(1, 17, 1.0), (97, 10007, 1.3), (5000, 300001, 1.0), (70000, 200003, 0.6)]:
        cdf = oracle.zipf_cdf(d, z)
        fact = oracle.generate_zipf_counter(cdf, oracle.random_bijection(d, 3), 3, 0, n)
        c1 = oracle.count_frequencies(fact, d)
        assert np.array_equal(oracle.count_frequencies_mt(fact, d), c1)
        off, rk = oracle.build_index(c1, n)
        off2, rk2 = oracle.build_index_radix(c1, n)
        assert np.array_equal(off, off2) and np.array_equal(rk, rk2)
        for dt in (np.uint16, np.uint32, np.uint64):
            dim = rng.integers(0, np.iinfo(dt).max, size=d, dtype=dt)
            assert np.array_equal(oracle.gather_mt(fact, dim), oracle.gather(fact, dim))
        meas = rng.integers(1, 101, size=n, dtype=np.uint64)
        ce, se = oracle.aggregate_count_sum(fact, meas, d)
        cm, sm = oracle.aggregate_count_sum_mt(fact, meas, d)
        assert np.array_equal(ce, cm) and np.array_equal(se, sm)
        cat = rng.integers(0, 1000, size=d, dtype=np.int32)
        price = np.exp(3 + rng.standard_normal(d)).astype(np.float32)
        supp = rng.integers(0, 2**63, size=d, dtype=np.uint64)
        flag = rng.integers(0, 2**16, size=d, dtype=np.uint16)
        words = oracle.build_bitmap_lt_i32(cat, 100)
        assert np.array_equal(words, words_from_bits(np.nonzero(cat < 100)[0], d))
        exp = oracle.select_gather_sum(fact, words, cat, price, supp, flag, 1000, base=11)
        got = oracle.select_gather_sum_mt(fact, words, cat, price, supp, flag, 1000, base=11)
        for g, e in zip(got[:5], exp[:5]):
            assert np.array_equal(g, e)
        assert np.allclose(got[5], exp[5], rtol=1e-12, atol=0)
    # radix build_index on tie-heavy profiles and the reference KATs
    for c in kat["build_index"]:
        o, r = oracle.build_index_radix(np.array(c["counts"], np.uint64), c["total"])
        assert o.tolist() == c["offsets"] and r.tolist() == c["ranks"]
    for c in kat["build_index_invalid"]:
        with pytest.raises(OracleError):
            oracle.build_index_radix(np.array(c["counts"], np.uint64), c["total"])
    for _ in range(5):
        cnt = rng.integers(0, 4, size=20000).astype(np.uint64) * rng.integers(0, 2, size=20000).astype(np.uint64)
        cnt[rng.integers(0, 20000, 50)] = rng.integers(1, 1 << 20, 50).astype(np.uint64)
        a = oracle.build_index(cnt)
        b = oracle.build_index_radix(cnt)
        assert np.array_equal(a[0], b[0]) and np.array_equal(a[1], b[1])
    for i in range(len(ref_cases)):
        c = ref_cases.case(i)
        assert np.array_equal(oracle.count_frequencies_mt(c["fact"], c["d"]), c["counts"])
        o, r = oracle.build_index_radix(c["counts"])
        assert np.array_equal(o, c["offsets"]) and np.array_equal(r, c["ranks"])
    # domain violations: the first offending row overall, whichever chunk it is in
    fact = np.full(100003, 3, np.uint32)
    fact[77777], fact[90000] = 0, 99
    assert oracle.find_domain_violation_mt(fact, 10) == 77777
    for fn in (lambda: oracle.count_frequencies_mt(fact, 10),
               lambda: oracle.gather_mt(fact, np.arange(10, dtype=np.uint32)),
               lambda: oracle.aggregate_count_sum_mt(fact, None, 10)):
        with pytest.raises(OracleError) as e:
            fn()
        assert (e.value.status, e.value.row, e.value.value) == (DOMAIN, 77777, 0)
    # value-column fixtures: kind 0 = the reference bench's dim column formula
    v = oracle.fill_column(0, np.uint64, 1000, 42)
    assert all(int(v[i]) == oracle.splitmix64(42 ^ (0xd1000000 + i)) for i in range(0, 1000, 97))
    q = oracle.fill_column(1, np.int64, 100000, 7, 1, 100)
    assert q.min() == 1 and q.max() == 100

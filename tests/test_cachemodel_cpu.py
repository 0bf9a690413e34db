"""Cache model (proj/src/cachemodel.cpp): the oracle's C
restatement pinned against the reference's own known answers
(proj/tests/test_cachemodel.cpp) and against the reference library's outputs
(tests/golden/ref_cachemodel.npz, live when oracle/_ref is present)."""
import json
import os

import numpy as np
import pytest

from oracle.oracle import OracleError

GOLDEN = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "ref_cachemodel.npz")


def test_kat_line_frequencies(oracle):
    # test_cachemodel.cpp:18-25: freq layout sums adjacent ranks
    f = oracle.line_frequencies([0.4, 0.3, 0.2, 0.1], "freq", 8, 4, 0)
    assert np.allclose(f, [0.7, 0.3], rtol=0, atol=1e-15)
    # :27-37: one element per line -> rand is a permutation of freq
    vf = np.random.default_rng(1).random(100)
    vf /= vf.sum()
    a = oracle.line_frequencies(vf, "freq", 4, 4, 7)
    b = oracle.line_frequencies(vf, "rand", 4, 4, 7)
    assert np.array_equal(np.sort(a), np.sort(b))
    # :39-47: uniform stays uniform
    for layout in ("freq", "rand"):
        f = oracle.line_frequencies(np.full(64, 1 / 64), layout, 64, 4, 3)
        assert np.allclose(f, 0.25, rtol=0, atol=1e-15)
    # :49-52: empty -> InvalidArgument
    with pytest.raises(OracleError):
        oracle.line_frequencies([], "freq", 64, 4, 0)


def test_kat_estimate_hit_rate(oracle):
    # test_cachemodel.cpp:55-66
    assert oracle.estimate_hit_rate([1.0], 1) == 1.0
    assert oracle.estimate_hit_rate([1.0], 64) == 1.0
    four = [0.25] * 4
    assert oracle.estimate_hit_rate(four, 4) == 1.0
    assert oracle.estimate_hit_rate(four, 3) < 1.0
    with pytest.raises(OracleError):
        oracle.estimate_hit_rate(four, 0)
    # :79-99: monotone in capacity, within [0, 1]
    rng = np.random.default_rng(42)
    for _ in range(10):
        lines = int(rng.integers(2, 400))
        f = rng.integers(1, 1001, size=lines).astype(np.float64)
        f /= f.sum()
        prev = 0.0
        s = 1
        while s <= lines + 4:
            est = oracle.estimate_hit_rate(f, s)
            assert prev - 1e-12 <= est <= 1.0
            prev = est
            s = 2 * s + 1
    # :101-110: skew toward the hot line never hurts
    prev = -1.0
    for d in np.arange(0.0, 0.5, 0.05):
        est = oracle.estimate_hit_rate([0.5 + d, 0.5 - d], 1)
        assert est >= prev - 1e-12
        prev = est


def test_kat_simulate_lru_and_trace(oracle):
    # test_cachemodel.cpp:112-131
    assert oracle.simulate_lru([1, 1, 1, 1], 1) == (4, 3, 1)
    assert oracle.simulate_lru([1, 2, 1, 2], 1)[1] == 0
    assert oracle.simulate_lru([1, 2, 1, 2], 2)[1] == 2
    assert oracle.simulate_lru([], 4) == (0, 0, 0)
    # :133-143: a cache larger than the footprint leaves only cold misses
    tr = np.random.default_rng(5).integers(0, 300, size=20000).astype(np.uint32)
    acc, hits, distinct = oracle.simulate_lru(tr, 512)
    assert hits == acc - distinct
    # :187-198: trace_from_column boundary arithmetic
    assert list(oracle.trace_from_column([1, 16, 17], 64, 4)) == [0, 0, 1]
    assert list(oracle.trace_from_column([33], 64, 4)) == [2]
    assert list(oracle.trace_from_column([1, 2, 9], 4, 4)) == [0, 1, 8]
    with pytest.raises(OracleError):
        oracle.trace_from_column([0], 64, 4)


def test_simulate_lru_matches_stack_distance(oracle):
    """test_cachemodel.cpp:145-185: an access hits iff fewer than S distinct
    lines were referenced since the previous access to the same line."""
    tr = np.random.default_rng(17).integers(0, 40, size=1500).astype(np.uint32)
    for s in (1, 3, 8, 21, 64):
        exp = 0
        last = {}
        for k, x in enumerate(tr):
            if x in last and len(set(tr[last[x] + 1:k].tolist())) < s:
                exp += 1
            last[x] = k
        assert oracle.simulate_lru(tr, s)[1] == exp


def _golden():
    z = np.load(GOLDEN)
    meta = json.loads(bytes(z["meta"]).decode())
    return z, meta


def test_cache_model_matches_reference_fixtures(oracle):
    z, meta = _golden()
    for i, m in enumerate(meta):
        lf = oracle.line_frequencies(z[f"c{i}_value_freqs"], m["layout"], m["line_bytes"],
                                     m["element_bytes"], m["seed"])
        assert np.array_equal(lf, z[f"c{i}_line_freqs"]), i  # bit-exact
        for s, exp in zip(m["caches"], m["estimate"]):
            assert oracle.estimate_hit_rate(lf, s) == exp, (i, s)  # bit-exact
        tr = oracle.trace_from_column(z[f"c{i}_fact"], m["line_bytes"], m["element_bytes"])
        assert np.array_equal(tr, z[f"c{i}_trace"]), i
        for s, exp in zip(m["caches"], m["lru"]):
            assert list(oracle.simulate_lru(tr, s)) == exp, (i, s)


def test_cache_model_matches_reference_live(oracle, reference):
    rng = np.random.default_rng(9)
    for _ in range(5):
        d = int(rng.integers(1, 3000))
        vf = rng.random(d)
        vf /= vf.sum()
        for layout in ("freq", "rand"):
            seed = int(rng.integers(0, 2**63))
            a = oracle.line_frequencies(vf, layout, 64, 4, seed)
            b = reference.line_frequencies(vf, layout, 64, 4, seed)
            assert np.array_equal(a, b)
            for s in (1, 7, 100):
                assert oracle.estimate_hit_rate(a, s) == reference.estimate_hit_rate(b, s)
        tr = rng.integers(0, 500, size=5000).astype(np.uint32)
        assert oracle.simulate_lru(tr, 37) == reference.simulate_lru(tr, 37)


def test_libskx_simulate_lru_host_matches_reference_fixtures():
    """The product library's host LRU simulator (no GPU needed) against the
    reference's outputs."""
    from paper_1910_10063_b200 import skewdx as sx
    z, meta = _golden()
    for i, m in enumerate(meta):
        for s, exp in zip(m["caches"], m["lru"]):
            st = sx.simulate_lru(z[f"c{i}_trace"], s)
            assert [st.accesses, st.hits, st.distinct_lines] == exp, (i, s)
    assert sx.simulate_lru([1, 1, 1, 1], 1).hit_rate() == 0.75
    assert sx.simulate_lru([], 4).hit_rate() == 0.0

"""Regenerate the golden fixtures in this directory from the REFERENCE itself.

Run in the build container (where /root/reference exists):

    make -C oracle ref && python tests/golden/make_golden.py

* kat.json      -- the reference's own hand-computed known-answer vectors,
                   transcribed from proj/tests/test_*.cpp (file:line in each
                   entry).  The Fig. 2 popularity fixture is stored as its
                   multiset (counts are order-insensitive; test_permindex.cpp:33).
* ref_cases.npz -- seeded workloads run through the unmodified reference
                   library (oracle/_ref/libskewdx_ref.so): generate_fact_column
                   (rand layout), count_frequencies, rebuild, recode_fact,
                   permute_dimension, materialize (both layouts), aggregate_count,
                   aggregate_sum, select (both layouts), permute_bitmap,
                   heavy_hitter_count.

The GPU box has no /root/reference, so these committed files are what the
tests compare against there.
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle.oracle import Oracle, Reference  # noqa: E402

# (D, N, z, seed): shapes used by the reference's own tests
# (test_operators.cpp:28-39 make_workload and the cases at :68-73, :144-153,
# :155-167, :176-191, :211-237) plus ragged / multi-tile / D=1 edges.
CASES = [
    (8, 64, 1.0, 3),
    (211, 5000, 0.0, 17),
    (211, 5000, 1.0, 17),
    (211, 5000, 2.0, 17),
    (300, 8000, 1.2, 5),
    (400, 9000, 1.5, 31),
    (123, 4567, 0.9, 41),
    (500, 20000, 1.5, 53),
    (97, 3000, 1.1, 67),
    (5000, 60000, 1.0, 71),
    (1, 10, 0.5, 1),
    (4096, 100003, 1.25, 42),
    (70001, 250001, 1.25, 9),
    (200, 5000, 0.7, 13),
    (2000, 7, 1.0, 5),
]


def splitmix_dim(o, d, seed):
    # bench dataset dim column: splitmix64(seed ^ (0xd1000000 + i)) (dataset.cpp:35-38)
    return np.array([o.splitmix64(seed ^ (0xD1000000 + i)) & 0xFFFFFFFF for i in range(d)],
                    dtype=np.uint32)


def main():
    o, r = Oracle(), Reference()
    arrays = {}
    meta = []
    for ci, (d, n, z, seed) in enumerate(CASES):
        fact = r.generate_fact_column(d, n, z, seed, "rand")
        counts = r.count_frequencies(fact, d)
        offsets, ranks = r.rebuild(fact, d)
        recoded = r.recode_fact(fact, offsets, ranks)
        dim = splitmix_dim(o, d, seed)
        dim_perm = r.permute_dimension(dim, offsets, ranks)
        mat_rand = r.materialize(fact, dim)
        mat_freq = r.materialize(recoded, dim_perm)
        measure = np.array([o.splitmix64(seed * 7 + k) % 100 + 1 for k in range(n)], np.uint32)
        sums = r.aggregate_sum(recoded, measure, d)
        counts_freq = r.aggregate_count(recoded, d)
        rng = np.random.default_rng(seed)
        bits = rng.integers(0, 2, size=d).astype(np.uint8)
        words = np.zeros((d + 63) // 64, np.uint64)
        for i in np.nonzero(bits)[0]:
            words[i >> 6] |= np.uint64(1) << np.uint64(i & 63)
        words_perm = r.permute_bitmap(words, d, offsets, ranks)
        sel_rand = r.select(fact, words, d)
        sel_freq = r.select(recoded, words_perm, d)
        hk = min(13, d)
        hh_ids, hh_counts, _ = r.heavy_hitter_count(recoded, d, 13)
        p = f"c{ci}_"
        arrays.update({
            p + "fact": fact, p + "counts": counts, p + "offsets": offsets, p + "ranks": ranks,
            p + "recoded": recoded, p + "dim": dim, p + "dim_perm": dim_perm,
            p + "mat_rand": mat_rand, p + "mat_freq": mat_freq, p + "measure": measure,
            p + "sums": sums, p + "counts_freq": counts_freq, p + "words": words,
            p + "words_perm": words_perm, p + "sel_rand": sel_rand, p + "sel_freq": sel_freq,
            p + "hh_ids": hh_ids, p + "hh_counts": hh_counts,
        })
        meta.append({"d": d, "n": n, "z": z, "seed": seed, "hh_k": hk})
    arrays["meta"] = np.frombuffer(json.dumps(meta).encode(), dtype=np.uint8)
    np.savez_compressed(os.path.join(HERE, "ref_cases.npz"), **arrays)
    print("wrote ref_cases.npz with", len(CASES), "cases")


if __name__ == "__main__":
    main()

"""Regenerate tests/golden/ref_cachemodel.npz from the REFERENCE itself.

    make -C oracle ref && python tests/golden/make_golden_cachemodel.py

Seeded cache-model workloads run through the unmodified reference library
(oracle/_ref/libskewdx_ref.so, proj/src/cachemodel.cpp): line_frequencies for
both layouts and several geometries, estimate_hit_rate over a sweep of cache
sizes, simulate_lru and trace_from_column on columns drawn by the reference's
generate_fact_column.  The GPU box has no /root/reference: the committed file
is what the tests compare against there.
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle.oracle import Reference  # noqa: E402

# (D, z, layout, line_bytes, element_bytes, seed, N for the LRU trace)
CASES = [
    (1, 1.0, "freq", 64, 4, 0, 100),
    (7, 0.0, "rand", 4, 4, 7, 500),
    (5000, 0.8, "freq", 64, 4, 3, 20000),
    (5000, 0.8, "rand", 64, 4, 3, 20000),
    (65536, 1.0, "freq", 64, 4, 31, 200000),
    (65536, 1.0, "rand", 64, 4, 31, 200000),
    (20000, 1.3, "freq", 128, 8, 11, 50000),
    (20000, 1.3, "rand", 128, 8, 11, 50000),
    (3001, 2.0, "rand", 32, 2, 5, 10000),
]
CACHES = [1, 3, 64, 512, 4096]


def main():
    ref = Reference()
    arrays, meta = {}, []
    for i, (d, z, layout, lb, eb, seed, n) in enumerate(CASES):
        vf = ref.zipf_frequencies(d, z)
        lf = ref.line_frequencies(vf, layout, lb, eb, seed)
        est = [ref.estimate_hit_rate(lf, s) for s in CACHES]
        fact = ref.generate_fact_column(d, n, z, seed, layout=layout)
        trace = ref.trace_from_column(fact, lb, eb)
        lru = [ref.simulate_lru(trace, s) for s in CACHES]
        arrays[f"c{i}_value_freqs"] = vf
        arrays[f"c{i}_line_freqs"] = lf
        arrays[f"c{i}_fact"] = fact
        arrays[f"c{i}_trace"] = trace
        meta.append({"d": d, "z": z, "layout": layout, "line_bytes": lb, "element_bytes": eb,
                     "seed": seed, "n": n, "caches": CACHES, "estimate": est,
                     "lru": [list(x) for x in lru]})
    arrays["meta"] = np.frombuffer(json.dumps(meta).encode(), np.uint8)
    np.savez_compressed(os.path.join(HERE, "ref_cachemodel.npz"), **arrays)
    print("wrote", len(CASES), "cases")


if __name__ == "__main__":
    main()

"""Host simulation of the histogram's shared-memory tables on the C4 stream
(D=2^26, Zipf 1.25, seed 51): the fraction of rows that miss the table and
become global reductions, for (a) the round-1 dynamic table (one CTA's
~2^30/444 rows, first keys claim slots) and (b) the sampled hot set (2^20
strided samples, keys hit >= 2 times by band, hottest first, greedy
two-choice fill).  Used in profiles/r2_experiments.md §4.

  python tools/hist_table_sim.py [cap]
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle.oracle import Oracle  # noqa: E402

cap = int(sys.argv[1]) if len(sys.argv) > 1 else 6144
o = Oracle()
d, z, seed, T = 1 << 26, 1.25, 51, 8192
cdf = o.zipf_cdf(d, z)
r2i = o.random_bijection(d, seed)


def h1(k):
    return ((k * 0x9E3779B1) & 0xFFFFFFFF) >> 19


def h2(k):
    return (((k * 0x85EBCA77) + 0x6A09E667) & 0xFFFFFFFF) >> 19


# (a) dynamic table over one CTA's rows
m = (1 << 30) // 444
rows = o.generate_zipf_counter_mt(cdf, r2i, seed, m, os.cpu_count() or 1).astype(np.uint64)
tab = np.zeros(T, np.int64)
cold = 0
for k, a, b in zip(rows.tolist(), h1(rows).tolist(), h2(rows).tolist()):
    if tab[a] == k or tab[b] == k:
        continue
    if tab[a] == 0:
        tab[a] = k
    elif tab[b] == 0:
        tab[b] = k
    else:
        cold += 1
print("dynamic table: cold fraction", cold / m)
# (b) sampled hot set (2^20 samples of a 2^24-row stream: the same sample size)
n = 1 << 24
fact = o.generate_zipf_counter_mt(cdf, r2i, seed, n, os.cpu_count() or 1)
cnt = np.bincount(fact, minlength=d + 1)
keys, hits = np.unique(fact[np.arange(1 << 20) * (n >> 20)], return_counts=True)
bands = [0, 4096, 512, 64, 16, 8, 4, 3, 2]
hot = []
for i in range(1, len(bands)):
    sel = (hits >= bands[i]) & ((hits < bands[i - 1]) if bands[i - 1] else True)
    hot += keys[sel].tolist()
hot = hot[:cap]
tab = np.zeros(T, np.int64)
for k in hot:
    a, b = h1(k), h2(k)
    if tab[a] == 0:
        tab[a] = k
    elif tab[b] == 0:
        tab[b] = k
covered = sum(cnt[k] for k in tab if k) / n
print("sampled hot set: keys", len(hot), "cold fraction", 1 - covered,
      "ideal (top cap keys)", 1 - np.sort(cnt)[::-1][:cap].sum() / n)

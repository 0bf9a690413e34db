"""Run each hot kernel once inside a cudaProfilerStart/Stop window so that
`ncu --profile-from-start off` captures exactly those launches.

  python tools/profile_kernels.py [--ops gather_freq,gather_rand,groupby,histogram,select]
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1910_10063_b200 import dataset as dsm  # noqa: E402
from paper_1910_10063_b200 import skewdx as sx  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--ops", default="gather_freq,gather_rand,groupby,histogram,select")
p.add_argument("--z", type=float, default=1.0)
p.add_argument("--rows", type=int, default=1 << 30)
p.add_argument("--domain", type=int, default=1 << 27)
p.add_argument("--policy", type=int, default=1)
a = p.parse_args()
ops = a.ops.split(",")
ctx = sx.context(0)
ctx.set_gather_policy(a.policy)
g = None
if any(o.startswith("gather") or o == "histogram" for o in ops):
    g = dsm.make_gather_dataset(a.domain, a.rows, a.z, 42, torch.int64)
    out = torch.empty(a.rows, dtype=torch.int64, device="cuda")
    for _ in range(2):
        sx.materialize(g.fact_freq, g.dim_freq, out=out)
        sx.materialize(g.fact_rand, g.dim_rand, out=out)
gb = None
if "groupby" in ops:
    gb = dsm.make_groupby_dataset(1 << 24, a.rows, 1.0, 43)
    for _ in range(2):
        sx.aggregate_count_sum(gb.fact_freq, gb.qty, 1 << 24)
if "histogram" in ops:
    sx.histogram_u32(g.fact_rand, a.domain)
sel = None
if "select" in ops:  # C5: 2^31 rows, D=2^25, reordered layout, category < 100
    d5, n5 = 1 << 25, 1 << 31
    f5 = dsm.make_rand_fact(d5, n5, 1.0, 42, dsm.shard_of(n5))
    idx5 = sx.build_index(sx.FrequencyProfile(sx.histogram_u32(f5, d5), n5))
    f5 = sx.recode_fact(f5, idx5)
    cat = sx.permute_dimension(dsm.fill_column(1, torch.int32, d5, 11, 0, 1000), idx5)
    price = sx.permute_dimension(dsm.fill_column(2, torch.float32, d5, 12, 3.0, 1.0), idx5)
    supp = sx.permute_dimension(dsm.fill_column(0, torch.int64, d5, 13), idx5)
    flag = sx.permute_dimension(dsm.fill_column(0, torch.int16, d5, 14), idx5)
    bm = sx.build_bitmap_lt(cat, 100)
    del idx5
    sel = (f5, bm, cat, price, supp, flag)
    sx.select_gather_sum(*sel, 1000)
torch.cuda.synchronize()
torch.cuda.profiler.start()
for o in ops:
    if o == "gather_freq":
        sx.materialize(g.fact_freq, g.dim_freq, out=out, sync=False)
    elif o == "gather_rand":
        sx.materialize(g.fact_rand, g.dim_rand, out=out, sync=False)
    elif o == "groupby":
        sx.aggregate_count_sum(gb.fact_freq, gb.qty, 1 << 24, sync=False)
    elif o == "histogram":
        sx.histogram_u32(g.fact_rand, a.domain, sync=False)
    elif o == "select":
        sx.select_gather_sum(*sel, 1000)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
ctx.sync()
print("profiled", ops)

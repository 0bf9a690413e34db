"""Build BASELINE workloads with the bench's own dataset functions and run the
chosen hot kernels once inside a cudaProfilerStart/Stop window, so that
`ncu --profile-from-start off` captures exactly those launches.

  python tools/profile_r2.py --ops gather_c2,groupby_c3,index_c4,select_c5,gather_c1
"""
import argparse
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1910_10063_b200 import dataset as ds  # noqa: E402
from paper_1910_10063_b200 import skewdx as sx  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--ops", default="gather_c2,groupby_c3,index_c4,select_c5")
p.add_argument("--z", type=float, default=1.0)
p.add_argument("--reps", type=int, default=1)
a = p.parse_args()
ops = a.ops.split(",")
ctx = sx.context(0)
work = {}
if "gather_c2" in ops or "gather_c2_rand" in ops:
    w2 = ds.C2
    g = ds.make_gather_dataset(w2.d, w2.n, a.z, w2.seed, torch.int64)
    out = torch.empty(w2.n, dtype=torch.int64, device="cuda")
    work["gather_c2"] = lambda: sx.materialize(g.fact_freq, g.dim_freq, out=out, sync=False)
    work["gather_c2_rand"] = lambda: sx.materialize(g.fact_rand, g.dim_rand, out=out, sync=False)
if "gather_c1" in ops:
    c1 = ds.make_c1_dataset()
    o1 = torch.empty(ds.C1.n, dtype=torch.int32, device="cuda")
    work["gather_c1"] = lambda: sx.materialize(c1.g.fact_freq, c1.price_freq, out=o1, sync=False)
if "groupby_c3" in ops:
    w3 = ds.C3  # (each op binds its own workload: the closures run after all are built)
    gd = ds.make_groupby_dataset(w3.d, w3.n, w3.z, w3.seed)
    c3 = torch.empty(w3.d, dtype=torch.uint64, device="cuda")
    s3 = torch.empty(w3.d, dtype=torch.uint64, device="cuda")
    work["groupby_c3"] = lambda: sx.aggregate_count_sum(gd.fact_freq, gd.qty, w3.d, counts=c3,
                                                        sums=s3, sync=False)
if "index_c4" in ops:
    w4 = ds.C4
    ib = ds.make_index_build_dataset()
    h4 = torch.empty(w4.d, dtype=torch.uint32, device="cuda")
    f4 = torch.empty_like(ib.fact)

    def c4():
        sx.histogram_u32(ib.fact, w4.d, h4, sync=False)
        idx = sx.build_index(sx.FrequencyProfile(h4, w4.n), sync=False)
        sx.recode_fact(ib.fact, idx, out=f4, sync=False)
        sx.permute_dimension(ib.dim_i, idx, sync=False)
        sx.permute_dimension(ib.dim_f, idx, sync=False)
    work["index_c4"] = c4
if "select_c5" in ops:
    sd = ds.make_select_dataset()
    cap = ds.C5.n // 5
    o5 = tuple(torch.empty(cap, dtype=t, device="cuda") for t in
               (torch.uint32, torch.int32, torch.float32, torch.uint64, torch.uint16)) + (
        torch.empty(1000, dtype=torch.float64, device="cuda"),
        torch.zeros(1, dtype=torch.uint64, device="cuda"))
    work["select_c5"] = lambda: sx.select_gather_sum(sd.fact, sd.bitmap, sd.cat, sd.price, sd.supp,
                                                     sd.flag, 1000, out=o5, sync=False)
for o in ops:  # warm: scratch arenas grown, attributes set
    work[o]()
torch.cuda.synchronize()
ctx.sync()
torch.cuda.profiler.start()
for _ in range(a.reps):
    for o in ops:
        work[o]()
torch.cuda.synchronize()
torch.cuda.profiler.stop()
ctx.sync()
print("profiled", ops)

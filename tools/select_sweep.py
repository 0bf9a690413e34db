"""C5: select rows whose category < 100 (bitmap over the dimension), gather the
four dimension columns (int32 category, float32 lognormal price, int64
supplier, int16 flag) for the selected rows and SUM(price) per category in
fp64.  2^31 FK rows Zipf(1.0) over 2^25 keys by default; both layouts."""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1910_10063_b200 import dataset as dsm  # noqa: E402
from paper_1910_10063_b200 import skewdx as sx  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--rows", type=int, default=1 << 31)
p.add_argument("--domain", type=int, default=1 << 25)
p.add_argument("--z", type=float, default=1.0)
p.add_argument("--steps", type=int, default=5)
a = p.parse_args()
ctx = sx.context(0)
d, n = a.domain, a.rows
C = __import__("ctypes")
fact = dsm.make_rand_fact(d, n, a.z, 42, dsm.shard_of(n))
counts = sx.histogram_u32(fact, d, sync=False)
idx = sx.build_index(sx.FrequencyProfile(counts, n), sync=False)
fact_freq = sx.recode_fact(fact, idx, sync=False)
cat = dsm.fill_column(1, torch.int32, d, 11, 0, 1000)
price = dsm.fill_column(2, torch.float32, d, 12, 3.0, 1.0)
supp = dsm.fill_column(0, torch.int64, d, 13)
flag = dsm.fill_column(0, torch.int16, d, 14)
ctx.sync()
bm = sx.build_bitmap_lt(cat, 100)
layouts = {"rand": (fact, cat, price, supp, flag, bm),
           "freq": (fact_freq, sx.permute_dimension(cat, idx), sx.permute_dimension(price, idx),
                    sx.permute_dimension(supp, idx), sx.permute_dimension(flag, idx),
                    sx.permute_bitmap(bm, idx))}
cap = n // 5
dev = "cuda"
o_off = torch.empty(cap, dtype=torch.uint32, device=dev)
o_cat = torch.empty(cap, dtype=torch.int32, device=dev)
o_pr = torch.empty(cap, dtype=torch.float32, device=dev)
o_su = torch.empty(cap, dtype=torch.int64, device=dev)
o_fl = torch.empty(cap, dtype=torch.int16, device=dev)
sums = torch.empty(1000, dtype=torch.float64, device=dev)
cnt = torch.zeros(1, dtype=torch.uint64, device=dev)
P = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
res = {}
for name, (f, c_, p_, s_, fl_, b_) in layouts.items():
    def step():
        ctx.call("skx_select_gather_sum", P(f), n, P(b_.words), d, P(c_), P(p_), P(s_), P(fl_), 0,
                 1000, cap, P(o_off), P(o_cat), P(o_pr), P(o_su), P(o_fl), P(sums), P(cnt), ctx.stream(),
                 sync=False)
    for _ in range(3):
        step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(a.steps):
        step()
    e1.record()
    torch.cuda.synchronize()
    ctx.sync()
    ms = e0.elapsed_time(e1) / a.steps
    k = int(cnt.item())
    assert k <= cap, "output capacity exceeded"
    alg = n * 4 + k * (4 + 4 + 4 + 8 + 2) + 1000 * 8
    res[name] = {"ms": round(ms, 3), "selected": k, "selectivity": round(k / n, 4),
                 "rows_per_s": n / (ms * 1e-3), "alg_bytes": alg,
                 "frac": round(alg / (ms * 1e-3) / 6545.3e9, 4),
                 "sum_total": float(sums.sum().item())}
print(json.dumps({"workload": "C5", "rows": n, "domain": d, "z": a.z, **res}))

"""C4 index build timing: histogram (u32) -> sort-by-count -> recode -> permute
two dims (int32, float32), D=2^26, 2^30 rows, Zipf s=1.25 (configurable)."""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1910_10063_b200 import dataset as dsm  # noqa: E402
from paper_1910_10063_b200 import skewdx as sx  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--z", type=float, default=1.25)
p.add_argument("--rows", type=int, default=1 << 30)
p.add_argument("--domain", type=int, default=1 << 26)
p.add_argument("--reps", type=int, default=3)
p.add_argument("--hist-mode", type=int, default=-1, help="skx_set_histogram_mode (-1: default)")
a = p.parse_args()
ctx = sx.context(0)
if a.hist_mode >= 0:
    ctx.check(ctx.lib.skx_set_histogram_mode(ctx.handle, a.hist_mode))
d, n = a.domain, a.rows
fact = dsm.make_rand_fact(d, n, a.z, 42, dsm.shard_of(n))
dim_i = dsm.fill_column(0, torch.int32, d, 1)
dim_f = torch.randn(d, device="cuda")
counts = torch.empty(d, dtype=torch.uint32, device="cuda")
fact_freq = torch.empty_like(fact)
torch.cuda.synchronize()
res = {}
for rep in range(a.reps + 1):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
    ev[0].record()
    sx.histogram_u32(fact, d, counts, sync=False)
    ev[1].record()
    idx = sx.build_index(sx.FrequencyProfile(counts, n), sync=False)
    ev[2].record()
    sx.recode_fact(fact, idx, out=fact_freq, sync=False)
    ev[3].record()
    pi = sx.permute_dimension(dim_i, idx, sync=False)
    pf = sx.permute_dimension(dim_f, idx, sync=False)
    ev[4].record()
    torch.cuda.synchronize()
    ctx.sync()
    if rep == 0:
        continue  # warm-up (scratch allocation)
    for k, (i, j) in {"histogram": (0, 1), "sort": (1, 2), "recode": (2, 3), "permute2": (3, 4),
                      "total": (0, 4)}.items():
        res.setdefault(k, []).append(ev[i].elapsed_time(ev[j]))
out = {k: round(min(v), 3) for k, v in res.items()}
alg = n * 12 + d * 28
out["alg_bytes"] = alg
out["frac_total"] = round(alg / (out["total"] * 1e-3) / 6545.3e9, 4)
out["rows_per_s"] = n / (out["total"] * 1e-3)
print(json.dumps({"z": a.z, "domain": d, "rows": n, "hist_mode": a.hist_mode, **out}))

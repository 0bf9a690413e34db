"""C3 group-by timing sweep: COUNT+SUM(int64 qty) over 2^30 recoded rows, D=2^24."""
import argparse
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1910_10063_b200 import dataset as dsm  # noqa: E402
from paper_1910_10063_b200 import skewdx as sx  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--z", default="1.0")
p.add_argument("--hot", default="0")
p.add_argument("--rows", type=int, default=1 << 30)
p.add_argument("--domain", type=int, default=1 << 24)
p.add_argument("--modes", default="0,2", help="skx_set_aggregate_mode values")
a = p.parse_args()
ctx = sx.context(0)
for z in [float(x) for x in a.z.split(",")]:
    g = dsm.make_groupby_dataset(a.domain, a.rows, z, 43)
    ref = None
    for hot, amode in [(int(h), int(am)) for h in a.hot.split(",") for am in a.modes.split(",")]:
        ctx.check(ctx.lib.skx_set_aggregate_mode(ctx.handle, amode))
        for mode in ("count_sum", "count"):
            def step():
                if mode == "count_sum":
                    return sx.aggregate_count_sum(g.fact_freq, g.qty, a.domain, hot_threshold=hot, sync=False)
                return sx.aggregate_count(g.fact_freq, a.domain, hot_threshold=hot, sync=False)
            for _ in range(3):
                r = step()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for _ in range(5):
                r = step()
            e1.record()
            torch.cuda.synchronize()
            ctx.sync()
            ms = e0.elapsed_time(e1) / 5
            c = r[0] if mode == "count_sum" else r
            if ref is None:
                ref = c.clone()
            bytes_ = a.rows * (12 if mode == "count_sum" else 4) + a.domain * (16 if mode == "count_sum" else 8)
            print(json.dumps({"z": z, "hot": hot, "agg_mode": amode, "mode": mode, "ms": round(ms, 3),
                              "rows_per_s": a.rows / (ms * 1e-3),
                              "frac": round(bytes_ / (ms * 1e-3) / 6545.3e9, 4),
                              "counts_equal": bool(torch.equal(c, ref))}), flush=True)
    del g
    torch.cuda.empty_cache()

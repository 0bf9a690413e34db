"""C4 recode / histogram / permute times under each cudaLimitMaxL2FetchGranularity (skx_set_l2_fetch_granularity)."""
import sys, os, json, subprocess
sys.path.insert(0, os.getcwd())
import torch
from paper_1910_10063_b200 import dataset as ds, skewdx as sx
ctx = sx.context(0)
ib = ds.make_index_build_dataset()
w = ds.C4
h = torch.empty(w.d, dtype=torch.uint32, device="cuda")
out = torch.empty_like(ib.fact)
sx.histogram_u32(ib.fact, w.d, h)
idx = sx.build_index(sx.FrequencyProfile(h, w.n))
res = {}
for g in (64, 32, 128, 64):
    ctx.check(ctx.lib.skx_set_l2_fetch_granularity(ctx.handle, g))
    for name, fn in (("recode", lambda: sx.recode_fact(ib.fact, idx, out=out, sync=False)),
                     ("hist", lambda: sx.histogram_u32(ib.fact, w.d, h, sync=False)),
                     ("permute", lambda: sx.permute_dimension(ib.dim_i, idx, sync=False))):
        for _ in range(3): fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10): fn()
        e1.record(); torch.cuda.synchronize()
        res.setdefault(name, []).append((g, round(e0.elapsed_time(e1) / 10, 3)))
print(json.dumps(res))

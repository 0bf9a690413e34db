"""Sweep gather variants on the C2 workload: layout x policy x L2 fetch
granularity x Zipf s.  Prints one JSON object per cell (CUDA-event timing,
10 launches after 3 warm-ups).

  python tools/gather_sweep.py [--z 0.5,1.0,1.5] [--policies 1,2] [--gran 0,32]
"""
import argparse
import ctypes as C
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1910_10063_b200 import dataset as dsm  # noqa: E402
from paper_1910_10063_b200 import skewdx as sx  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--z", default="1.0")
p.add_argument("--policies", default="1,3,7,9,11,15,0")
p.add_argument("--gran", default="0,32")
p.add_argument("--rows", type=int, default=1 << 30)
p.add_argument("--domain", type=int, default=1 << 27)
p.add_argument("--width", type=int, default=8)
p.add_argument("--steps", type=int, default=10)
p.add_argument("--tiers", default="0:160:0.6", help="comma list of smemKB:l1KB:l2frac")
a = p.parse_args()
ctx = sx.context(0)
info = (C.c_uint64 * 6)()
ctx.lib.skx_device_info(ctx.handle, info, 6)
print(json.dumps({"device_info": dict(zip(["num_sms", "smem_optin", "l2_bytes", "persist_max",
                                           "window_max", "l2_fetch_gran"], list(info)))}))
peak = 6545.3
dt = {2: torch.int16, 4: torch.int32, 8: torch.int64}[a.width]
for z in [float(x) for x in a.z.split(",")]:
    ctx.set_gather_policy(1)
    g = dsm.make_gather_dataset(a.domain, a.rows, z, 42, dt)
    out = torch.empty(a.rows, dtype=dt, device="cuda")
    ref = None
    for gran in [int(x) for x in a.gran.split(",")]:
        if gran:
            ctx.check(ctx.lib.skx_set_l2_fetch_granularity(ctx.handle, gran))
        cells = []
        for pol in [int(x) for x in a.policies.split(",")]:
            if pol & 38:
                for t in a.tiers.split(","):
                    cells.append((pol, t))
            else:
                cells.append((pol, None))
        for pol, tier in cells:
            if tier:
                sk, kb, fr = tier.split(":")
                ctx.check(ctx.lib.skx_set_gather_tiers(ctx.handle, int(sk) * 1024, int(kb) * 1024,
                                                       float(fr)))
            ctx.set_gather_policy(pol)
            ctx.check(ctx.lib.skx_reset_persisting_l2(ctx.handle))
            for layout in ("freq", "rand"):
                f, d = g.fact(layout), g.dim(layout)
                for _ in range(3):
                    sx.materialize(f, d, out=out, sync=False)
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(a.steps):
                    sx.materialize(f, d, out=out, sync=False)
                e1.record()
                torch.cuda.synchronize()
                ctx.sync()
                ms = e0.elapsed_time(e1) / a.steps
                if ref is None:
                    ref = out.clone()
                ok = bool(torch.equal(out, ref))
                gbs = a.rows * (4 + a.width) / (ms * 1e-3) / 1e9
                print(json.dumps({"z": z, "policy": pol, "tier": tier, "layout": layout,
                                  "ms": round(ms, 4), "rows_per_s": a.rows / (ms * 1e-3),
                                  "alg_GBps": round(gbs, 1), "frac": round(gbs / peak, 4),
                                  "equal": ok}), flush=True)
    del g, out, ref
    torch.cuda.empty_cache()

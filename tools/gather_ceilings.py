"""Ceilings of the gather kernel on B200: streams only, L1-resident random,
L2-resident random and DRAM-resident random dimension reads (2^30 rows, int64)."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1910_10063_b200 import dataset as dsm  # noqa: E402
from paper_1910_10063_b200 import skewdx as sx  # noqa: E402

ctx = sx.context(0)
n = 1 << 30
out = torch.empty(n, dtype=torch.int64, device="cuda")
pols = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "1,3").split(",")]
for name, d, z in [("stream_only(z=4)", 1 << 20, 4.0), ("L1_random(D=2^13,z=0)", 1 << 13, 0.0),
                   ("smem_fit(D=2^14,z=0)", 1 << 14, 0.0), ("L2_random(D=2^20,z=0)", 1 << 20, 0.0),
                   ("L2_random(D=2^23,z=0)", 1 << 23, 0.0), ("DRAM_random(D=2^27,z=0)", 1 << 27, 0.0)]:
    cdf = torch.from_numpy(sx.zipf_cdf(d, z)).cuda()
    fact = sx.generate_zipf(cdf, n, 7)
    dim = dsm.fill_column(0, torch.int64, d, 3)
    for pol in pols:
        ctx.set_gather_policy(pol)
        for _ in range(3):
            sx.materialize(fact, dim, out=out, sync=False)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            sx.materialize(fact, dim, out=out, sync=False)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 10
        print(json.dumps({"case": name, "policy": pol, "ms": round(ms, 3),
                          "alg_frac": round(n * 12 / (ms * 1e-3) / 6545.3e9, 3)}), flush=True)
    del fact, dim, cdf

"""Cache model (csrc/cachemodel.cu) applied to the C2
gather on B200 geometry: predicted LRU hit rates of the dimension reads for
both layouts and s in {0.5, 1.0, 1.5}, for an L1-sized cache (one SM, 228 KB)
and for L2 (126 MB).  128-byte lines of int64 values (16 per line).  Prints
JSON lines; compared with ncu in DESIGN.md / profiles/r1_experiments.md."""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1910_10063_b200 import skewdx as sx  # noqa: E402

d = int(sys.argv[1]) if len(sys.argv) > 1 else 1 << 27
geom = sx.CacheGeometry(1, 128, 8)
caches = {"L1_228KB": 228 * 1024 // 128, "L2_126MB": 126 * (1 << 20) // 128,
          "L2_half_63MB": 63 * (1 << 20) // 128}
for z in (0.5, 1.0, 1.5):
    cdf = sx.zipf_cdf(d, z)
    vf = torch.from_numpy(cdf).cuda()
    vf[1:] -= vf[:-1].clone()  # per-rank frequencies from the CDF
    for layout in (sx.Layout.freq, sx.Layout.rand):
        t0 = time.perf_counter()
        lf = sx.line_frequencies(vf, layout, geom, 42)
        res = {name: round(sx.estimate_hit_rate(lf, s), 4) for name, s in caches.items()}
        print(json.dumps({"z": z, "layout": layout.name, "domain": d, "lines": lf.numel(), **res,
                          "model_s": round(time.perf_counter() - t0, 3)}), flush=True)

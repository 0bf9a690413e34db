import sys, json, torch
sys.path.insert(0, '/root/repo')
from paper_1910_10063_b200 import skewdx as sx
d = 1 << 27
cdf = torch.from_numpy(sx.zipf_cdf(d, 1.0)).cuda()
vf = cdf.clone(); vf[1:] -= cdf[:-1]
vf[:8192] = 0  # hot keys caught by the per-CTA tables
tot = float(vf.sum())
vf /= tot
for name, eb in (("u32", 4), ("u16", 2), ("u8", 1)):
    geom = sx.CacheGeometry(1, 128, eb)
    lf = sx.line_frequencies(vf, sx.Layout.rand, geom, 42)
    for cap_mb in (64, 126):
        h = sx.estimate_hit_rate(lf, (cap_mb << 20) // 128)
        print(json.dumps({"counter": name, "L2_MB": cap_mb, "cold_fraction": tot, "pred_hit": round(h, 4)}))

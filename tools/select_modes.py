"""C5 (BASELINE configs[4], dataset.make_select_dataset): the selection fused
(offsets + 4 gathered columns + category sums) and offsets only, timed with
CUDA events after warm-up.  With SKX_LIBSKX pointing at library variants
(tools/ab.sh) this is the A/B harness for the selection kernels; --modes
selects skx_set_select_mode values when the library has that entry."""
import argparse
import ctypes as C
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1910_10063_b200 import dataset as ds  # noqa: E402
from paper_1910_10063_b200 import skewdx as sx  # noqa: E402

p = argparse.ArgumentParser()
p.add_argument("--steps", type=int, default=10)
p.add_argument("--modes", default="")
p.add_argument("--once", action="store_true", help="one launch per mode (for ncu)")
a = p.parse_args()
ctx = sx.context(0)
sd = ds.make_select_dataset()
n, d = sd.n, sd.d
cap = n // 5
dev = "cuda"
P = lambda t: C.c_void_p(t.data_ptr())  # noqa: E731
res = {}
outs = {}
for mode in [int(m) for m in a.modes.split(",")] if a.modes else [0]:
    if a.modes:
        ctx.check(ctx.lib.skx_set_select_mode(ctx.handle, mode))
    out = (torch.empty(cap, dtype=torch.uint32, device=dev), torch.empty(cap, dtype=torch.int32, device=dev),
           torch.empty(cap, dtype=torch.float32, device=dev), torch.empty(cap, dtype=torch.int64, device=dev),
           torch.empty(cap, dtype=torch.int16, device=dev), torch.empty(1000, dtype=torch.float64, device=dev),
           torch.zeros(1, dtype=torch.uint64, device=dev))
    o_off = torch.empty(n, dtype=torch.uint32, device=dev)
    cnt2 = torch.zeros(1, dtype=torch.uint64, device=dev)

    def fused():
        ctx.call("skx_select_gather_sum", P(sd.fact), n, P(sd.bitmap.words), d, P(sd.cat), P(sd.price),
                 P(sd.supp), P(sd.flag), 0, 1000, cap, *[P(t) for t in out], ctx.stream(), sync=False)

    def offsets():
        ctx.call("skx_select_offsets", P(sd.fact), n, P(sd.bitmap.words), d, 0, P(o_off), P(cnt2),
                 ctx.stream(), sync=False)
    for name, fn in (("fused", fused), ("offsets", offsets)):
        if a.once:
            fn()
            ctx.sync()
            continue
        for _ in range(3):
            fn()
        ctx.sync()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(a.steps):
            fn()
        e1.record()
        ctx.sync()
        res[f"mode{mode}_{name}_ms"] = round(e0.elapsed_time(e1) / a.steps, 3)
    k = int(out[6].item())
    outs[mode] = [t[:k].clone() for t in out[:5]] + [out[5].clone(), o_off[:int(cnt2.item())].clone()]
    res[f"mode{mode}_selected"] = k
if a.modes:
    ctx.check(ctx.lib.skx_set_select_mode(ctx.handle, 0))
if len(outs) == 2:
    o0, o1 = outs.values()
    res["modes_equal"] = all(torch.equal(x, y) for x, y in zip(o0[:5] + o0[6:], o1[:5] + o1[6:]))
    res["sums_equal"] = bool(torch.equal(o0[5], o1[5]))
print(json.dumps(res))

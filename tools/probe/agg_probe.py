"""Drive agg_probe.cu at C3 (2^30 rows, D=2^24, int64 qty 1..100, reordered Zipf)."""
import ctypes as C
import json
import os
import subprocess
import sys

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from paper_1910_10063_b200 import dataset as dsm  # noqa: E402
from paper_1910_10063_b200 import skewdx as sx  # noqa: E402

so = os.path.join(HERE, "agg_probe.so")
if not os.path.exists(so):
    subprocess.check_call(["nvcc", "-O3", "-shared", "-Xcompiler", "-fPIC", "-std=c++17",
                           "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
                           os.path.join(HERE, "agg_probe.cu"), "-o", so])
lib = C.CDLL(so)
lib.probe_agg.argtypes = [C.c_int, C.c_int, C.c_uint32, C.c_void_p, C.c_void_p, C.c_uint64,
                          C.c_void_p, C.c_uint32, C.c_void_p]
n, d = 1 << 30, 1 << 24
zs = [float(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "1.0").split(",")]
what = sys.argv[2] if len(sys.argv) > 2 else "time"
ctx = sx.context(0)
pairs = torch.zeros(2 * d, dtype=torch.int64, device="cuda")
stream = torch.cuda.current_stream().cuda_stream
cfgs = [(t, h, 148) for t in (0, 1, 2, 3, 4, 5) for h in (16384,)]
cfgs += [(0, h, 148) for h in (4096, 8192, 12288)]
for z in zs:
    g = dsm.make_groupby_dataset(d, n, z, 43)
    fk, qty = g.fact_freq, g.qty
    lib_ms = None
    if what == "time":
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for _ in range(3):
            sx.aggregate_count_sum(fk, qty, d, sync=False)
        e0.record()
        for _ in range(5):
            sx.aggregate_count_sum(fk, qty, d, sync=False)
        e1.record()
        torch.cuda.synchronize()
        print(json.dumps({"z": z, "case": "library aggregate_sum", "ms": e0.elapsed_time(e1) / 5}),
              flush=True)
    for tail, hot, grid in cfgs:
        def run():
            rc = lib.probe_agg(tail, grid, hot, fk.data_ptr(), qty.data_ptr(), n, pairs.data_ptr(),
                               (1 << 21) - 1, stream)
            assert rc == 0, rc
        if what != "time":
            run()
            continue
        for _ in range(3):
            run()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            run()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        print(json.dumps({"z": z, "tail": tail, "hot": hot, "grid": grid, "ms": round(ms, 3),
                          "frac": round(n * 12 / (ms * 1e-3) / 6545.3e9, 3)}), flush=True)
    torch.cuda.synchronize()

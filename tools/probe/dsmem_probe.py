"""Drive tools/probe/dsmem_probe.cu: DSMEM / smem-replica / global gathers of a
frequency-sorted int64 dimension (D=2^27) under Zipf FKs.  Prints JSON lines."""
import ctypes as C
import json
import os
import subprocess
import sys

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
from paper_1910_10063_b200 import dataset as dsm  # noqa: E402
from paper_1910_10063_b200 import skewdx as sx  # noqa: E402

so = os.path.join(HERE, "dsmem_probe.so")
if not os.path.exists(so):
    subprocess.check_call(["nvcc", "-O3", "-shared", "-Xcompiler", "-fPIC", "-std=c++17",
                           "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
                           os.path.join(HERE, "dsmem_probe.cu"), "-o", so])
lib = C.CDLL(so)
lib.probe_gather.argtypes = [C.c_int, C.c_int, C.c_int, C.c_uint32, C.c_uint32, C.c_void_p,
                             C.c_uint64, C.c_void_p, C.c_void_p, C.c_void_p]

ctx = sx.context(0)
n = int(os.environ.get("PROBE_ROWS", 1 << 30))
d = 1 << 27
dim = dsm.fill_column(0, torch.int64, d, 3)
out = torch.empty(n, dtype=torch.int64, device="cuda")
ref = torch.empty(n, dtype=torch.int64, device="cuda")
stream = torch.cuda.current_stream().cuda_stream
zs = [float(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "1.0,1.5,0.5").split(",")]


def timeit(fn, reps=5):
    for _ in range(3):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


configs = [(0, 1, 0, 0)]
configs += [(2, 1, 0, loc) for loc in (4096, 16384, 24576)]
configs += [(1, c, sl, 0) for c in (2, 4, 8, 16) for sl in (8192, 16384, 24576)]
configs += [(3, c, sl, loc) for c in (8, 16) for (sl, loc) in ((16384, 4096), (20480, 4096),
                                                                 (12288, 8192))]
for z in zs:
    cdf = torch.from_numpy(sx.zipf_cdf(d, z)).cuda()
    fact = sx.generate_zipf(cdf, n, 7)
    del cdf
    ctx.set_gather_policy(129)
    lib_ms = timeit(lambda: sx.materialize(fact, dim, out=ref, sync=False))
    print(json.dumps({"z": z, "case": "library", "ms": round(lib_ms, 3)}), flush=True)
    for mode, cl, sl, loc in configs:
        grid = (148 // cl) * cl

        def run():
            rc = lib.probe_gather(mode, cl, grid, sl, loc, fact.data_ptr(), n, dim.data_ptr(),
                                  out.data_ptr(), stream)
            if rc:
                raise RuntimeError(f"launch rc {rc}")
        try:
            ms = timeit(run)
            ok = bool(torch.equal(out, ref))
        except RuntimeError as e:
            print(json.dumps({"z": z, "mode": mode, "cluster": cl, "err": str(e)}), flush=True)
            continue
        print(json.dumps({"z": z, "mode": mode, "cluster": cl, "slice": sl, "local": loc,
                          "grid": grid, "ms": round(ms, 3), "ok": ok,
                          "frac": round(n * 12 / (ms * 1e-3) / 6545.3e9, 3)}), flush=True)
    del fact

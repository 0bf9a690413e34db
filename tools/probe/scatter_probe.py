"""Drive scatter_probe.cu: 2^27 random 8-byte writes / reads / REDs into a 2^30-entry
(8 GiB) array.  argv[1] = 'time' (CUDA events) or 'ncu' (one launch per mode)."""
import ctypes as C
import json
import os
import subprocess
import sys

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
so = os.path.join(HERE, "scatter_probe.so")
if not os.path.exists(so):
    subprocess.check_call(["nvcc", "-O3", "-shared", "-Xcompiler", "-fPIC", "-std=c++17",
                           "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
                           os.path.join(HERE, "scatter_probe.cu"), "-o", so])
lib = C.CDLL(so)
lib.probe_scatter.argtypes = [C.c_int, C.c_void_p, C.c_uint64, C.c_uint64, C.c_void_p, C.c_int,
                              C.c_void_p]
n = 1 << 30
count = 1 << 27
dst = torch.zeros(n, dtype=torch.int64, device="cuda")
sink = torch.zeros(1, dtype=torch.int64, device="cuda")
s = torch.cuda.current_stream().cuda_stream
what = sys.argv[1] if len(sys.argv) > 1 else "time"
for mode in (0, 1, 2, 3):
    def run():
        assert lib.probe_scatter(mode, dst.data_ptr(), n - 1, count, sink.data_ptr(), 148 * 8,
                                 s) == 0
    if what == "ncu":
        run()
        torch.cuda.synchronize()
        continue
    for _ in range(2):
        run()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        run()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(json.dumps({"mode": mode, "ms": round(ms, 3), "Mops_per_ms": round(count / ms / 1e6, 1)}),
          flush=True)

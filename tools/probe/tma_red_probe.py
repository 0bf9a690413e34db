"""Stream + random L2 reductions: per-lane loads vs TMA bulk copies
(tools/probe/tma_red_probe.cu).  4 GiB of u32, ~37% of values add 1 to a
random word of a 32 MB table.  Prints ms per mode and grid."""
import ctypes as C
import json
import os
import subprocess

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
so = os.path.join(HERE, "tma_red_probe.so")
if not os.path.exists(so):
    subprocess.check_call(["nvcc", "-O3", "-shared", "-Xcompiler", "-fPIC", "-std=c++17",
                           "-gencode", "arch=compute_100a,code=sm_100a",
                           os.path.join(HERE, "tma_red_probe.cu"), "-o", so])
lib = C.CDLL(so)
lib.probe_tma_red.argtypes = [C.c_int, C.c_void_p, C.c_uint64, C.c_void_p, C.c_uint32, C.c_void_p,
                              C.c_int, C.c_void_p]
nsm = torch.cuda.get_device_properties(0).multi_processor_count
n = 1 << 30
a = torch.randint(0, 2**31, (n,), dtype=torch.int32, device="cuda")
tab = torch.zeros(8 << 20, dtype=torch.int32, device="cuda")
out = torch.zeros(4, dtype=torch.int32, device="cuda")
s = torch.cuda.current_stream().cuda_stream
for mode in (2, 3, 0, 1):
    for per in (2, 4):
        grid = nsm * per
        f = lambda: lib.probe_tma_red(mode, a.data_ptr(), n, tab.data_ptr(), (8 << 20) - 1,
                                      out.data_ptr(), grid, s)
        for _ in range(3):
            assert f() == 0
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5):
            f()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        print(json.dumps({"mode": ["ld+red", "tma+red", "ld", "tma"][mode], "ctas_per_sm": per,
                          "ms": round(ms, 3), "stream_GBps": round(4 * n / ms / 1e6, 1)}), flush=True)

"""Fire-and-forget reductions: local smem vs distributed smem (cluster 2..16)
vs global REDs into an L2-resident 32 MB table.  Prints G reds/s chip-wide."""
import ctypes as C
import json
import os
import subprocess

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
so = os.path.join(HERE, "dsmem_red_probe.so")
if not os.path.exists(so):
    subprocess.check_call(["nvcc", "-O3", "-shared", "-Xcompiler", "-fPIC", "-std=c++17",
                           "-gencode", "arch=compute_100a,code=sm_100a",
                           os.path.join(HERE, "dsmem_red_probe.cu"), "-o", so])
lib = C.CDLL(so)
lib.probe_red.argtypes = [C.c_int, C.c_int, C.c_int, C.c_uint32, C.c_void_p, C.c_uint32,
                          C.c_void_p, C.c_int, C.c_void_p]
nsm = torch.cuda.get_device_properties(0).multi_processor_count
s = torch.cuda.current_stream().cuda_stream
gw = 8 << 20
gtab = torch.zeros(gw, dtype=torch.int32, device="cuda")
out = torch.zeros(4096, dtype=torch.int32, device="cuda")
iters = 2048
for mode, cl in [(0, 1), (2, 1), (1, 2), (1, 4), (1, 8), (1, 16)]:
    mc = lib.probe_max_clusters(cl)
    grid = (mc * cl) if mode == 1 and mc > 0 else nsm
    grid = grid // cl * cl
    rc = 0
    for r in range(2):
        rc |= lib.probe_red(mode, cl, iters, 1 + r, gtab.data_ptr(), gw, out.data_ptr(), grid, s)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for r in range(5):
        rc |= lib.probe_red(mode, cl, iters, 9 + r, gtab.data_ptr(), gw, out.data_ptr(), grid, s)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(json.dumps({"mode": ["local", "dsmem", "global"][mode], "cluster": cl, "grid": grid,
                      "max_clusters": mc, "rc": rc, "ms": round(ms, 4),
                      "Greds_per_s": round(grid * 1024 * iters / ms / 1e6, 1),
                      "per_SM_per_clk": round(grid * 1024 * iters / ms / 1e6 / grid / 1.9, 2)}),
          flush=True)

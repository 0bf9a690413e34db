"""Effective L2 capacity for random reads: dimension of M MB read uniformly at
random (no other traffic); prints time per read; run under ncu for DRAM bytes."""
import ctypes as C
import json
import os
import subprocess
import sys

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
so = os.path.join(HERE, "l2cap_probe.so")
if not os.path.exists(so):
    subprocess.check_call(["nvcc", "-O3", "-shared", "-Xcompiler", "-fPIC",
                           "-gencode", "arch=compute_100a,code=sm_100a",
                           os.path.join(HERE, "l2cap_probe.cu"), "-o", so])
lib = C.CDLL(so)
lib.probe_pure.argtypes = [C.c_void_p, C.c_uint64, C.c_int, C.c_uint64, C.c_void_p, C.c_int,
                           C.c_void_p, C.c_int]
MODE = int(os.environ.get("PROBE_LD", 0))
grid = int(os.environ.get("PROBE_GRID", 148 * 8))
iters = int(os.environ.get("PROBE_ITERS", 256))
out = torch.empty(grid * 256, dtype=torch.int64, device="cuda")
s = torch.cuda.current_stream().cuda_stream
sizes = [int(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "16,32,48,64,80,96,112,128,160").split(",")]
big = torch.randint(0, 2**62, (max(sizes) << 17,), dtype=torch.int64, device="cuda")
for mb in sizes:
    D = mb << 17  # MB of int64
    for _ in range(3):
        lib.probe_pure(big.data_ptr(), D, iters, 1, out.data_ptr(), grid, s, MODE)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for r in range(5):
        lib.probe_pure(big.data_ptr(), D, iters, 7 + r, out.data_ptr(), grid, s, MODE)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    reads = grid * 256 * iters
    print(json.dumps({"ld": MODE, "MB": mb, "ms": round(ms, 4), "Greads_per_s": round(reads / ms / 1e6, 1)}),
          flush=True)

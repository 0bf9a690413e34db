"""Does a line streamed from HBM by one die reach the other die from L2?  Both dies
read the same 4 GiB array (mode 1) vs the grid reading it once (mode 0)."""
import ctypes as C
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
import importlib.util  # noqa: E402
_spec = importlib.util.spec_from_file_location("dsp", os.path.join(os.path.dirname(os.path.abspath(__file__)), "dsplit_probe.py"))
_m = importlib.util.module_from_spec(_spec)
_spec.loader.exec_module(_m)
_lib, die_map = _m._lib, _m.die_map

g, _, _ = die_map()
lib = _lib("die_probe")
lib.probe_stream.argtypes = [C.c_void_p, C.c_uint64, C.c_void_p, C.c_void_p, C.c_int, C.c_void_p,
                             C.c_int, C.c_void_p]
n = 1 << 30
a = torch.randint(0, 2**31, (n,), dtype=torch.int32, device="cuda")
die = torch.tensor(g, dtype=torch.uint8, device="cuda")
ctr = torch.zeros(2, dtype=torch.int32, device="cuda")
out = torch.empty(1024, dtype=torch.int64, device="cuda")
s = torch.cuda.current_stream().cuda_stream
for mode in (0, 1, 2):
    for gm in (2, 4, 8):
        f = lambda: lib.probe_stream(a.data_ptr(), n, die.data_ptr(), ctr.data_ptr(), mode,
                                     out.data_ptr(), gm * len(g), s)
        for _ in range(3):
            f()
        if os.environ.get("NCU") == "1":
            torch.cuda.synchronize()
            continue
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            f()
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 10
        print(json.dumps({"mode": mode, "grid_per_sm": gm, "ms": round(ms, 3),
                          "GBps_of_array": round(4 * n / ms / 1e6, 1)}), flush=True)

"""Capacity of L2 for random 32-bit global reductions: whole table from every SM
vs a table split between the two dies (each die reduces into its own half)."""
import ctypes as C
import importlib.util
import json
import os

import torch

_spec = importlib.util.spec_from_file_location(
    "dsp", os.path.join(os.path.dirname(os.path.abspath(__file__)), "dsplit_probe.py"))
_m = importlib.util.module_from_spec(_spec)
_spec.loader.exec_module(_m)
g, _, _ = _m.die_map()
lib = _m._lib("die_probe")
lib.probe_red_split.argtypes = [C.c_void_p, C.c_uint64, C.c_int, C.c_uint64, C.c_void_p, C.c_int,
                                C.c_void_p]
nsm = len(g)
s = torch.cuda.current_stream().cuda_stream
tab = torch.zeros(512 << 18, dtype=torch.int32, device="cuda")  # 512 MB
sgrid = nsm * 8
die = torch.tensor(g, dtype=torch.uint8, device="cuda")
same = torch.zeros(nsm, dtype=torch.uint8, device="cuda")
rnd = torch.zeros(nsm, dtype=torch.uint8)
rnd[torch.randperm(nsm, generator=torch.Generator().manual_seed(5))[: nsm // 2]] = 1
rnd = rnd.cuda()
for mb in (32, 48, 64, 80, 96, 128, 160, 256):
    Dh = (mb << 18) // 2
    for name, grp in (("die", die), ("random", rnd), ("one_half", same)):
        f = lambda seed: lib.probe_red_split(tab.data_ptr(), Dh, 256, seed, grp.data_ptr(), sgrid, s)
        for r in range(3):
            f(1 + r)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for r in range(5):
            f(7 + r)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        print(json.dumps({"MB_total": mb, "groups": name, "ms": round(ms, 4),
                          "Greds_per_s": round(sgrid * 256 * 256 / ms / 1e6, 1)}), flush=True)

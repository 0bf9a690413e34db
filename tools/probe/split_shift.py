"""Die-split random reads: contiguous halves vs interleaved chunks of 2^shift
int64 entries (chunk parity = die).  Which interleave keeps the doubled L2?"""
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
lib.probe_split.argtypes = [C.c_void_p, C.c_uint64, C.c_int, C.c_uint64, C.c_void_p, C.c_void_p,
                            C.c_int, C.c_void_p, C.c_int]
nsm = len(g)
s = torch.cuda.current_stream().cuda_stream
big = torch.randint(0, 2**62, (256 << 17,), dtype=torch.int64, device="cuda")
sgrid = nsm * 8
sout = torch.empty(sgrid * 256, dtype=torch.int64, device="cuda")
die = torch.tensor(g, dtype=torch.uint8, device="cuda")
rnd = torch.zeros(nsm, dtype=torch.uint8)
rnd[torch.randperm(nsm, generator=torch.Generator().manual_seed(5))[: nsm // 2]] = 1
rnd = rnd.cuda()
for mb in (96, 128):
    Dh = (mb << 17) // 2
    for name, grp in (("die", die), ("random", rnd)):
        for shift in (-1, 4, 5, 6, 8, 10, 12, 14, 16, 18, 20):
            f = lambda seed: lib.probe_split(big.data_ptr(), Dh, 256, seed, grp.data_ptr(),
                                             sout.data_ptr(), sgrid, s, shift)
            for r in range(3):
                f(1 + r)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            for r in range(5):
                f(7 + r)
            e1.record()
            torch.cuda.synchronize()
            ms = e0.elapsed_time(e1) / 5
            print(json.dumps({"MB": mb, "groups": name, "shift": shift, "ms": round(ms, 4),
                              "Greads_per_s": round(sgrid * 256 * 256 / ms / 1e6, 1)}), flush=True)

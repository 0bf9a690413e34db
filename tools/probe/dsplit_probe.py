"""Die-split gather probe at C2 (2^30 Zipf(s) FK rows, freq layout, D=2^27 int64).
usage: dsplit_probe.py [s] ; env DSPLIT_RUNS="mode:shift:hot:grid,..."  NCU=1 runs each once
Prints the die map then one JSON line per variant (ms, and equality with mode 0)."""
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


def _lib(name):
    so = os.path.join(HERE, name + ".so")
    if not os.path.exists(so):
        subprocess.check_call(["nvcc", "-O3", "-shared", "-Xcompiler", "-fPIC", "-lineinfo",
                               "-gencode", "arch=compute_100a,code=sm_100a",
                               os.path.join(HERE, name + ".cu"), "-o", so])
    return C.CDLL(so)


def die_map(iters=512, mb=40):
    """SM -> die (0/1) from the pair test of die_probe.cu (SM 0's die = 1)."""
    lib = _lib("die_probe")
    lib.probe_pair.argtypes = [C.c_void_p, C.c_uint64, C.c_int, C.c_uint64, C.c_int, C.c_int,
                               C.c_void_p, C.c_void_p, C.c_int, C.c_void_p]
    nsm = torch.cuda.get_device_properties(0).multi_processor_count
    s = torch.cuda.current_stream().cuda_stream
    D = mb << 17
    tab = torch.randint(0, 2**62, (2 * D,), dtype=torch.int64, device="cuda")
    out = torch.empty(nsm * 1024, dtype=torch.int64, device="cuda")
    cyc = torch.zeros(nsm, dtype=torch.int64, device="cuda")
    res = []
    for j in range(1, nsm):
        for r in range(2):
            lib.probe_pair(tab.data_ptr(), D, iters, 11 + r, 0, j, out.data_ptr(), cyc.data_ptr(), nsm, s)
        torch.cuda.synchronize()
        res.append(int(cyc[0]))
    lo, hi = min(res), max(res)
    thr = (lo + hi) / 2
    g = [1] + [1 if c > thr else 0 for c in res]
    return g, lo, hi


if __name__ == "__main__":
    z = float(sys.argv[1]) if len(sys.argv) > 1 else 1.0
    g, lo, hi = die_map()
    print(json.dumps({"die_map": g, "n_die1": sum(g), "lo": lo, "hi": hi}), flush=True)
    lib = _lib("dsplit_probe")
    lib.probe_dg.argtypes = [C.c_int, C.c_void_p, C.c_uint64, C.c_void_p, C.c_uint64, C.c_void_p,
                             C.c_void_p, C.c_void_p, C.c_uint32, C.c_int, C.c_int, C.c_void_p]
    n, d = 1 << 30, 1 << 27
    dim = dsm.fill_column(0, torch.int64, d, 3)
    cdf = torch.from_numpy(sx.zipf_cdf(d, z)).cuda()
    fact = sx.generate_zipf(cdf, n, 7)
    del cdf
    out = torch.empty(n, dtype=torch.int64, device="cuda")
    ref = torch.empty(n, dtype=torch.int64, device="cuda")
    die = torch.tensor(g, dtype=torch.uint8, device="cuda")
    ctr = torch.zeros(2, dtype=torch.int32, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    nsm = len(g)
    ncu = os.environ.get("NCU") == "1"
    runs = os.environ.get("DSPLIT_RUNS", "0:4:0:8,3:4:0:2,1:4:0:2,1:5:0:2,1:7:0:2,1:9:0:2,"
                                         "2:4:65536:2,2:4:1048576:2,5:4:0:2")

    def run(mode, shift, hot, gm, o):
        assert lib.probe_dg(mode, fact.data_ptr(), n // 4, dim.data_ptr(), d, o.data_ptr(),
                            die.data_ptr(), ctr.data_ptr(), hot, shift, gm * nsm, s) == 0

    run(0, 4, 0, 8, ref)
    torch.cuda.synchronize()
    for spec in runs.split(","):
        mode, shift, hot, gm = (int(x) for x in spec.split(":"))
        out.fill_(0)
        if ncu:
            run(mode, shift, hot, gm, out)
            torch.cuda.synchronize()
            continue
        for _ in range(3):
            run(mode, shift, hot, gm, out)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            run(mode, shift, hot, gm, out)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 10
        eq = bool(torch.equal(out, ref)) if mode != 5 else None
        print(json.dumps({"z": z, "mode": mode, "shift": shift, "hot": hot, "grid_per_sm": gm,
                          "ms": round(ms, 3), "frac": round(12 * n / ms / 1e6 / 6545.3, 4),
                          "equal": eq}), flush=True)

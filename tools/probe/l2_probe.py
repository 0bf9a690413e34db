"""Drive tools/probe/l2_probe.cu at C2 (D=2^27 int64, 2^30 Zipf rows, freq layout)."""
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

so = os.path.join(HERE, "l2_probe.so")
if not os.path.exists(so):
    subprocess.check_call(["nvcc", "-O3", "-shared", "-Xcompiler", "-fPIC", "-std=c++17",
                           "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
                           os.path.join(HERE, "l2_probe.cu"), "-o", so])
lib = C.CDLL(so)
lib.probe_l2.argtypes = [C.c_int, C.c_int, C.c_uint64, C.c_float, C.c_uint32, C.c_void_p,
                         C.c_uint64, C.c_void_p, C.c_void_p, C.c_void_p]
lib.probe_setaside.argtypes = [C.c_uint64]

ctx = sx.context(0)
n = 1 << 30
d = 1 << 27
dim = dsm.fill_column(0, torch.int64, d, 3)
out = torch.empty(n, dtype=torch.int64, device="cuda")
ref = torch.empty(n, dtype=torch.int64, device="cuda")
stream = torch.cuda.current_stream().cuda_stream
pmax = torch.cuda.get_device_properties(0).persisting_l2_cache_max_size if hasattr(
    torch.cuda.get_device_properties(0), "persisting_l2_cache_max_size") else 82903040
MB = 1 << 20
zs = [float(x) for x in (sys.argv[1] if len(sys.argv) > 1 else "1.0").split(",")]


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


# (h, K entries, setaside bytes, window bytes, hit ratio, grid)
MODE = os.environ.get("PROBE_MODE", "grid")
cfgs = []
if MODE == "grid":
    for grid in (296, 444, 592, 888):
        cfgs.append((0, 0, 0, 0, 1.0, grid))
        cfgs.append((8, 0, 0, 0, 1.0, grid))
        for K in (8 * MB, 12 * MB, 16 * MB):
            for h in (4, 5, 6, 7):
                cfgs.append((h, K, 0, 0, 1.0, grid))
if MODE == "split":
    for grid in (444, 592):
        cfgs.append((0, 0, 0, 0, 1.0, grid))
        for K in (1 * MB, 4 * MB, 8 * MB, 12 * MB, 16 * MB):
            cfgs.append((9, K, 0, 0, 1.0, grid))
            cfgs.append((10, K, 0, 0, 1.0, grid))
if MODE == "tail":
    for K in (1 * MB, 16 * MB):
        for h in (0, 10, 15, 16, 17, 11, 12, 13, 14):
            cfgs.append((h, K, 0, 0, 1.0, 592))
if MODE == "tma":
    for K in (256 * 1024, 1 * MB, 4 * MB, 16 * MB):
        for h in (0, 18, 19, 20, 10):
            cfgs.append((h, K, 0, 0, 1.0, 592))
if MODE == "st":
    for h in (0, 60, 61, 62):
        cfgs.append((h, 0, 0, 0, 1.0, 592))
if MODE == "pf":
    for K in (1 * MB, 16 * MB):
        for h in (0, 50, 51, 10, 52, 53):
            cfgs.append((h, K, 0, 0, 1.0, 592))
if MODE == "atom":
    for K in (1 * MB, 4 * MB, 16 * MB):
        for h in (0, 40, 41, 10, 42):
            cfgs.append((h, K, 0, 0, 1.0, 592))
if MODE == "tmastore":
    for grid in (296, 444, 592):
        cfgs.append((0, 0, 0, 0, 1.0, grid))
        cfgs.append((30, 0, 0, 0, 1.0, grid))
gran = int(os.environ.get("PROBE_GRAN", "0"))
if gran:
    assert lib.probe_set_granularity(gran) == 0
for z in zs:
    cdf = torch.from_numpy(sx.zipf_cdf(d, z)).cuda()
    fact = sx.generate_zipf(cdf, n, 7)
    del cdf
    ctx.set_gather_policy(129)
    lib_ms = timeit(lambda: sx.materialize(fact, dim, out=ref, sync=False))
    print(json.dumps({"z": z, "case": "library", "ms": round(lib_ms, 3)}), flush=True)
    for h, K, sa, win, hr, grid in cfgs:
        rc = lib.probe_setaside(sa)
        if rc:
            print(json.dumps({"z": z, "setaside": sa, "err": rc}), flush=True)
            continue

        def run():
            rc = lib.probe_l2(h, grid, win, hr, K, fact.data_ptr(), n, dim.data_ptr(),
                              out.data_ptr(), stream)
            if rc:
                raise RuntimeError(f"launch rc {rc}")
        try:
            ms = timeit(run)
            ok = bool(torch.equal(out, ref))
        except RuntimeError as e:
            print(json.dumps({"z": z, "h": h, "err": str(e)}), flush=True)
            continue
        lib.probe_setaside(0)
        print(json.dumps({"z": z, "h": h, "K_MB": K * 8 // MB, "setaside_MB": sa // MB,
                          "win_MB": win // MB, "hit": hr, "grid": grid, "ms": round(ms, 3),
                          "ok": ok, "frac": round(n * 12 / (ms * 1e-3) / 6545.3e9, 3)}),
              flush=True)
    del fact

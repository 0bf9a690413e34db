"""Which SMs share an L2 half, and does splitting a random-read table between the
two SM groups recover the full L2 for random reads?  (tools/probe/die_probe.cu)

1. pair test: SM 0 and SM j each read their own 40 MB table at random; cycles of
   SM 0 rise when j shares its die (80 MB competing for one half).
2. split test: all SMs read random entries of the half of an M-MB table their
   group owns, for the discovered grouping and for controls.
Prints JSON lines."""
import ctypes as C
import json
import os
import subprocess
import sys

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
so = os.path.join(HERE, "die_probe.so")
if not os.path.exists(so):
    subprocess.check_call(["nvcc", "-O3", "-shared", "-Xcompiler", "-fPIC",
                           "-gencode", "arch=compute_100a,code=sm_100a",
                           os.path.join(HERE, "die_probe.cu"), "-o", so])
lib = C.CDLL(so)
lib.probe_pair.argtypes = [C.c_void_p, C.c_uint64, C.c_int, C.c_uint64, C.c_int, C.c_int,
                           C.c_void_p, C.c_void_p, C.c_int, C.c_void_p]
lib.probe_split.argtypes = [C.c_void_p, C.c_uint64, C.c_int, C.c_uint64, C.c_void_p, C.c_void_p,
                            C.c_int, C.c_void_p]
lib.probe_smids.argtypes = [C.c_void_p, C.c_int, C.c_void_p]

nsm = torch.cuda.get_device_properties(0).multi_processor_count
s = torch.cuda.current_stream().cuda_stream
big = torch.randint(0, 2**62, (256 << 17,), dtype=torch.int64, device="cuda")

# --- 1. pair test -----------------------------------------------------------
PAIR_MB = int(os.environ.get("PAIR_MB", 40))
D = PAIR_MB << 17
grid = nsm
out = torch.empty(grid * 1024, dtype=torch.int64, device="cuda")
cyc = torch.zeros(nsm, dtype=torch.int64, device="cuda")
iters = int(os.environ.get("PAIR_ITERS", 2048))
ref = int(os.environ.get("PAIR_REF", 0))


def pair(a, b):
    cyc.zero_()
    for r in range(2):  # first launch warms, second is measured
        assert lib.probe_pair(big.data_ptr(), D, iters, 11 + r, a, b, out.data_ptr(),
                              cyc.data_ptr(), grid, s) == 0
    torch.cuda.synchronize()
    c = cyc.cpu()
    return int(c[a]), int(c[b]) if b >= 0 else 0


alone, _ = pair(ref, -1)
rows = []
for j in range(nsm):
    if j == ref:
        continue
    ca, cb = pair(ref, j)
    rows.append((j, ca, cb))
print(json.dumps({"pair_alone_cycles": alone, "pair_mb_each": PAIR_MB}), flush=True)
vals = sorted(r[1] for r in rows)
thr = (vals[0] + vals[-1]) / 2
same = [ref] + [j for j, ca, cb in rows if ca > thr]
print(json.dumps({"pair": [[j, ca, cb] for j, ca, cb in rows]}), flush=True)
print(json.dumps({"threshold": thr, "same_die_as_ref": sorted(same), "n_same": len(same),
                  "min": vals[0], "max": vals[-1]}), flush=True)

# --- 2. split test ------------------------------------------------------------
disc = torch.zeros(nsm, dtype=torch.uint8)
for j in same:
    disc[j] = 1
cands = {
    "discovered": disc,
    "half_smid": torch.tensor([1 if i < nsm // 2 else 0 for i in range(nsm)], dtype=torch.uint8),
    "parity": torch.tensor([i & 1 for i in range(nsm)], dtype=torch.uint8),
    "all_same": torch.zeros(nsm, dtype=torch.uint8),
}
g = torch.Generator().manual_seed(5)
cands["random"] = torch.randperm(nsm, generator=g)[: nsm // 2]
rnd = torch.zeros(nsm, dtype=torch.uint8)
rnd[cands["random"]] = 1
cands["random"] = rnd
sgrid = nsm * 8
sout = torch.empty(sgrid * 256, dtype=torch.int64, device="cuda")
siters = 256
for mb in [int(x) for x in os.environ.get("SPLIT_MB", "64,96,128,160,192").split(",")]:
    Dh = (mb << 17) // 2
    for name, grp in cands.items():
        gd = grp.cuda()
        for r in range(3):
            lib.probe_split(big.data_ptr(), Dh, siters, 1 + r, gd.data_ptr(), sout.data_ptr(), sgrid, s)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for r in range(5):
            lib.probe_split(big.data_ptr(), Dh, siters, 7 + r, gd.data_ptr(), sout.data_ptr(), sgrid, s)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        print(json.dumps({"split": name, "MB_total": mb, "ms": round(ms, 4),
                          "Greads_per_s": round(sgrid * 256 * siters / ms / 1e6, 1)}), flush=True)

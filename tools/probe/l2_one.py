"""Run one l2_probe configuration twice (for ncu: profile the 2nd launch of k_l2).
usage: l2_one.py z h K_entries grid [h K grid ...]"""
import ctypes as C
import os
import sys

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from paper_1910_10063_b200 import dataset as dsm  # noqa: E402
from paper_1910_10063_b200 import skewdx as sx  # noqa: E402

lib = C.CDLL(os.path.join(HERE, "l2_probe.so"))
lib.probe_l2.argtypes = [C.c_int, C.c_int, C.c_uint64, C.c_float, C.c_uint32, C.c_void_p,
                         C.c_uint64, C.c_void_p, C.c_void_p, C.c_void_p]
n, d = 1 << 30, 1 << 27
z = float(sys.argv[1])
gran = int(os.environ.get("PROBE_GRAN", "0"))
if gran:
    assert lib.probe_set_granularity(gran) == 0
dim = dsm.fill_column(0, torch.int64, d, 3)
out = torch.empty(n, dtype=torch.int64, device="cuda")
cdf = torch.from_numpy(sx.zipf_cdf(d, z)).cuda()
fact = sx.generate_zipf(cdf, n, 7)
stream = torch.cuda.current_stream().cuda_stream
args = sys.argv[2:]
for i in range(0, len(args), 3):
    h, K, grid = int(args[i]), int(args[i + 1]), int(args[i + 2])
    for _ in range(2):
        assert lib.probe_l2(h, grid, 0, 1.0, K, fact.data_ptr(), n, dim.data_ptr(),
                            out.data_ptr(), stream) == 0
    torch.cuda.synchronize()
print("done")

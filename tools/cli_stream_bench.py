"""Time the index CLI on a 2^28-row (1 GiB) SKDX fact column (Zipf(1.0) over
2^24 ids, original layout): index build (streamed histogram + device sort) and
index apply (streamed recode).  Wall clock around each command; the page cache
is warm after the file is written, so this is the pipeline, not the disk."""
import json
import os
import struct
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from oracle.oracle import Oracle  # noqa: E402  (fixture generator, not the measured path)

CLI = os.path.join(ROOT, "paper_1910_10063_b200", "skewdx_b200_cli")
n, d = 1 << 28, 1 << 24
orc = Oracle()
fact = orc.generate_zipf_counter(orc.zipf_cdf(d, 1.0), orc.random_bijection(d, 5), 5, 0, n)
tmp = tempfile.mkdtemp()
f = os.path.join(tmp, "f.skdx")
with open(f, "wb") as fh:
    fh.write(b"SKDX" + struct.pack("<IQ", 1, n) + fact.astype(np.uint32).tobytes())
res = {"rows": n, "domain": d, "file_bytes": os.path.getsize(f)}
for name, args in [("build", ["index", "build", "--fact", f, "--d", str(d), "--out", f + ".skpi"]),
                   ("apply", ["index", "apply", "--index", f + ".skpi", "--fact", f,
                              "--fact-out", f + ".r"])]:
    best = 1e9
    for _ in range(3):
        t0 = time.perf_counter()
        r = subprocess.run([CLI, *args], capture_output=True, text=True)
        best = min(best, time.perf_counter() - t0)
        assert r.returncode == 0, r.stderr
    res[name + "_s"] = round(best, 3)
    res[name + "_GBps_of_fact"] = round(4 * n / best / 1e9, 2)
print(json.dumps(res))

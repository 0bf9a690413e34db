"""A small forced partitioned gather (policy 129 | 8192 | 16384), sized for a
compute-sanitizer memcheck / racecheck run (closed on this pool: the wrapper refuses it, so the
shared-memory hand-offs of k_pg_part / k_pg_emit_s are argued in gather.cu and covered by the
parity tests).  One ragged launch per width over a dimension just past two hot prefixes (1 partition) and one
with 3 partitions; results checked against numpy."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_1910_10063_b200 import skewdx as sx  # noqa: E402

ctx = sx.context(0)
ctx.set_gather_policy(129 | 8192 | 16384)
rng = np.random.default_rng(3)
for npdt in (np.uint32, np.uint64):
    w = np.dtype(npdt).itemsize
    hot = (32 << 20) // w
    for d in (2 * hot + 1, 5 * hot + 77):
        dim_np = rng.integers(0, np.iinfo(npdt).max, size=d, dtype=npdt)
        n = (1 << 22) + 8192 + 5
        fact_np = rng.integers(1, d + 1, size=n, dtype=np.uint32)
        fact_np[::7] = rng.integers(1, 1000, size=fact_np[::7].size)
        dim = torch.from_numpy(dim_np.view(np.int64 if w == 8 else np.int32)).cuda()
        fact = torch.from_numpy(fact_np.view(np.int32)).cuda().view(torch.uint32)
        out = sx.materialize(fact, dim)
        plan = ctx.gather_last_plan()
        got = out.cpu().numpy().view(npdt)
        ok = np.array_equal(got, dim_np[fact_np.astype(np.int64) - 1])
        print(npdt.__name__, d, "partitioned" if plan["partitioned"] else "one-pass", "ok" if ok else "MISMATCH")
        assert ok and plan["partitioned"]
print("done")

"""Multi-rank path of bench.py (torchrun, row shards, all-reduced histogram,
max-over-ranks timing, rank-0 JSON line) as a logic dry run on ONE GPU: two
ranks share cuda:0 and use host-side gloo collectives, so no kernel waits on
another rank's kernel.  Scaling numbers come only from the real N-GPU run."""
import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu


def test_bench_two_ranks_dry_run():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    env = dict(os.environ, SKX_BENCH_ONE_GPU="1", SKX_BENCH_DIST_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", "29547", "bench.py", "--gpus", "2",
           "--steps", "3", "--warmup", "3", "--rows", str(1 << 24), "--domain", str(1 << 20),
           "--no-cpu", "--no-e2e"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-4000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]  # rank 0 only
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["config"]["rows_total"] == 2 << 24
    assert d["rand_layout"]["outputs_equal"] and d["index_build"]["deterministic"]
    assert d["value"] > 0 and d["scaling"] == "weak"

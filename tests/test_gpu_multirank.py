"""The multi-GPU path on the one available GPU.

* dist.py's orchestration with the REAL kernels (GpuExecutor): two ranks share
  cuda:0 and combine over gloo (host-staged), so no kernel waits on another
  rank's kernel; the concatenated shard outputs must equal the N=1 outputs
  (index, recode, gather, group-by through the packed combine, config-5
  offsets and exactly combined category sums) and a violation in one shard
  must raise the same DomainViolation on both ranks.
* libskx's NCCL communicator (skx_comm_init_rank / skx_comm_init_all) with
  one rank: every collective entry runs and keeps the identity semantics.
* bench.py's torchrun path in strong-scaling mode as a 2-rank dry run.
Scaling numbers come only from the real N-GPU run."""
import ctypes as C
import json
import os
import socket
import subprocess
import sys

import numpy as np
import pytest
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
pytestmark = pytest.mark.gpu

D, N = 1 << 16, (1 << 22) + 12345


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _inputs(sx, ds, shard):
    fact = ds.make_rand_fact(D, N, 1.1, 77, shard)
    dim = ds.fill_column(ds.KIND_RAW, torch.int64, D, 78)
    qty = ds.fill_column(ds.KIND_UNIFORM, torch.int64, shard.rows, ds.qty_seed(79, shard.begin), 1,
                         100)
    cat = ds.fill_column(ds.KIND_UNIFORM, torch.int32, D, 80, 0, 1000)
    price = ds.fill_column(ds.KIND_LOGNORMAL, torch.float32, D, 81, 3.0, 1.0)
    supp = ds.fill_column(ds.KIND_RAW, torch.int64, D, 82)
    flag = ds.fill_column(ds.KIND_RAW, torch.int16, D, 83)
    return fact, dim, qty, (cat, price, supp, flag)


def _run(sx, ds, sdist, coll, shard):
    ex = sdist.GpuExecutor()
    fact, dim, qty, cols = _inputs(sx, ds, shard)
    idx, _ = sdist.rebuild(fact, D, N, ex, coll, shard)
    rec = ex.recode(fact, idx)
    dperm = ex.permute(dim, idx)
    out = sdist.gather(rec, dperm, ex)
    st = {}
    counts, sums = sdist.aggregate(rec, qty, D, ex, coll, shard, hot=1024, stats=st)
    cat_p = tuple(ex.permute(c, idx) for c in cols)
    bm = sx.build_bitmap_lt(cat_p[0], 100)
    sel = sdist.select_gather_sum(rec, bm, cat_p, 1000, ex, coll, shard, capacity=shard.rows)
    torch.cuda.synchronize()
    k = int(sel[6].item())
    res = {"off": idx.offsets, "rk": idx.ranks, "rec": rec, "out": out, "counts": counts,
           "sums": sums, "sel_off": sel[0][:k], "sel_price": sel[2][:k], "cat_sums": sel[5]}
    res = {a: b.cpu().numpy() for a, b in res.items()}
    res["path"] = st.get("path", "single")
    bad = fact.clone()
    if shard.rank == 1 or shard.world == 1:
        bad[17] = D + 9
    try:
        sdist.rebuild(bad, D, N, ex, coll, shard)
        res["raised"] = -1
    except sx.DomainViolation as e:
        res["raised"] = e.row()
    return res


def _worker(rank, world, port, out_dir):
    import torch.distributed as dist
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1910_10063_b200 import dataset as ds
    from paper_1910_10063_b200 import dist as sdist
    from paper_1910_10063_b200 import skewdx as sx
    coll = sdist.default_collectives(0)
    res = _run(sx, ds, sdist, coll, sdist.shard_for(N))
    np.savez(os.path.join(out_dir, f"r{rank}.npz"), **res)
    dist.destroy_process_group()


def test_dist_two_ranks_equal_one(tmp_path):
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    import torch.multiprocessing as mp
    mp.spawn(_worker, args=(2, _free_port(), str(tmp_path)), nprocs=2, join=True)
    from paper_1910_10063_b200 import dataset as ds
    from paper_1910_10063_b200 import dist as sdist
    from paper_1910_10063_b200 import skewdx as sx
    one = _run(sx, ds, sdist, sdist.Single(), sdist.shard_for(N, 0, 1))
    r = [np.load(tmp_path / f"r{k}.npz") for k in range(2)]
    b1 = sdist.shard_for(N, 1, 2).begin
    for k in range(2):
        assert np.array_equal(r[k]["off"], one["off"]) and np.array_equal(r[k]["rk"], one["rk"])
        assert int(r[k]["raised"]) == b1 + 17  # same global row on both ranks
    assert int(one["raised"]) == 17
    for key in ("rec", "out"):
        assert np.array_equal(np.concatenate([r[0][key], r[1][key]]), one[key]), key
    assert str(r[0]["path"]) == "packed"
    assert np.array_equal(r[0]["counts"], one["counts"]) and np.array_equal(r[0]["sums"], one["sums"])
    for key in ("sel_off", "sel_price"):
        assert np.array_equal(np.concatenate([r[0][key], r[1][key]]), one[key]), key
    # the exact fixed-point combine rounds once: bit-identical to the one-GPU sums
    assert np.array_equal(r[0]["cat_sums"], one["cat_sums"])


def test_nccl_communicator_one_rank():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_1910_10063_b200 import _native
    from paper_1910_10063_b200 import dist as sdist
    lib = _native.load()
    buf = C.create_string_buffer(128)
    assert lib.skx_comm_unique_id(buf) == 0
    coll = sdist.SkxCollectives(0, 1, 0, buf.raw)
    try:
        a = torch.arange(1000, dtype=torch.int64, device="cuda")
        u = torch.arange(1000, dtype=torch.int32, device="cuda").view(torch.uint32)
        f = torch.linspace(0, 1, 1000, dtype=torch.float64, device="cuda")
        assert torch.equal(coll.allreduce(a.clone()), a)
        assert torch.equal(coll.allreduce(u.clone()).view(torch.int32), u.view(torch.int32))
        assert torch.equal(coll.reduce(f.clone(), 0), f)
        assert torch.equal(coll.allreduce(a.clone(), sdist.MAX), a)
        assert torch.equal(coll.allgather(a), a)
        assert lib.skx_comm_sync(coll.handle) == 0
        n, r0, nl = C.c_int(), C.c_int(), C.c_int()
        lib.skx_comm_info(coll.handle, C.byref(n), C.byref(r0), C.byref(nl))
        assert (n.value, r0.value, nl.value) == (1, 0, 1)
        # bad arguments are rejected before NCCL
        assert lib.skx_reduce(coll.handle, (C.c_void_p * 1)(a.data_ptr()), 10, 99, 0, 0, None) == 1
        assert lib.skx_reduce(coll.handle, (C.c_void_p * 1)(a.data_ptr()), 10, 3, 0, 5, None) == 1
    finally:
        coll.close()
    # single process, all local devices (here: one)
    h = C.c_void_p()
    dev = (C.c_int * 1)(0)
    assert lib.skx_comm_init_all(1, dev, C.byref(h)) == 0
    x = torch.arange(64, dtype=torch.int64, device="cuda")
    stream = (C.c_void_p * 1)(torch.cuda.current_stream().cuda_stream)
    assert lib.skx_allreduce(h, (C.c_void_p * 1)(x.data_ptr()), 64, 3, 0, stream) == 0
    torch.cuda.synchronize()
    assert torch.equal(x, torch.arange(64, dtype=torch.int64, device="cuda"))
    assert lib.skx_comm_ctx(h, 0) and not lib.skx_comm_ctx(h, 1)
    assert lib.skx_comm_destroy(h) == 0


def test_combine_kernels_vs_numpy():
    """skx_groupby_pack / unpack and the select-sum partials, on the device,
    against their numpy restatement."""
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_1910_10063_b200 import dist as sdist
    ex = sdist.GpuExecutor()
    rng = np.random.default_rng(3)
    d, hot = 100003, 4096
    c = rng.integers(0, 1 << 20, size=d, dtype=np.uint64)
    s = rng.integers(0, 1 << 36, size=d, dtype=np.uint64)
    c[7], s[hot + 5] = np.uint64(1 << 40), np.uint64(3 << 38)  # hot key large; tail sum near 2^40
    ct = torch.from_numpy(c.view(np.int64)).cuda().view(torch.uint64)
    st = torch.from_numpy(s.view(np.int64)).cuda().view(torch.uint64)
    buf, guard = ex.groupby_pack(ct, st, hot)
    b = buf.cpu().view(torch.int64).numpy().view(np.uint64)
    assert np.array_equal(b[:hot], c[:hot]) and np.array_equal(b[hot:2 * hot], s[:hot])
    assert np.array_equal(b[2 * hot:], (c[hot:] << np.uint64(40)) | s[hot:])
    g = guard.cpu().view(torch.int64).numpy().view(np.uint64)
    assert g[0] == c[hot:].max() and g[1] == s[hot:].max()
    c2, s2 = torch.empty_like(ct), torch.empty_like(st)
    ex.groupby_unpack(buf, d, hot, c2, s2)
    assert torch.equal(c2.view(torch.int64), ct.view(torch.int64))
    assert torch.equal(s2.view(torch.int64), st.view(torch.int64))


def test_bench_two_ranks_dry_run():
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    env = dict(os.environ, SKX_BENCH_ONE_GPU="1", SKX_BENCH_DIST_BACKEND="gloo")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()), "bench.py",
           "--gpus", "2", "--steps", "3", "--warmup", "3", "--rows", str(1 << 24), "--domain",
           str(1 << 20), "--no-cpu", "--no-e2e", "--configs", "c2,c3"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stderr[-4000:]
    lines = [ln for ln in r.stdout.splitlines() if ln.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]  # rank 0 only
    d = json.loads(lines[0])
    assert d["n_gpus"] == 2 and d["scaling"] == "strong"
    assert d["config"]["rows_total"] == 1 << 24 and d["config"]["rows_per_gpu"] == 1 << 23
    assert d["rand_layout"]["outputs_equal"] and d["index_build"]["deterministic"]
    assert d["value"] > 0
    gb = d["groupby_c3"]
    assert gb["combine"]["path"] == "packed" and "reduce" in gb["phases_ms"]

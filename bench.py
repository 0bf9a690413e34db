#!/usr/bin/env python
"""Benchmark of the skew-reordered FK-join gather (+ group-by) on B200.

Headline workload (BASELINE.json configs[1], "Large FK-join gather"): a
dimension of 2^27 keys with an int64 value column (1 GiB), 2^30 int32 FK rows
drawn Zipf(s) over ranks with ranks scattered to ids by a seeded random
bijection, the skew-aware index built on the GPU (histogram -> sort-by-count
-> recode -> permute), and the timed step is one gather
``out[k] = dim_freq[fact_freq[k]-1]`` over every fact row of the (reordered)
layout -- one ``skx_gather_u64`` launch.  Scaling is weak: every GPU owns a
2^30-row shard of the fact table (rows partitioned, no data-path collective
for the gather) and the dimension columns are replicated; the index build
all-reduces the per-GPU histograms.

Prints ONE JSON line (rank 0).  ``--impl reference`` times the reference's
CPU path on the host instead.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

D_C2, N_C2, SEED = 1 << 27, 1 << 30, 42
# BASELINE.json's metric, verbatim.  `value` is quoted on configs[1] (the C2 gather, the
# configuration the metric names that fits one GPU); the group-by's line is `groupby_c3`.
METRIC = "fact rows/s for skew-reordered FK-join gather + group-by; % of HBM roofline"
METRIC_NOTE = ("value = C2 skew-reordered FK-join gather rows/s (configs[1]); roofline.frac = its "
               "fraction of the HBM roofline; the group-by (configs[2]) is groupby_c3 in this line")
D_C3 = 1 << 24
CPU_SAMPLE_ROWS = 1 << 27


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=30)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", choices=["ours", "reference"], default="ours")
    p.add_argument("--z", type=float, default=1.0, help="Zipf exponent (C2 sweeps 0.5/1.0/1.5)")
    p.add_argument("--rows", type=int, default=N_C2, help="fact rows per GPU")
    p.add_argument("--domain", type=int, default=D_C2)
    p.add_argument("--no-extras", action="store_true", help="skip rand-layout / group-by lines")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu", action="store_true")
    p.add_argument("--policy", type=int, default=129,
                   help="skx_set_gather_policy bits (include/skx.h); 129 = library default")
    return p.parse_args()


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            pk = json.load(f)
        return float(pk["hbm_gbs"]), "measured"
    except Exception:  # noqa: BLE001
        return 6650.0, "fallback"


def ncu_traffic(name):
    """Per-launch DRAM bytes from the committed ncu --set full capture."""
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            return json.load(f).get(name)
    except Exception:  # noqa: BLE001
        return None


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled DURING the timed region."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "20"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:  # noqa: BLE001
            self.proc = None

    def stop(self):
        if self.proc is None:
            return None
        self.proc.terminate()
        try:
            out, _ = self.proc.communicate(timeout=5)
        except Exception:  # noqa: BLE001
            self.proc.kill()
            out, _ = self.proc.communicate()
        rows = []
        for line in out.strip().splitlines():
            parts = [x.strip() for x in line.split(",")]
            if len(parts) == 6:
                try:
                    rows.append((float(parts[0]), float(parts[1]), parts[2:]))
                except ValueError:
                    pass
        if not rows:
            return None
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for _, _, r in rows for i, v in enumerate(r) if v == "Active"})
        return {"sm_mhz": statistics.median(r[0] for r in rows), "sm_max_mhz": max(r[1] for r in rows),
                "samples": len(rows), "reasons": reasons}


# ---------------------------------------------------------------------------
# CPU side (rank 0, N=1): the reference's path on the host's cores
# ---------------------------------------------------------------------------
REF_NOTE = ("the reference's KernelTable/parallel_materialize gathers u32 values only "
            "(kernels.hpp:21-23), so it runs on the dimension truncated to u32: half the value "
            "bytes of the int64 workload, which favours the reference")


def _ref_parallel_materialize_rows_per_s(ref, fact_np, dim_np, threads, steps, warmup=1):
    """The unmodified reference's public parallel_materialize (parallel.cpp:87-100,
    incl. its serial domain scan and output allocation), median of `steps`."""
    import ctypes as C
    import numpy as np
    dim32 = np.ascontiguousarray(dim_np.astype(np.uint32))
    fp, dp = fact_np.ctypes.data_as(C.c_void_p), dim32.ctypes.data_as(C.c_void_p)
    for _ in range(max(0, warmup - 1)):
        ref.L.ref_time_parallel_materialize(fp, len(fact_np), dp, len(dim32), threads, 1)
    ns = ref.L.ref_time_parallel_materialize(fp, len(fact_np), dp, len(dim32), threads,
                                             max(1, steps))
    out32 = np.empty(len(fact_np), np.uint32)
    kns = ref.L.ref_time_gather_kernel(fp, len(fact_np), dp, out32.ctypes.data_as(C.c_void_p),
                                       threads, 3)
    return len(fact_np) / (ns * 1e-9), len(fact_np) / (kns * 1e-9), ref.active_kernels_name()


def _port_rows_per_s(orc, fact_np, dim_np, threads, steps, warmup=1):
    import numpy as np
    out = np.empty(len(fact_np), np.uint64)
    for _ in range(max(1, warmup)):
        orc.parallel_gather_u64(fact_np, dim_np, out, threads)
    ts = []
    for _ in range(max(1, steps)):
        t0 = time.perf_counter()
        orc.parallel_gather_u64(fact_np, dim_np, out, threads)
        ts.append(time.perf_counter() - t0)
    return len(fact_np) / statistics.median(ts)


def cpu_gather_baseline(fact_np, dim_np, steps=3):
    """The reference's own parallel_materialize (oracle/_ref, built from the
    reference sources) on a bounded sample of the C2 workload with all host
    threads; the int64 port of the same algorithm and the reference's raw
    KernelTable gather are reported beside it."""
    from oracle.oracle import Oracle, Reference
    orc = Oracle()
    threads = os.cpu_count() or 1
    port = _port_rows_per_s(orc, fact_np, dim_np, threads, steps)
    try:
        ref = Reference()
        value, kernel, table = _ref_parallel_materialize_rows_per_s(ref, fact_np, dim_np, threads,
                                                                    steps)
        return {"value": value, "unit": "rows/s", "cores": threads, "kind": "reference",
                "sample": (f"{len(fact_np)} rows of the same reordered (freq) FK shard, full "
                           f"{len(dim_np)}-key dimension; unmodified reference "
                           f"parallel_materialize ({table} KernelTable), {threads} threads, "
                           f"median of {steps}; {REF_NOTE}"),
                "reference_kernel_only_rows_per_s": kernel,
                "port_i64_rows_per_s": port}
    except Exception as e:  # noqa: BLE001
        return {"value": port, "unit": "rows/s", "cores": threads, "kind": "port",
                "sample": (f"{len(fact_np)} rows of the same reordered (freq) FK shard, full "
                           f"{len(dim_np)}-key int64 dimension; parallel_materialize port "
                           f"(parallel.cpp:87-100, i64 width), {threads} threads, median of "
                           f"{steps}"),
                "reference_note": f"oracle/_ref unavailable: {e}"}


def _cpu_extra(fn):
    """CPU reference timings beside the C3/C4/C5 lines: never fatal."""
    try:
        return fn()
    except Exception as e:  # noqa: BLE001
        return {"unavailable": f"{type(e).__name__}: {e}"}


def cpu_groupby_reference(fact_np, qty_np, d):
    """C3 on the host: the reference's parallel_aggregate (hybrid, h=8192, all
    threads; COUNT only -- parallel.cpp:131-216) on a 2^26-row sample and its
    single-thread aggregate_sum (operators.cpp:107-118, the reference has no
    parallel SUM) on a 2^24-row sample, both of the recoded C3 FK column."""
    import ctypes as C

    import numpy as np
    from oracle.oracle import Reference
    ref = Reference()
    threads = os.cpu_count() or 1
    f = np.ascontiguousarray(fact_np[:1 << 26])
    ns = ref.L.ref_time_parallel_aggregate(f.ctypes.data_as(C.c_void_p), len(f), d, threads, 2,
                                           8192, 3)
    f2 = np.ascontiguousarray(fact_np[:1 << 24])
    q2 = np.ascontiguousarray(qty_np[:1 << 24].astype(np.uint32))  # 1..100 fits u32
    ns2 = ref.L.ref_time_aggregate_sum(f2.ctypes.data_as(C.c_void_p), q2.ctypes.data_as(C.c_void_p),
                                       len(f2), d, 1)
    return {"parallel_aggregate_count_rows_per_s": len(f) / (ns * 1e-9), "threads": threads,
            "aggregate_sum_1thread_rows_per_s": len(f2) / (ns2 * 1e-9), "kind": "reference",
            "sample": f"{len(f)} / {len(f2)} rows of the recoded C3 FK column (D={d})",
            "heavy_hitters": cpu_heavy_hitters_reference(f, d)}


def cpu_heavy_hitters_reference(fact_np, d, k=8192):
    """Q3a on the host: the reference's heavy_hitter_count (operators.cpp:184-203,
    single thread) on a 2^26-row sample of the recoded C3 column."""
    import ctypes as C

    import numpy as np
    from oracle.oracle import Reference
    ref = Reference()
    f = np.ascontiguousarray(fact_np)
    ids = np.empty(k, np.uint32)
    cnt = np.empty(k, np.uint64)
    ln = C.c_uint64(0)
    cl = C.c_int(0)
    ts = []
    for _ in range(3):
        t0 = time.perf_counter()
        ref.L.ref_heavy_hitter_count(f.ctypes.data_as(C.c_void_p), len(f), d, k,
                                     ids.ctypes.data_as(C.c_void_p), cnt.ctypes.data_as(C.c_void_p),
                                     C.byref(ln), C.byref(cl))
        ts.append(time.perf_counter() - t0)
    return {"heavy_hitter_count_1thread_rows_per_s": len(f) / statistics.median(ts[1:]),
            "kind": "reference", "sample": f"{len(f)} rows, k={k}, D={d}"}


def cpu_rebuild_reference(fact_np, d):
    """C4 on the host: the reference's rebuild (count_frequencies + build_index,
    single thread -- the reference has no parallel index build) at the
    CPU-runnable scale of BASELINE configs[0] (D=2^22, 2^24 rows)."""
    import ctypes as C

    import numpy as np
    from oracle.oracle import Reference
    ref = Reference()
    f = np.ascontiguousarray(fact_np)
    ns = ref.L.ref_time_rebuild(f.ctypes.data_as(C.c_void_p), len(f), d, 1)
    return {"rebuild_1thread_ms": ns * 1e-6, "rows_per_s": len(f) / (ns * 1e-9), "kind": "reference",
            "sample": f"{len(f)} Zipf(1.25) rows over D={d} (configs[0] scale)"}


def cpu_select_reference(fact_np, words_np, bits):
    """C5 selection on the host: the reference's parallel_select
    (parallel.cpp:102-129, all threads) with the same permuted bitmap on a
    2^26-row sample of the recoded FK column."""
    import ctypes as C

    import numpy as np
    from oracle.oracle import Reference
    ref = Reference()
    threads = os.cpu_count() or 1
    f = np.ascontiguousarray(fact_np)
    w = np.ascontiguousarray(words_np)
    sel = C.c_uint64(0)
    ns = ref.L.ref_time_parallel_select(f.ctypes.data_as(C.c_void_p), len(f),
                                        w.ctypes.data_as(C.c_void_p), bits, threads, 3,
                                        C.byref(sel))
    return {"parallel_select_rows_per_s": len(f) / (ns * 1e-9), "threads": threads,
            "selected": int(sel.value), "kind": "reference",
            "sample": f"{len(f)} rows of the recoded C5 FK column, permuted bitmap over D={bits}"}


def run_reference_arm(args):
    """--impl reference: the reference's CPU gather on a bounded sample of the
    same workload, all host threads, K timed steps after W warm-ups."""
    import numpy as np
    from oracle.oracle import Oracle, Reference
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    orc = Oracle()
    threads = os.cpu_count() or 1
    d = args.domain
    rows = min(CPU_SAMPLE_ROWS, args.rows)
    # Inputs: the counter-based Zipf draw of the same (D, s, seed), ids = ranks
    # (the skew-reordered layout, Layout::freq up to empirical tie order).
    cdf = orc.zipf_cdf(d, args.z)
    fact = orc.generate_zipf_counter_mt(cdf, None, SEED, rows, threads)
    dim = np.random.default_rng(SEED).integers(0, 2**63, size=d, dtype=np.uint64)
    port = _port_rows_per_s(orc, fact, dim, threads, args.steps, args.warmup)
    extra = {"port_i64_rows_per_s": port}
    try:
        ref = Reference()
        value, kernel, table = _ref_parallel_materialize_rows_per_s(ref, fact, dim, threads,
                                                                    args.steps, args.warmup)
        kind = "reference"
        sample = (f"{rows} rows per step of the C2 workload (D={d}, s={args.z}, reordered layout); "
                  f"unmodified reference parallel_materialize ({table} KernelTable), {threads} "
                  f"threads, median of {args.steps} steps; {REF_NOTE}")
        extra["reference_kernel_only_rows_per_s"] = kernel
    except Exception as e:  # noqa: BLE001
        value, kind = port, "port"
        sample = (f"{rows} rows per step of the C2 workload (D={d}, s={args.z}, int64 dim, "
                  f"reordered layout); parallel_materialize port (i64) over chunk_spans, "
                  f"{threads} threads")
        extra["reference_note"] = f"oracle/_ref unavailable: {e}"
    ms = 1e3 * rows / value
    line = {
        "impl": "reference", "metric": METRIC, "metric_note": METRIC_NOTE,
        "value": value, "unit": "rows/s", "n_gpus": args.gpus, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "int64", "data": "synthetic",
        "config": {"workload": "C2 large FK-join gather (BASELINE configs[1])", "domain": d,
                   "rows_per_step_sampled": rows, "z": args.z, "value": "int64",
                   "layout": "freq (skew-reordered)", "seed": SEED},
        "cpu_baseline": {"value": value, "unit": "rows/s", "cores": threads, "kind": kind,
                         "sample": sample},
        "e2e": {"value": value, "unit": "rows/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    line.update(extra)
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------
# GPU side
# ---------------------------------------------------------------------------
def timed_launches(fn, steps, warmup, stream, dist_on, ctx=None):
    """W warm-ups; then K steps bracketed by barrier + synchronize, one CUDA
    event per step on the launching stream.  Returns (total_ms, [per-step ms],
    libskx kernel launches inside the timed region)."""
    import torch
    import torch.distributed as dist
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    if dist_on:
        dist.barrier()
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
    l0 = ctx.launches() if ctx is not None else 0
    ev[0].record(stream)
    for i in range(steps):
        fn()
        ev[i + 1].record(stream)
    launches = (ctx.launches() - l0) if ctx is not None else 0
    torch.cuda.synchronize()
    if dist_on:
        dist.barrier()
    per = [ev[i].elapsed_time(ev[i + 1]) for i in range(steps)]
    return ev[0].elapsed_time(ev[steps]), per, launches


def reduce_to_root(t):
    """NCCL reduce to rank 0 (the BASELINE combine step).  The gloo backend,
    used only for the single-GPU multi-rank dry run (SKX_BENCH_DIST_BACKEND),
    all-reduces instead."""
    import torch.distributed as dist
    if dist.get_backend() == "nccl":
        dist.reduce(t, dst=0)
    else:
        dist.all_reduce(t)


def max_over_ranks(x, dist_on):
    import torch
    import torch.distributed as dist
    if not dist_on:
        return x
    t = torch.tensor([x], dtype=torch.float64, device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def run_ours(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_1910_10063_b200 import dataset as ds_mod
    from paper_1910_10063_b200 import skewdx as sx

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # SKX_BENCH_ONE_GPU=1 + SKX_BENCH_DIST_BACKEND=gloo: every rank on cuda:0, host-side
    # collectives -- a logic dry run of the multi-rank path on a one-GPU box (no kernel
    # waits on another rank's kernel).  Timings from it are not scaling numbers.
    if os.environ.get("SKX_BENCH_ONE_GPU") == "1":
        local = 0
    torch.cuda.set_device(local)
    dist_on = world > 1
    if dist_on:
        backend = os.environ.get("SKX_BENCH_DIST_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)
    ctx = sx.context(local)
    ctx.set_gather_policy(args.policy)
    peak, peak_kind = load_peaks()

    d = args.domain
    rows_local = args.rows  # weak scaling: fixed rows per GPU
    n_total = rows_local * world
    shard = ds_mod.Shard(rank, world, rank * rows_local, (rank + 1) * rows_local)
    t0 = time.perf_counter()
    data = ds_mod.make_gather_dataset(d, n_total, args.z, SEED, torch.int64, shard)
    setup_s = time.perf_counter() - t0
    stream = torch.cuda.current_stream()
    out = torch.empty(rows_local, dtype=torch.int64, device="cuda")

    def step_freq():
        sx.materialize(data.fact_freq, data.dim_freq, out=out, ctx=ctx, sync=False)

    sampler = ClockSampler(local)
    sampler.start()
    total_ms, per, launches = timed_launches(step_freq, args.steps, args.warmup, stream, dist_on,
                                             ctx)
    clocks = sampler.stop()
    ctx.sync()  # raises on a deferred domain violation
    total_ms = max_over_ranks(total_ms, dist_on)
    value = n_total * args.steps / (total_ms * 1e-3)
    alg_bytes = rows_local * (4 + 8)  # FK read + int64 output write per row
    avg_launch_s = statistics.mean(per) * 1e-3
    achieved = alg_bytes / avg_launch_s / 1e9
    out_freq = out.clone()

    extras = {}
    if not args.no_extras:
        # original (rand) layout through the same kernel, same timing rules
        outr = torch.empty_like(out)

        def step_rand():
            sx.materialize(data.fact_rand, data.dim_rand, out=outr, ctx=ctx, sync=False)
        tr, per_r, _ = timed_launches(step_rand, args.steps, args.warmup, stream, dist_on)
        tr = max_over_ranks(tr, dist_on)
        # CorrectnessError gate of bench.cpp:300-304: both layouts, same result
        same = bool(torch.equal(outr, out_freq))
        extras["rand_layout"] = {
            "value": n_total * args.steps / (tr * 1e-3), "unit": "rows/s",
            "roofline_frac": alg_bytes / (statistics.mean(per_r) * 1e-3) / 1e9 / peak,
            "freq_over_rand": (n_total * args.steps / (total_ms * 1e-3)) / (n_total * args.steps / (tr * 1e-3)),
            "outputs_equal": same}
        if not same:
            raise SystemExit("CorrectnessError: rand and freq layouts disagree")
        del outr
        # Index build on this workload, warm (scratch already allocated):
        # per-GPU u32 histogram -> NCCL all-reduce -> sort -> recode -> permute.
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
        hist_counts = torch.empty(d, dtype=torch.uint32, device="cuda")
        fact_tmp = torch.empty_like(data.fact_rand)
        ib = []
        for rep in range(3):
            if dist_on:
                dist.barrier()
            ev[0].record()
            sx.histogram_u32(data.fact_rand, d, hist_counts, ctx=ctx, sync=False)
            ev[1].record()
            ds_mod._allreduce_u32(hist_counts)
            idx2 = sx.build_index(sx.FrequencyProfile(hist_counts, n_total), ctx=ctx, sync=False)
            ev[2].record()
            sx.recode_fact(data.fact_rand, idx2, out=fact_tmp, ctx=ctx, sync=False)
            ev[3].record()
            sx.permute_dimension(data.dim_rand, idx2, ctx=ctx, sync=False)
            ev[4].record()
            torch.cuda.synchronize()
            ib.append([ev[i].elapsed_time(ev[i + 1]) for i in range(4)])
        ctx.sync()
        same_idx = bool(torch.equal(idx2.offsets, data.index.offsets)) and bool(
            torch.equal(fact_tmp, data.fact_freq))
        best = min(ib, key=sum)
        extras["index_build"] = {
            "histogram_ms": round(best[0], 3), "allreduce_sort_ms": round(best[1], 3),
            "recode_ms": round(best[2], 3), "permute_ms": round(best[3], 3),
            "total_ms": round(sum(best), 3), "deterministic": same_idx,
            "note": ("per-GPU u32 histogram, NCCL all-reduce (N>1), sort-by-count of D=%d, "
                     "recode of the local shard, permute of the int64 dim; warm, best of 3, "
                     "CUDA events" % d)}
        # Cache model (csrc/cachemodel.cu) on the empirical profile: predicted
        # dimension line misses of this gather vs the ncu-measured DRAM traffic.
        def model():
            vf = hist_counts.view(torch.int32).long()[idx2.offsets.view(torch.int32).long() - 1]
            vf = vf.double() / float(n_total)  # rank order
            geom = sx.CacheGeometry(1, 128, 8)
            eff = 64 << 20  # random-read capacity of the L2 (profiles/r1_experiments.md §10)
            res = {"geometry": "128 B lines of int64, L2 random-read capacity 64 MiB"}
            for name, lay in (("freq", sx.Layout.freq), ("rand", sx.Layout.rand)):
                lf = sx.line_frequencies(vf, lay, geom, SEED)
                h = sx.estimate_hit_rate(lf, eff // 128)
                res[name] = {"pred_l2_hit": h, "pred_line_misses": (1.0 - h) * rows_local}
            tr = ncu_traffic("gather_c2")
            if tr:
                res["freq"]["ncu_line_misses"] = (tr - rows_local * 12) / 128.0
            trr = ncu_traffic("gather_c2_rand")
            if trr:
                res["rand"]["ncu_line_misses"] = (trr - rows_local * 12) / 128.0
            return res
        if rank == 0:
            extras["cache_model"] = _cpu_extra(model)
        del hist_counts, fact_tmp, idx2

    # e2e through the C-ABI host-buffer entry (pinned host fact+dim in, out back)
    e2e = None
    if not args.no_e2e:
        import ctypes as C
        f_h = data.fact_freq.cpu().pin_memory()
        d_h = data.dim_freq.cpu().pin_memory()
        o_h = torch.empty(rows_local, dtype=torch.int64).pin_memory()
        lib = ctx.lib

        def e2e_step():
            ctx.check(lib.skx_materialize_host(ctx.handle, 8, C.c_void_p(f_h.data_ptr()), rows_local,
                                               C.c_void_p(d_h.data_ptr()), d,
                                               C.c_void_p(o_h.data_ptr())))
        e2e_step()
        e_steps = max(1, min(args.steps, 3))
        if dist_on:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(e_steps):
            e2e_step()
        te = max_over_ranks(time.perf_counter() - t0, dist_on)
        if not torch.equal(o_h[:1 << 20].cuda(), out_freq[:1 << 20]):
            raise SystemExit("CorrectnessError: host-buffer path disagrees with device path")
        e2e = {"value": n_total * e_steps / te, "unit": "rows/s",
               "h2d_bytes_per_step": rows_local * 4 + d * 8, "d2h_bytes_per_step": rows_local * 8,
               "path": "skx_materialize_host (pinned host fact+dim -> device -> pinned host out, "
                       "chunked 2-stream pipeline)"}
        del f_h, d_h, o_h

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        m = min(CPU_SAMPLE_ROWS, rows_local)
        cpu = cpu_gather_baseline(data.fact_freq[:m].cpu().numpy(),
                                  data.dim_freq.cpu().numpy().view(np.uint64))

    if not args.no_extras:
        # The rest of the BASELINE C2 sweep (s = 0.5 and 1.5; s = 1.0 is the headline),
        # both layouts, same kernel and timing rules.
        sweep = {}
        for zz in (0.5, 1.5):
            g = ds_mod.make_gather_dataset(d, n_total, zz, SEED, torch.int64, shard)
            for lay, f, dm in (("freq", g.fact_freq, g.dim_freq), ("rand", g.fact_rand, g.dim_rand)):
                ts, per_s, _ = timed_launches(
                    lambda f=f, dm=dm: sx.materialize(f, dm, out=out, ctx=ctx, sync=False),
                    max(3, min(args.steps, 10)), args.warmup, stream, dist_on)
                ts = max_over_ranks(ts, dist_on)
                ms = ts / max(3, min(args.steps, 10))
                sweep[f"s{zz}_{lay}"] = {"ms_per_step": ms,
                                         "value": n_total / (ms * 1e-3), "unit": "rows/s",
                                         "roofline_frac": alg_bytes / (statistics.mean(per_s) * 1e-3)
                                         / 1e9 / peak}
            del g
            torch.cuda.empty_cache()
        extras["c2_s_sweep"] = sweep

    groupby = None
    if not args.no_extras:
        del data, out, out_freq
        torch.cuda.empty_cache()
        gdat = ds_mod.make_groupby_dataset(D_C3, rows_local * world, 1.0, SEED + 1,
                                           ds_mod.Shard(rank, world, rank * rows_local,
                                                        (rank + 1) * rows_local))
        counts = torch.empty(D_C3, dtype=torch.uint64, device="cuda")
        sums = torch.empty(D_C3, dtype=torch.uint64, device="cuda")

        def step_gb():
            ctx.call("skx_aggregate", C_ptr(gdat.fact_freq), C_ptr(gdat.qty), 8, rows_local, D_C3, 0,
                     C_ptr(counts), C_ptr(sums), ctx.stream(), sync=False)
            if dist_on:  # per-GPU partials combined with NCCL reduce (BASELINE config 3)
                reduce_to_root(counts.view(torch.int64))
                reduce_to_root(sums.view(torch.int64))
        tg, per_g, _ = timed_launches(step_gb, args.steps, args.warmup, stream, dist_on)
        ctx.sync()
        tg = max_over_ranks(tg, dist_on)
        gb_bytes = rows_local * 12 + D_C3 * 16
        groupby = {"workload": "C3 group-by COUNT+SUM(int64 qty), D=2^24, s=1.0, reordered",
                   "value": rows_local * world * args.steps / (tg * 1e-3), "unit": "rows/s",
                   "ms_per_step": tg / args.steps,
                   "roofline": {"bound": "hbm", "achieved": gb_bytes / (statistics.mean(per_g) * 1e-3) / 1e9,
                                "peak": peak, "unit": "GB/s",
                                "frac": gb_bytes / (statistics.mean(per_g) * 1e-3) / 1e9 / peak,
                                "traffic": ncu_traffic("groupby_c3"),
                                "alg_bytes_per_step": gb_bytes}}
        # Q3a heavy hitters: counts of the k = 8192 hottest ids of
        # the recoded C3 column -- the device part of heavy_hitter_count
        # (operators.cpp:184-203); the top-k ordering of k pairs is host work.
        hh = torch.empty(8192, dtype=torch.uint64, device="cuda")

        def step_hh():
            ctx.call("skx_heavy_hitter_count", C_ptr(gdat.fact_freq), rows_local, D_C3, 8192,
                     C_ptr(hh), ctx.stream(), sync=False)
            if dist_on:
                reduce_to_root(hh.view(torch.int64))
        th, per_h, _ = timed_launches(step_hh, args.steps, args.warmup, stream, dist_on)
        ctx.sync()
        th = max_over_ranks(th, dist_on)
        hb = rows_local * 4 + 8192 * 8
        groupby["heavy_hitters_k8192"] = {
            "value": rows_local * world * args.steps / (th * 1e-3), "unit": "rows/s",
            "ms_per_step": th / args.steps,
            "roofline_frac": hb / (statistics.mean(per_h) * 1e-3) / 1e9 / peak}
        del hh
        if rank == 0 and world == 1 and not args.no_cpu:
            groupby["cpu_reference"] = _cpu_extra(lambda: cpu_groupby_reference(
                gdat.fact_freq[:1 << 26].cpu().numpy(), gdat.qty[:1 << 24].cpu().numpy(), D_C3))
        del gdat, counts, sums
        torch.cuda.empty_cache()
        extras.update(other_configs(args, ctx, stream, dist_on, rank, world, peak))

    if rank == 0:
        line = {
            "metric": METRIC, "metric_note": METRIC_NOTE,
            "value": value, "unit": "rows/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": total_ms / args.steps, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "int64", "data": "synthetic",
            "config": {"workload": "C2 large FK-join gather (BASELINE configs[1])", "domain": d,
                       "rows_per_gpu": rows_local, "rows_total": n_total, "z": args.z,
                       "value": "int64", "layout": "freq (skew-reordered)", "seed": SEED,
                       "parallelism": f"dp{world} (fact rows sharded, dimension replicated)",
                       "l2": "inputs larger than L2 (4 GiB FK + 8 GiB output + 1 GiB dim per step)",
                       "gather_policy": args.policy},
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "peak_kind": peak_kind,
                         "frac_vs_nominal_8000": achieved / 8000.0,
                         "traffic": ncu_traffic("gather_c2"),
                         # DRAM bytes actually moved per launch (ncu) over the live launch time:
                         # how close the kernel runs to the HBM peak with its real traffic
                         "traffic_GBps": (ncu_traffic("gather_c2") or 0) / statistics.mean(per) / 1e6,
                         "alg_bytes_per_launch": alg_bytes,
                         "avg_launch_ms": statistics.mean(per)},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": int(launches),
            "clocks": clocks,
            "setup_s": round(setup_s, 2),
        }
        line.update(extras)
        if groupby:
            line["groupby_c3"] = groupby
        print(json.dumps(line), flush=True)
    if dist_on:
        dist.barrier()
        dist.destroy_process_group()


def other_configs(args, ctx, stream, dist_on, rank, world, peak):
    """The remaining BASELINE configs, each timed like the headline (W
    warm-ups, K launches between barriers, CUDA events, max over ranks):
    C1 small gather (both layouts), C4 index build at scale, C5 select +
    4-column gather + per-category fp64 SUM."""
    import numpy as np
    import torch

    from paper_1910_10063_b200 import dataset as ds_mod
    from paper_1910_10063_b200 import skewdx as sx
    out = {}
    k = max(3, min(args.steps, 10))

    # C1: D=2^22 int32 price (uniform 1..1e6), 2^24 int32 FKs per GPU, s=1.0.
    d1, n1 = 1 << 22, 1 << 24
    g = ds_mod.make_gather_dataset(d1, n1 * world, 1.0, SEED + 7, torch.int32,
                                   ds_mod.Shard(rank, world, rank * n1, (rank + 1) * n1))
    price = ds_mod.fill_column(ds_mod.KIND_UNIFORM, torch.int32, d1, SEED + 8, 1, 1000000)
    price_f = sx.permute_dimension(price, g.index, sync=False)
    o1 = torch.empty(n1, dtype=torch.int32, device="cuda")
    c1 = {}
    for layout, f, dm in (("freq", g.fact_freq, price_f), ("rand", g.fact_rand, price)):
        t, per, _ = timed_launches(lambda f=f, dm=dm: sx.materialize(f, dm, out=o1, ctx=ctx, sync=False),
                                   k * 10, args.warmup, stream, dist_on)
        t = max_over_ranks(t, dist_on)
        c1[layout] = {"value": n1 * world * k * 10 / (t * 1e-3), "unit": "rows/s",
                      "us_per_launch": 1e3 * t / (k * 10),
                      "roofline_frac": n1 * 8 / (statistics.mean(per) * 1e-3) / 1e9 / peak}
    c1["note"] = ("L2-resident 16 MiB dimension; back-to-back launches (inputs 192 MiB > L2), "
                  "per-launch time includes launch overhead")
    out["gather_c1"] = c1
    del g, price, price_f, o1

    # C4: index build at scale, D=2^26, s=1.25, 2^30 rows per GPU.
    d4, n4 = 1 << 26, 1 << 30
    sh = ds_mod.Shard(rank, world, rank * n4, (rank + 1) * n4)
    fact = ds_mod.make_rand_fact(d4, n4 * world, 1.25, SEED + 9, sh)
    dim_i = ds_mod.fill_column(ds_mod.KIND_RAW, torch.int32, d4, SEED + 10)
    dim_f = ds_mod.fill_column(ds_mod.KIND_RAW, torch.int32, d4, SEED + 11).view(torch.float32)
    counts = torch.empty(d4, dtype=torch.uint32, device="cuda")
    ff = torch.empty_like(fact)

    def c4_step():
        sx.histogram_u32(fact, d4, counts, ctx=ctx, sync=False)
        ds_mod._allreduce_u32(counts)
        idx = sx.build_index(sx.FrequencyProfile(counts, n4 * world), ctx=ctx, sync=False)
        sx.recode_fact(fact, idx, out=ff, ctx=ctx, sync=False)
        sx.permute_dimension(dim_i, idx, ctx=ctx, sync=False)
        sx.permute_dimension(dim_f, idx, ctx=ctx, sync=False)
    t4, _, _ = timed_launches(c4_step, 3, 1, stream, dist_on)
    ctx.sync()
    t4 = max_over_ranks(t4, dist_on) / 3
    alg4 = n4 * 12 + d4 * 28
    out["index_build_c4"] = {"ms_per_build": t4, "rows_per_s": n4 * world / (t4 * 1e-3),
                             "roofline_frac": alg4 / (t4 * 1e-3) / 1e9 / peak,
                             "alg_bytes": alg4,
                             "note": "histogram + all-reduce + sort + recode + permute int32 and "
                                     "float32 dims; warm"}
    del fact, dim_i, dim_f, counts, ff
    torch.cuda.empty_cache()
    if rank == 0 and world == 1 and not args.no_cpu:
        small = ds_mod.make_rand_fact(1 << 22, 1 << 24, 1.25, SEED + 9, ds_mod.shard_of(1 << 24))
        out["index_build_c4"]["cpu_reference"] = _cpu_extra(
            lambda: cpu_rebuild_reference(small.cpu().numpy(), 1 << 22))
        del small

    # C5: 2^31 rows (per GPU), D=2^25, category < 100, 4-column gather + fp64 SUM(price).
    d5, n5 = 1 << 25, 1 << 31
    sh = ds_mod.Shard(rank, world, rank * n5, (rank + 1) * n5)
    fact = ds_mod.make_rand_fact(d5, n5 * world, 1.0, SEED + 12, sh)
    counts = sx.histogram_u32(fact, d5, ctx=ctx, sync=False)
    ds_mod._allreduce_u32(counts)
    idx = sx.build_index(sx.FrequencyProfile(counts, n5 * world), ctx=ctx, sync=False)
    fact_f = sx.recode_fact(fact, idx, ctx=ctx, sync=False)
    del fact, counts
    cat = sx.permute_dimension(ds_mod.fill_column(ds_mod.KIND_UNIFORM, torch.int32, d5, SEED + 13, 0, 1000), idx)
    prc = sx.permute_dimension(ds_mod.fill_column(ds_mod.KIND_LOGNORMAL, torch.float32, d5, SEED + 14, 3.0, 1.0), idx)
    sup = sx.permute_dimension(ds_mod.fill_column(ds_mod.KIND_RAW, torch.int64, d5, SEED + 15), idx)
    flg = sx.permute_dimension(ds_mod.fill_column(ds_mod.KIND_RAW, torch.int16, d5, SEED + 16), idx)
    bm = sx.build_bitmap_lt(cat, 100)  # category < 100, already in rank space
    cap = n5 // 5
    bufs = [torch.empty(cap, dtype=t, device="cuda")
            for t in (torch.uint32, torch.int32, torch.float32, torch.int64, torch.int16)]
    sums = torch.empty(1000, dtype=torch.float64, device="cuda")
    cnt = torch.zeros(1, dtype=torch.uint64, device="cuda")

    def c5_step():
        ctx.call("skx_select_gather_sum", C_ptr(fact_f), n5, C_ptr(bm.words), d5, C_ptr(cat),
                 # base 0: shard-local offsets (global ones exceed the reference's u32
                 # row offsets, operators.cpp:88-90, once 2^31 rows per GPU x N > 2^32)
                 C_ptr(prc), C_ptr(sup), C_ptr(flg), 0, 1000, cap, *[C_ptr(b) for b in bufs],
                 C_ptr(sums), C_ptr(cnt), ctx.stream(), sync=False)
        if dist_on:  # per-category fp64 partials reduced to rank 0
            reduce_to_root(sums)
    t5, per5, _ = timed_launches(c5_step, k, args.warmup, stream, dist_on)
    ctx.sync()
    t5 = max_over_ranks(t5, dist_on)
    sel = int(cnt.item())
    if sel > cap:
        raise SystemExit("C5 output capacity exceeded")
    alg5 = n5 * 4 + sel * 22 + 1000 * 8
    out["select_c5"] = {"value": n5 * world * k / (t5 * 1e-3), "unit": "rows/s",
                        "ms_per_step": t5 / k, "selected": sel, "selectivity": sel / n5,
                        "roofline_frac": alg5 / (statistics.mean(per5) * 1e-3) / 1e9 / peak,
                        "alg_bytes_per_step": alg5}
    if rank == 0 and world == 1 and not args.no_cpu:
        out["select_c5"]["cpu_reference"] = _cpu_extra(lambda: cpu_select_reference(
            fact_f[:1 << 26].cpu().numpy(), bm.words.view(torch.int64).cpu().numpy().view(np.uint64),
            d5))
    del fact_f, cat, prc, sup, flg, bm, bufs, sums, cnt, idx
    torch.cuda.empty_cache()
    return out


def C_ptr(t):
    import ctypes as C
    return C.c_void_p(t.data_ptr())


def main():
    args = parse()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference_arm(args)
    else:
        run_ours(args)


if __name__ == "__main__":
    main()

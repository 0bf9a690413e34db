"""World-size-2 tests of the multi-GPU host logic (paper_1910_10063_b200/dist.py)
over gloo on CPU, with the oracle as the per-shard executor: the sharded
results after the collectives must equal the single-process oracle on the
whole column (the same contract the NCCL path has on B200s)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from oracle.oracle import Oracle


class OracleExecutor:
    """CPU stand-in for GpuExecutor (TEST ONLY): same tensor contract."""

    def __init__(self):
        self.o = Oracle()

    def histogram_u32(self, fact, d):
        c = self.o.count_frequencies(fact.numpy(), d)
        return torch.from_numpy(c.astype(np.uint32))

    def build_index(self, counts_u32, total):
        off, rk = self.o.build_index(counts_u32.numpy().astype(np.uint64), total)
        return (torch.from_numpy(off), torch.from_numpy(rk))

    def recode(self, fact, index):
        return torch.from_numpy(self.o.recode_fact(fact.numpy(), index[1].numpy()))

    def gather(self, fact, dim):
        return torch.from_numpy(self.o.gather(fact.numpy(), dim.numpy()))

    def aggregate(self, fact, measure, d):
        c, s = self.o.aggregate_count_sum(fact.numpy(), measure.numpy().view(np.uint64), d)
        return torch.from_numpy(c), torch.from_numpy(s)

    def select(self, fact, bitmap, base):
        words, bits = bitmap
        return torch.from_numpy(self.o.select_offsets(fact.numpy(), words, bits, base))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, d, n, out_dir):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_1910_10063_b200 import dist as sdist
    o = Oracle()
    ex = OracleExecutor()
    cdf = o.zipf_cdf(d, 1.1)
    r2i = o.random_bijection(d, 5)
    shard = sdist.shard_for(n)
    fact = torch.from_numpy(o.generate_zipf_counter(cdf, r2i, 5, shard.begin, shard.rows))
    # index build: local histogram + all-reduce + identical sort
    off, rk = sdist.rebuild(fact, d, n, ex)
    rec = ex.recode(fact, (off, rk))
    # group-by on the recoded shard, reduced to rank 0
    meas = torch.from_numpy((np.arange(shard.begin, shard.end, dtype=np.int64) % 97) + 1)
    counts, sums = sdist.aggregate(rec, meas, d, ex)
    # selection: per-shard offsets with base, gathered in rank order
    words = np.zeros((d + 63) // 64, np.uint64)
    words[::3] = np.uint64(0x5555555555555555)
    sel = sdist.select(fact, (words, d), shard, ex)
    if rank == 0:
        np.savez(os.path.join(out_dir, "r0.npz"), off=off.numpy(), rk=rk.numpy(),
                 counts=counts.numpy(), sums=sums.numpy(), sel=sel.numpy(), words=words)
    np.save(os.path.join(out_dir, f"rec{rank}.npy"), rec.numpy())
    dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_sharded_path_equals_whole_column(tmp_path, world):
    d, n = 3001, 200003
    mp.spawn(_worker, args=(world, _free_port(), d, n, str(tmp_path)), nprocs=world, join=True)
    o = Oracle()
    cdf = o.zipf_cdf(d, 1.1)
    fact = o.generate_zipf_counter(cdf, o.random_bijection(d, 5), 5, 0, n)
    off, rk = o.rebuild(fact, d)
    r0 = np.load(tmp_path / "r0.npz")
    assert np.array_equal(r0["off"], off) and np.array_equal(r0["rk"], rk)
    rec = np.concatenate([np.load(tmp_path / f"rec{r}.npy") for r in range(world)])
    assert np.array_equal(rec, o.recode_fact(fact, rk))
    meas = (np.arange(n, dtype=np.int64) % 97) + 1
    c, s = o.aggregate_count_sum(rec, meas.view(np.uint64), d)
    assert np.array_equal(r0["counts"], c) and np.array_equal(r0["sums"], s)
    assert np.array_equal(r0["sel"].astype(np.uint32), o.select_offsets(fact, r0["words"], d))


def test_shard_for_matches_chunk_spans():
    from paper_1910_10063_b200 import dist as sdist
    o = Oracle()
    for n, w in [(0, 2), (7, 3), (1 << 20, 8), (1000003, 4)]:
        spans = o.chunk_spans(n, w)
        for r in range(w):
            s = sdist.shard_for(n, r, w)
            assert (s.begin, s.end) == spans[r]

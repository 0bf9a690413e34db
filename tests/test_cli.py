"""The index build/apply CLI (skewdx_b200_cli; reference tools/benchcli
main.cpp:101-134, generate.cpp:52-80): usage and data errors on the host
(CPU tests), and on the GPU the streamed index build/apply against the
oracle, byte for byte on the SKPI/SKDX files, across chunk edges."""
import os
import struct
import subprocess

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CLI = os.path.join(ROOT, "paper_1910_10063_b200", "skewdx_b200_cli")


@pytest.fixture(scope="module")
def cli():
    from paper_1910_10063_b200 import build
    build.build_all()
    return CLI


def run(cli, *args, env=None):
    e = dict(os.environ)
    e.update(env or {})
    r = subprocess.run([cli, *map(str, args)], capture_output=True, text=True, env=e, timeout=600)
    return r.returncode, r.stderr


def write_skdx(path, values):
    v = np.asarray(values, np.uint32)
    with open(path, "wb") as f:
        f.write(b"SKDX" + struct.pack("<IQ", 1, v.size) + v.tobytes())


def skpi_bytes(offsets, ranks):
    o, r = np.asarray(offsets, np.uint32), np.asarray(ranks, np.uint32)
    return b"SKPI" + struct.pack("<IQ", 1, o.size) + o.tobytes() + r.tobytes()


def read_skdx(path):
    b = open(path, "rb").read()
    assert b[:4] == b"SKDX" and struct.unpack("<IQ", b[4:16])[0] == 1
    n = struct.unpack("<IQ", b[4:16])[1]
    v = np.frombuffer(b[16:], np.uint32)
    assert v.size == n
    return v


# ---- host-side behaviour (no GPU needed) ------------------------------------

def test_cli_usage_errors(cli, tmp_path):
    assert run(cli)[0] == 1
    assert run(cli, "index")[0] == 1
    assert run(cli, "index", "frobnicate")[0] == 1
    rc, err = run(cli, "index", "build", "--out", tmp_path / "o.skpi")
    assert rc == 1 and "--fact is required" in err
    rc, err = run(cli, "index", "build", "--fact", tmp_path / "f", "--d", "x1", "--out", tmp_path / "o")
    assert rc == 1 and "--d" in err
    rc, err = run(cli, "index", "apply", "--fact", "a")
    assert rc == 1 and "--index is required" in err


def test_cli_data_errors(cli, tmp_path):
    rc, err = run(cli, "index", "apply", "--index", tmp_path / "missing.skpi", "--fact", "a",
                  "--fact-out", "b")
    assert rc == 2 and "cannot open for reading" in err
    idx = tmp_path / "i.skpi"
    idx.write_bytes(skpi_bytes([2, 1, 3], [2, 1, 3]))
    rc, err = run(cli, "index", "apply", "--index", idx, "--fact", "a")
    assert rc == 1 and "must be paired" in err  # InvalidArgument -> usage exit code
    rc, err = run(cli, "index", "apply", "--index", idx)
    assert rc == 1 and "nothing to do" in err
    bad = tmp_path / "bad.skpi"
    bad.write_bytes(skpi_bytes([1, 1, 3], [1, 2, 3]))
    rc, err = run(cli, "index", "apply", "--index", bad, "--dim", "a", "--dim-out", "b")
    assert rc == 2 and "not inverse bijections" in err
    magic = tmp_path / "m.skdx"
    magic.write_bytes(b"XXXX" + struct.pack("<IQ", 1, 0))
    rc, err = run(cli, "index", "build", "--fact", magic, "--out", tmp_path / "o.skpi")
    assert rc == 2 and "bad magic" in err
    short = tmp_path / "s.skdx"
    short.write_bytes(b"SKDX" + struct.pack("<IQ", 1, 5) + b"\0" * 8)
    rc, err = run(cli, "index", "build", "--fact", short, "--out", tmp_path / "o.skpi")
    assert rc == 2 and "length mismatch" in err
    empty = tmp_path / "e.skdx"
    write_skdx(empty, [])
    rc, err = run(cli, "index", "build", "--fact", empty, "--out", tmp_path / "o.skpi")
    assert rc == 2 and "fact column is empty" in err


# ---- the streamed GPU path ---------------------------------------------------

def _fact(oracle, d, n, z, seed):
    cdf = oracle.zipf_cdf(d, z)
    r2i = oracle.random_bijection(d, seed)
    return oracle.generate_zipf_counter(cdf, r2i, seed, 0, n)


@pytest.mark.gpu
@pytest.mark.parametrize("chunk", [100003, 1 << 24])
def test_cli_build_apply_vs_oracle(cli, oracle, tmp_path, chunk):
    d, n = 50000, (1 << 20) + 7
    fact = _fact(oracle, d, n, 1.0, 3)
    dim = np.random.default_rng(1).integers(0, 2**32, size=d, dtype=np.uint64).astype(np.uint32)
    write_skdx(tmp_path / "f.skdx", fact)
    write_skdx(tmp_path / "dim.skdx", dim)
    env = {"SKX_STREAM_CHUNK_ROWS": str(chunk)}
    rc, err = run(cli, "index", "build", "--fact", tmp_path / "f.skdx", "--d", d, "--out",
                  tmp_path / "i.skpi", env=env)
    assert rc == 0, err
    assert f"index build: domain {d} -> " in err
    off, rk = oracle.build_index(oracle.count_frequencies(fact, d), n)
    assert (tmp_path / "i.skpi").read_bytes() == skpi_bytes(off, rk)
    rc, err = run(cli, "index", "apply", "--index", tmp_path / "i.skpi", "--fact", tmp_path / "f.skdx",
                  "--fact-out", tmp_path / "r.skdx", "--dim", tmp_path / "dim.skdx", "--dim-out",
                  tmp_path / "p.skdx", env=env)
    assert rc == 0, err
    assert "index apply: recoded" in err and "index apply: permuted" in err
    assert np.array_equal(read_skdx(tmp_path / "r.skdx"), oracle.recode_fact(fact, rk))
    assert np.array_equal(read_skdx(tmp_path / "p.skdx"), oracle.permute_dimension(dim, off))


@pytest.mark.gpu
def test_cli_domain_default_and_violations(cli, oracle, tmp_path):
    d, n = 7000, 300001
    fact = _fact(oracle, d, n, 1.25, 9)
    fact[fact == fact.max()] = d  # the largest identifier sets D when --d is omitted
    write_skdx(tmp_path / "f.skdx", fact)
    env = {"SKX_STREAM_CHUNK_ROWS": "65536"}
    rc, err = run(cli, "index", "build", "--fact", tmp_path / "f.skdx", "--out", tmp_path / "i.skpi",
                  env=env)
    assert rc == 0 and f"domain {d} -> " in err, err
    off, rk = oracle.build_index(oracle.count_frequencies(fact, d), n)
    assert (tmp_path / "i.skpi").read_bytes() == skpi_bytes(off, rk)
    # first offending row (third chunk), reported like DomainViolation::what()
    bad = fact.copy()
    bad[200000] = d + 5
    bad[250000] = 0
    write_skdx(tmp_path / "b.skdx", bad)
    rc, err = run(cli, "index", "build", "--fact", tmp_path / "b.skdx", "--d", d, "--out",
                  tmp_path / "j.skpi", env=env)
    assert rc == 2 and f"domain violation at row 200000: value {d + 5} outside 1..{d}" in err, err
    rc, err = run(cli, "index", "apply", "--index", tmp_path / "i.skpi", "--fact", tmp_path / "b.skdx",
                  "--fact-out", tmp_path / "r.skdx", env=env)
    assert rc == 2 and "domain violation at row 200000" in err, err
    assert not (tmp_path / "r.skdx").exists()  # nothing written, as in the reference
    # in place: a failed apply leaves the input column untouched, and no temporary behind
    before = (tmp_path / "b.skdx").read_bytes()
    rc, err = run(cli, "index", "apply", "--index", tmp_path / "i.skpi", "--fact", tmp_path / "b.skdx",
                  "--fact-out", tmp_path / "b.skdx", env=env)
    assert rc == 2 and "domain violation at row 200000" in err, err
    assert (tmp_path / "b.skdx").read_bytes() == before
    assert not [p for p in os.listdir(tmp_path) if ".tmp." in p]


@pytest.mark.gpu
@pytest.mark.parametrize("chunk", [65536, 1 << 24])
def test_cli_apply_in_place(cli, oracle, tmp_path, chunk):
    """--fact-out == --fact: the reference reads the whole column before it
    writes (write_column(out, recode_fact(read_column(in)))), so the column is
    recoded in place; the streamed apply must not truncate its own input."""
    d, n = 9000, 400003
    fact = _fact(oracle, d, n, 1.0, 5)
    write_skdx(tmp_path / "f.skdx", fact)
    env = {"SKX_STREAM_CHUNK_ROWS": str(chunk)}
    rc, err = run(cli, "index", "build", "--fact", tmp_path / "f.skdx", "--d", d, "--out",
                  tmp_path / "i.skpi", env=env)
    assert rc == 0, err
    rc, err = run(cli, "index", "apply", "--index", tmp_path / "i.skpi", "--fact", tmp_path / "f.skdx",
                  "--fact-out", tmp_path / "f.skdx", env=env)
    assert rc == 0, err
    _, rk = oracle.build_index(oracle.count_frequencies(fact, d), n)
    assert np.array_equal(read_skdx(tmp_path / "f.skdx"), oracle.recode_fact(fact, rk))
    assert not [p for p in os.listdir(tmp_path) if ".tmp." in p]


@pytest.mark.gpu
def test_pinned_async_entry_points():
    """The streamed callers' C-ABI entries: pinned buffers, the context's two
    host streams, asynchronous copies both ways, a histogram on a host stream
    with a deferred domain violation reported by skx_sync on that stream."""
    import ctypes as C

    import torch

    from paper_1910_10063_b200 import DomainViolation
    from paper_1910_10063_b200 import skewdx as sx
    ctx = sx.context(0)
    lib, h = ctx.lib, ctx.handle
    n = 1 << 20
    pin = C.c_void_p()
    ctx.check(lib.skx_pinned_alloc(h, n * 4, C.byref(pin)))
    try:
        host = np.ctypeslib.as_array(C.cast(pin, C.POINTER(C.c_uint32)), shape=(n,))
        host[:] = np.arange(1, n + 1, dtype=np.uint32) % 1000 + 1
        dev = torch.empty(n, dtype=torch.int32, device="cuda")
        for slot in (0, 1):
            st = lib.skx_ctx_stream(h, slot)
            assert st
            ctx.check(lib.skx_copy_to_device_async(h, C.c_void_p(dev.data_ptr()), pin, n * 4, C.c_void_p(st)))
            counts = torch.zeros(1000, dtype=torch.int32, device="cuda")
            ctx.check(lib.skx_histogram_u32(h, C.c_void_p(dev.data_ptr()), n, 1000,
                                            C.c_void_p(counts.data_ptr()), 0, C.c_void_p(st)))
            ctx.check(lib.skx_sync(h, C.c_void_p(st)))
            exp = np.bincount(host.astype(np.int64) - 1, minlength=1000)
            assert np.array_equal(counts.cpu().numpy().astype(np.int64), exp)
            host2 = np.zeros(n, np.uint32)
            ctx.check(lib.skx_copy_to_host_async(h, host2.ctypes.data_as(C.c_void_p),
                                                 C.c_void_p(dev.data_ptr()), n * 4, C.c_void_p(st)))
            ctx.check(lib.skx_sync(h, C.c_void_p(st)))
            assert np.array_equal(host2, host)
        host[777] = 5000  # out of 1..1000
        st = lib.skx_ctx_stream(h, 1)
        ctx.check(lib.skx_copy_to_device_async(h, C.c_void_p(dev.data_ptr()), pin, n * 4, C.c_void_p(st)))
        ctx.check(lib.skx_histogram_u32(h, C.c_void_p(dev.data_ptr()), n, 1000,
                                        C.c_void_p(counts.data_ptr()), 1, C.c_void_p(st)))
        with pytest.raises(DomainViolation) as e:
            ctx.sync(C.c_void_p(st))
        assert e.value.row() == 777 and e.value.value() == 5000
        assert lib.skx_ctx_stream(h, 2) is None
    finally:
        ctx.check(lib.skx_pinned_free(h, pin))

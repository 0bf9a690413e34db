"""The reference's OWN test files for the path (proj/tests/test_permindex.cpp,
test_operators.cpp, test_parallel.cpp, test_cachemodel.cpp, test_columns.cpp), compiled
unmodified by oracle/Makefile
against the B200 drop-in (paper_1910_10063_b200/cpp/include + libskewdx_b200.so,
every hot-path call on the GPU) and a minimal doctest-compatible shim.  They
must pass on a B200 exactly as they pass against the reference library."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
REF = os.path.join(ROOT, "oracle", "_ref")
SUITES = ["test_permindex", "test_operators", "test_parallel", "test_cachemodel", "test_columns"]

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("suite", SUITES)
def test_reference_suite_passes_on_b200(suite):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    exe = os.path.join(REF, f"refsuite_{suite}")
    if not os.path.exists(exe):
        pytest.skip(f"{exe} not built (make -C oracle refsuite needs /root/reference)")
    r = subprocess.run([exe], capture_output=True, text=True, timeout=600)
    print(r.stdout[-2000:], r.stderr[-4000:])
    assert r.returncode == 0, r.stderr[-4000:]
    assert "0 failed" in r.stdout

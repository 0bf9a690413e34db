import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (runs the CUDA parity tests)")


@pytest.fixture(scope="session")
def oracle():
    from oracle.oracle import Oracle
    return Oracle()


@pytest.fixture(scope="session")
def reference():
    from oracle.oracle import REF_SO, Reference
    if not os.path.exists(REF_SO) and not os.path.isdir("/root/reference/proj/src"):
        pytest.skip("reference library not built here")
    return Reference()


@pytest.fixture(scope="session")
def kat():
    with open(os.path.join(GOLDEN, "kat.json")) as f:
        return json.load(f)


class RefCases:
    def __init__(self, path):
        self.z = np.load(path)
        self.meta = json.loads(bytes(self.z["meta"]).decode())

    def __len__(self):
        return len(self.meta)

    def case(self, i):
        p = f"c{i}_"
        out = {k[len(p):]: self.z[k] for k in self.z.files if k.startswith(p)}
        out.update(self.meta[i])
        return out


@pytest.fixture(scope="session")
def ref_cases():
    return RefCases(os.path.join(GOLDEN, "ref_cases.npz"))


def words_from_bits(bits, d):
    w = np.zeros((d + 63) // 64, np.uint64)
    for i in bits:
        w[i >> 6] |= np.uint64(1) << np.uint64(i & 63)
    return w

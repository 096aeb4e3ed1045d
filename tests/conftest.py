import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

GOLDEN = os.path.join(ROOT, "tests", "golden")
REFERENCE_SRC = "/root/reference/pkg/src"


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")


def has_gpu() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


class GoldenSet:
    """Cases of one fixture file (see tests/golden/make_golden.py)."""

    def __init__(self, name):
        self.data = dict(np.load(os.path.join(GOLDEN, name)))
        self.count = self.data["n__ptr"].size - 1

    def case(self, i):
        out = {}
        for k, v in self.data.items():
            if k.endswith("__ptr"):
                continue
            p = self.data[k + "__ptr"]
            out[k] = v[p[i]:p[i + 1]]
        out["n"] = int(out["n"][0])
        if not int(out.pop("weighted")[0]):
            out["w"] = out["w2"] = out["w2_raw"] = out["w_sd"] = None
        return out

    def __iter__(self):
        for i in range(self.count):
            yield self.case(i)


def load_golden(name):
    return GoldenSet(name)


@pytest.fixture(scope="session")
def kat():
    return load_golden("kat.npz")


@pytest.fixture(scope="session")
def fuzz():
    return load_golden("fuzz.npz")


@pytest.fixture(scope="session")
def medium():
    return load_golden("medium.npz")

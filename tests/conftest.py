"""Test configuration.

Markers: ``gpu`` tests need a CUDA device (the driver runs them with -m gpu on a B200);
everything else runs on a CPU-only host.  The oracle (oracle/segrange_port.py) is the
checker: tests may import it, the package never does.
"""

import json
import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

GOLDEN_DIR = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA GPU (B200); run with -m gpu")
    config.addinivalue_line("markers", "slow: large-size GPU test")


def cuda_available() -> bool:
    try:
        import torch

        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if cuda_available():
        return
    skip = pytest.mark.skip(reason="no CUDA device on this host")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


class Golden:
    def __init__(self):
        with open(os.path.join(GOLDEN_DIR, "golden.json")) as fh:
            self.meta = json.load(fh)
        self.arrays = np.load(os.path.join(GOLDEN_DIR, "golden.npz"))
        self.cases = self.meta["cases"]

    def select(self, **kw):
        out = []
        for c in self.cases:
            if all(c.get(k) == v for k, v in kw.items()):
                out.append(c)
        return out


def dec(v):
    if v is None:
        return None
    if "f" in v:
        return float.fromhex(v["f"])
    if "i" in v:
        return int(v["i"])
    return v["b"]


_GOLDEN = None


def golden() -> Golden:
    global _GOLDEN
    if _GOLDEN is None:
        _GOLDEN = Golden()
    return _GOLDEN


@pytest.fixture(scope="session")
def gold():
    return golden()


@pytest.fixture(scope="session")
def rt_pool():
    """Device runtimes keyed by locale count (all locales share the visible GPUs)."""
    import paper_2406_00158_b200 as sr

    pool = {}

    def get(p):
        if p not in pool:
            pool[p] = sr.Runtime(p)
        return pool[p]

    yield get
    for rt in pool.values():
        rt.close()


@pytest.fixture
def rt3(rt_pool):
    return rt_pool(3)


@pytest.fixture
def rt4(rt_pool):
    return rt_pool(4)


@pytest.fixture(scope="session")
def meta_rt():
    import paper_2406_00158_b200 as sr

    return {p: sr.Runtime(p, backend="meta") for p in (1, 2, 3, 4, 7)}

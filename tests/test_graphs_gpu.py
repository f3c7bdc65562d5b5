"""Cached element-wise plans over several segments of one GPU replay as one CUDA graph
(drk_graph_*).  The graph must read the vectors' current contents on every replay, wait for
asynchronous uploads like a direct launch, and count its kernels in drk_launch_count."""

import numpy as np
import pytest

import paper_2406_00158_b200 as sr
from paper_2406_00158_b200 import _lib, algorithms as A, kernels, plans, views

pytestmark = pytest.mark.gpu


def _graph_of(key_kind):
    for key, e in plans.CACHE._d.items():
        if key[0] == key_kind and isinstance(e.value, list) and e.value[2]:
            return e.value[2]
    return None


def test_transform_replays_as_graph():
    plans.CACHE.clear()
    with sr.Runtime(8, devices=[0]) as rt:
        n = 1_000_003
        x = sr.DistributedVector.from_numpy(rt, np.arange(n, dtype=np.float32))
        y = sr.DistributedVector(rt, n, dtype=np.float32)
        f = lambda v: v * 2.0 + 1.0  # noqa: E731
        for rep in range(4):
            k0 = _lib.launch_count()
            sr.transform(x, y, f)
            assert _lib.launch_count() - k0 == 8  # one kernel per segment, graph or not
            xv = np.arange(n, dtype=np.float32) + np.float32(rep)
            assert np.array_equal(y.to_numpy(), xv * np.float32(2.0) + np.float32(1.0))
            A.for_each(x, lambda v: v + 1.0)  # x changes between replays
        bound = _graph_of("for_each")
        assert bound is not None and isinstance(bound[0], kernels.BoundGraph)


def test_graph_waits_for_async_upload():
    plans.CACHE.clear()
    with sr.Runtime(4, devices=[0]) as rt:
        n = 1 << 20
        a = sr.DistributedVector(rt, n, dtype=np.float32)
        b = sr.DistributedVector(rt, n, dtype=np.float32)
        for _ in range(3):  # build and replay the copy plan
            A.copy(views.transform(a, lambda v: v * 3.0), b)
        host = sr.pinned_empty(n, np.float32)
        host[...] = np.arange(n, dtype=np.float32) % 11
        tk = a.upload(host, wait=False)
        A.copy(views.transform(a, lambda v: v * 3.0), b)  # must see the upload
        tk.wait()
        assert np.array_equal(b.to_numpy(), (np.arange(n, dtype=np.float32) % 11) * np.float32(3.0))
        bound = _graph_of("copy")
        assert bound is not None and isinstance(bound[0], kernels.BoundGraph)

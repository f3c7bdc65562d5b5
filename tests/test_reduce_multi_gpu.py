"""The multi-device batched reduce (drk_reduce_multi + per-GPU completion words), exercised on
one GPU: odd locales are served by a second DeviceState of device 0 (its own stream, result
slots, completion words and scratch), so the plan groups the segments into two "devices"
exactly as it does for two GPUs — one drk_reduce_multi call, two waits, partials decoded back
into segment order for the driver fold (reference algorithms.py:146-149)."""

import numpy as np
import pytest

import paper_2406_00158_b200 as sr
from paper_2406_00158_b200 import algorithms as A, bench as B, plans
from paper_2406_00158_b200.runtime import DeviceState
from oracle import segrange_port as O

pytestmark = pytest.mark.gpu


@pytest.fixture(params=["host", "fused"])
def split_rt(monkeypatch, request):
    rt = sr.Runtime(5, devices=[0], reduce_combine=request.param)
    alt = DeviceState(0, "cuda")
    orig = rt.state_of
    monkeypatch.setattr(rt, "state_of", lambda loc: alt if loc % 2 else orig(loc))
    plans.CACHE.clear()
    yield rt
    plans.CACHE.clear()
    rt.close()


def _plan(rt, r, op=A.add):
    return A._ReducePlan(rt, A._pieces(r), op)


@pytest.mark.parametrize("dtype", [np.int32, np.float32, np.float64, np.int64])
def test_reduce_multi_matches_oracle(split_rt, dtype):
    rt = split_rt
    n = 300_007
    x = O.mod_ints(7, 0, n, 2001, -1000).astype(dtype)
    v = sr.DistributedVector.from_numpy(rt, x)
    rt.synchronize()
    assert isinstance(_plan(rt, v).batch, A._MultiReduce)  # host mode runs it; fused mode folds in-kernel
    got = A.reduce(v, 0, A.add)
    want = O.reduce(x, 5, 0)
    assert type(got) is type(want)
    if np.dtype(dtype).kind == "i":
        assert got == want
    else:
        assert abs(got - want) <= 1e-5 * abs(want)
    assert A.reduce(v, 10**6, A.minimum) == min(10**6, x.min())
    assert A.reduce(v, -(10**6), A.maximum) == max(-(10**6), x.max())


def test_dot_multi_matches_oracle(split_rt):
    rt = split_rt
    n = 1 << 20
    x = O.unit_doubles(3, 0, n).astype(np.float32)
    y = O.unit_doubles(3, n, n).astype(np.float32)
    vx, vy = sr.DistributedVector.from_numpy(rt, x), sr.DistributedVector.from_numpy(rt, y)
    rt.synchronize()
    got = B.dot_product(vx, vy)
    want = O.dot(x, y, 5)
    assert abs(got - want) <= 1e-5 * abs(want)
    for _ in range(3):  # the cached plan, repeated (fresh epochs each call)
        assert B.dot_product(vx, vy) == got


def test_multi_reduce_under_profile(split_rt):
    """bench.py times kernels with kernels.profile(): the multi-device reduce then launches
    each GPU's batch through the profiler (both launches recorded), with the same result."""
    from paper_2406_00158_b200 import kernels

    rt = split_rt
    if rt.reduce_combine != "host":
        pytest.skip("the profiled multi-device launch is the host-combine path")
    x = O.mod_ints(9, 0, 100_003, 2001, -1000).astype(np.int64)
    v = sr.DistributedVector.from_numpy(rt, x)
    rt.synchronize()
    want = A.reduce(v, 0, A.add)
    with kernels.profile() as prof:
        got = A.reduce(v, 0, A.add)
    assert got == want == int(x.sum())
    assert len(prof.records.get("drk_reduce_batch", [])) == 2

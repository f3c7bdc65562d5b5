"""Scans of views fused into the scan kernel (no materialised intermediate): parity with the
oracle (the reference's materialise-then-accumulate path, oracle/segrange_port.py) on the
same inputs, through every scan schedule, at sizes that take the single-pass kernel and both
L2-kernel tile sizes; plus the launch count (one kernel per segment) and in-place scans.

Tolerances: bit-exact for integers, min/max and float data whose partial sums are exact;
relative 1e-5 (of the largest prefix magnitude) otherwise."""

import numpy as np
import pytest

from conftest import golden

import paper_2406_00158_b200 as sr
from paper_2406_00158_b200 import _lib, algorithms as A, views
from paper_2406_00158_b200.algorithms import _scan_aligned
from oracle import segrange_port as O

pytestmark = pytest.mark.gpu

SIZES = [1000, (3 << 20) + 7, (1 << 22) + 64]  # single-pass, single-pass (unaligned tail), L2 80 KB tiles


@pytest.fixture(params=["single", "batched", "device_carry", "host_carry"])
def schedule(request, monkeypatch):
    if request.param == "batched":
        monkeypatch.setattr(A, "_BATCH_MIN", 1)
    elif request.param != "single":
        monkeypatch.setattr(A, "_FORCE_MULTI_DEVICE_SCAN", True)
        monkeypatch.setattr(A, "_FORCE_HOST_CARRY", request.param == "host_carry")
    return request.param


def _sym(n, dt, seed=1, start=0):
    """{-1, 0, 1}: every partial sum is an exact small integer in any dtype."""
    return (O.mod_ints(seed, start, n, 3, -1)).astype(dt)


# (name, element function on one vector or a zip of two, arity, AOT kernel expected)
VIEWS = [
    ("product", lambda t: t[0] * t[1], 2),
    ("scale", lambda v: v * -2, 1),
    ("affine", lambda v: 2 * v + 0, 1),
    ("shift", lambda v: v - 0, 1),
    ("nvrtc_where", lambda v: np.where(v > 0, v * 3, -v) - 1, 1),
    ("nvrtc_zip", lambda t: np.minimum(t[0], t[1]) * 2 + t[1], 2),
]


def _host_values(fn, xs, arity, dt):
    with np.errstate(all="ignore"):
        v = fn(xs[0]) if arity == 1 else fn(tuple(xs))
    return np.asarray(v).astype(dt)


@pytest.mark.parametrize("n", SIZES)
@pytest.mark.parametrize("dt", [np.int32, np.float32, np.int64, np.float64], ids=lambda d: np.dtype(d).name)
@pytest.mark.parametrize("name,fn,arity", VIEWS, ids=[v[0] for v in VIEWS])
@pytest.mark.parametrize("p", [1, 3])
def test_fused_scan_matches_oracle(name, fn, arity, dt, n, p, rt_pool):
    rt = rt_pool(p)
    xs = [_sym(n, dt, seed=1 + k, start=k * n) for k in range(arity)]
    vs = [sr.DistributedVector.from_numpy(rt, x) for x in xs]
    view = views.transform(vs[0] if arity == 1 else views.zip(*vs), fn)
    vals = _host_values(fn, xs, arity, dt)
    for excl in (False, True):
        out = sr.DistributedVector(rt, n, dtype=dt)
        if excl:
            A.exclusive_scan(view, out, 5)
        else:
            A.inclusive_scan(view, out)
        exp, _ = O.scan(vals, p, dt, exclusive=excl, init=5 if excl else None)
        assert np.array_equal(out.to_numpy(), exp), (name, excl)


@pytest.mark.parametrize("case", [c for c in golden().cases if c["op"] == "scan_view"],
                         ids=lambda c: c["id"])
def test_scan_view_goldens_every_schedule(case, rt_pool, gold, schedule):
    x = O.generate(case["inputs"][0], np.int32)
    rt = rt_pool(case["p"])
    out = sr.DistributedVector(rt, case["n"], init=0, dtype=np.int32)
    A.inclusive_scan(views.transform(sr.DistributedVector.from_numpy(rt, x), lambda e: e * 3 - 1), out)
    assert np.array_equal(out.to_numpy(), gold.arrays[case["id"]])


@pytest.mark.parametrize("p", [1, 2, 5])
def test_fused_scan_partials_every_schedule(p, rt_pool, schedule):
    n = (1 << 21) + 33
    rt = rt_pool(p)
    x = _sym(n, np.int64, seed=9)
    v = sr.DistributedVector.from_numpy(rt, x)
    out = sr.DistributedVector(rt, n, dtype=np.int64)
    parts = _scan_aligned(views.transform(v, lambda e: e * 5 + 2), out, A.add, exclusive=False, init=None)
    exp, exp_parts = O.scan(x * 5 + 2, p)
    assert parts == exp_parts
    assert np.array_equal(out.to_numpy(), exp)


@pytest.mark.parametrize("dt", [np.float32, np.float64])
def test_fused_scan_float_accuracy(dt, rt_pool):
    n = (1 << 22) + 64
    rt = rt_pool(2)
    x = O.unit_doubles(3, 0, n).astype(dt)
    y = O.unit_doubles(3, n, n).astype(dt)
    vx, vy = sr.DistributedVector.from_numpy(rt, x), sr.DistributedVector.from_numpy(rt, y)
    out = sr.DistributedVector(rt, n, dtype=dt)
    A.inclusive_scan(views.transform(views.zip(vx, vy), lambda t: t[0] * t[1] + 0.25), out)
    ref = np.cumsum((x * y + dt(0.25)).astype(np.float64))
    got = out.to_numpy().astype(np.float64)
    rel = 1e-5 if dt == np.float32 else 1e-12
    assert np.max(np.abs(got - ref) / np.maximum(np.abs(ref), 1.0)) <= rel


@pytest.mark.parametrize("op,npop", [(A.maximum, np.maximum), (A.minimum, np.minimum), (A.multiply, None)])
def test_fused_scan_other_operators(op, npop, rt_pool):
    n = (1 << 22) + 64
    rt = rt_pool(3)
    x = O.unit_doubles(5, 0, n).astype(np.float32)
    v = sr.DistributedVector.from_numpy(rt, x)
    out = sr.DistributedVector(rt, n, dtype=np.float32)
    if npop is None:  # product scan of values in {1, -1}: exact
        xs = np.where(x > 0.5, np.float32(1), np.float32(-1))
        A.inclusive_scan(views.transform(v, lambda e: np.where(e > 0.5, 1.0, -1.0).astype(np.float32)), out, op)
        exp, _ = O.scan(xs, 3, ufunc=np.multiply)
    else:
        A.inclusive_scan(views.transform(v, lambda e: e * 2.0), out, op)
        exp, _ = O.scan((x * np.float32(2.0)).astype(np.float32), 3, ufunc=npop)
    assert np.array_equal(out.to_numpy(), exp)


@pytest.mark.parametrize("multi", [False, True])
def test_fused_scan_custom_combiner(multi, rt_pool, monkeypatch):
    if multi:
        monkeypatch.setattr(A, "_FORCE_MULTI_DEVICE_SCAN", True)
    n = (1 << 22) + 64
    rt = rt_pool(3)
    x = O.mod_ints(7, 0, n, 1000, -500).astype(np.int64)
    v = sr.DistributedVector.from_numpy(rt, x)
    out = sr.DistributedVector(rt, n, dtype=np.int64)
    op = sr.BinaryOp(lambda a, b: np.maximum(a, b) * 1)  # not a plain ufunc: a generated combiner
    parts = _scan_aligned(views.transform(v, lambda e: e * 3), out, op, exclusive=False, init=None)
    exp = np.maximum.accumulate(x * 3)
    assert np.array_equal(out.to_numpy(), exp)
    s = -(-n // 3)
    assert parts == [int(np.max(x[k * s:(k + 1) * s] * 3)) for k in range(3)]


def test_one_kernel_per_segment(rt_pool):
    n = 1 << 23
    for p in (1, 4):
        rt = rt_pool(p)
        x = O.unit_doubles(1, 0, n).astype(np.float32)
        v = sr.DistributedVector.from_numpy(rt, x)
        out = sr.DistributedVector(rt, n, dtype=np.float32)
        view = views.transform(v, lambda e: e * 2.5 + 1.0)
        A.inclusive_scan(view, out)  # warm (plans)
        rt.synchronize()
        k0 = _lib.launch_count()
        A.inclusive_scan(view, out)
        rt.synchronize()
        assert _lib.launch_count() - k0 == p  # one fused scan per segment, no map kernel


@pytest.mark.parametrize("dt", [np.int32, np.float64])
def test_fused_scan_in_place(dt, rt_pool):
    n = (1 << 22) + 64
    rt = rt_pool(2)
    x = _sym(n, dt)
    v = sr.DistributedVector.from_numpy(rt, x)
    A.inclusive_scan(views.transform(v, lambda e: e * 2), v)
    exp, _ = O.scan((x * 2).astype(dt), 2)
    assert np.array_equal(v.to_numpy(), exp)


@pytest.mark.slow
@pytest.mark.parametrize("dt", [np.int32, np.float32])
def test_fused_scan_large_tiles(dt, rt_pool):
    n = (1 << 25) + 16  # 160 KB tiles
    rt = rt_pool(1)
    x, y = _sym(n, dt, seed=2), _sym(n, dt, seed=3)
    vx, vy = sr.DistributedVector.from_numpy(rt, x), sr.DistributedVector.from_numpy(rt, y)
    out = sr.DistributedVector(rt, n, dtype=dt)
    A.exclusive_scan(views.transform(views.zip(vx, vy), lambda t: t[0] * t[1]), out, 0)
    exp, _ = O.scan((x * y).astype(dt), 1, exclusive=True, init=0)
    assert np.array_equal(out.to_numpy(), exp)

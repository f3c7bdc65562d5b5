"""Workload for compute-sanitizer (memcheck / racecheck / synccheck): every libdrk kernel
family once on small and ragged sizes, through the public API, checked against numpy.

    compute-sanitizer --tool memcheck  python tools/sanitize.py
    compute-sanitizer --tool racecheck python tools/sanitize.py --small

Covers map (copy, fill, iota, triad, Black-Scholes, NVRTC maps), reduce (dot, sum/min/max,
NVRTC reduce), scan (single-pass tiles, the L2 two-touch kernel, chained and batched over
segments), sort (both strategies: the radix sort, drk_gather, drk_sort_bounds) and the readback
kernel; round 2 adds fused view scans, the keep_tail L2 scan, both Black-Scholes tiers, float64
radix sorts with NaNs, CUDA-graph replays and the device / NCCL / fused reduce combines.
"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2406_00158_b200 as sr  # noqa: E402
from paper_2406_00158_b200 import algorithms as A, bench as B, views  # noqa: E402

small = "--small" in sys.argv
# segments >= 20000 elements take the L2 two-touch scan, smaller ones the single-pass scan
from paper_2406_00158_b200 import _lib  # noqa: E402

_lib.load().drk_tune(b"scan_l2_min", 20000)
rt = sr.Runtime(3)
rng = np.random.default_rng(0)
sizes = [1, 7, 4099, 100_003] + ([] if small else [(1 << 22) + 37])
for n in sizes:
    xf = rng.random(n).astype(np.float32)
    yf = rng.random(n).astype(np.float32)
    xi = rng.integers(-1000, 1000, n).astype(np.int32)
    vx, vy = sr.DistributedVector.from_numpy(rt, xf), sr.DistributedVector.from_numpy(rt, yf)
    vi = sr.DistributedVector.from_numpy(rt, xi)
    # map kernels
    a = sr.DistributedVector(rt, n, dtype=np.float32)
    B.stream_triad(a, vx, vy)
    assert np.array_equal(a.to_numpy(), xf + np.float32(3.0) * yf)
    A.fill(a, 2.5)
    A.transform(vx, a, lambda v: np.where(v > 0.5, v * v, -v))
    assert np.array_equal(a.to_numpy(), np.where(xf > 0.5, xf * xf, -xf))
    B.black_scholes_prices(a, *[sr.DistributedVector.from_numpy(rt, (90 + 20 * rng.random(n)).astype(np.float32))
                                for _ in range(2)],
                           *[sr.DistributedVector.from_numpy(rt, (0.1 + 0.2 * rng.random(n)).astype(np.float32))
                             for _ in range(3)])
    # reduce kernels
    d = B.dot_product(vx, vy)
    assert abs(d - float(np.dot(xf.astype(np.float64), yf))) <= 1e-5 * abs(d)
    assert A.reduce(vi, 0) == int(xi.astype(np.int64).sum())
    assert A.reduce(vi, 10**9, A.minimum) == int(xi.min())
    assert A.reduce(views.transform(vi, lambda v: v % 7), 0) == int((xi % 7).astype(np.int64).sum())
    # scan kernels (aligned, unaligned view, exclusive), chained and batched over the segments
    for batch_min in (1 << 20, 1):
        A._BATCH_MIN = batch_min
        o = sr.DistributedVector(rt, n, dtype=np.int32)
        A.inclusive_scan(vi, o)
        assert np.array_equal(o.to_numpy(), np.cumsum(xi.astype(np.int64)).astype(np.int32))
        if n > 3:
            o2 = sr.DistributedVector(rt, n - 3, dtype=np.int32)
            A.exclusive_scan(views.drop(vi, 3), o2, 5)
            exp = 5 + np.concatenate([[0], np.cumsum(xi[3:].astype(np.int64))[:-1]])
            assert np.array_equal(o2.to_numpy(), exp.astype(np.int32))
    A._BATCH_MIN = 1 << 20
    # sort (gather + sample strategies, keyed)
    for strategy in ("gather", "sample"):
        s = sr.DistributedVector.from_numpy(rt, xi)
        sr.sort(s, strategy=strategy)
        assert np.array_equal(s.to_numpy(), np.sort(xi))
        s = sr.DistributedVector.from_numpy(rt, xi)
        sr.sort(s, key=lambda v: v % 13, strategy=strategy)
        assert np.array_equal(s.to_numpy(), xi[np.argsort(xi % 13, kind="stable")])
    # round 2: fused view scans, the keep_tail L2 scan (8 sub-tiles forced), both
    # Black-Scholes tiers, float64 radix sort with NaNs, graph replays of a cached plan
    pf = sr.DistributedVector(rt, n, dtype=np.float32)
    A.inclusive_scan(views.transform(views.zip(vx, vy), lambda t: t[0] * t[1]), pf)
    A.inclusive_scan(views.transform(vx, lambda v: 2.5 * v + 1.0), pf)
    _lib.load().drk_tune(b"scan_l2_subs", 8)
    o = sr.DistributedVector(rt, n, dtype=np.int32)
    A.inclusive_scan(vi, o)
    assert np.array_equal(o.to_numpy(), np.cumsum(xi.astype(np.int64)).astype(np.int32))
    _lib.load().drk_tune(b"scan_l2_subs", 0)
    for precision in ("reference", "fast"):
        B.black_scholes_prices(a, *[sr.DistributedVector.from_numpy(rt, (90 + 20 * rng.random(n)).astype(np.float32))
                                    for _ in range(2)],
                               *[sr.DistributedVector.from_numpy(rt, (0.1 + 0.2 * rng.random(n)).astype(np.float32))
                                 for _ in range(3)], precision=precision)
    xd = rng.standard_normal(n)
    xd[::5] = np.nan
    s = sr.DistributedVector.from_numpy(rt, xd)
    sr.sort(s)
    assert np.array_equal(s.to_numpy(), np.sort(xd), equal_nan=True)
    for _ in range(3):  # a cached 3-segment plan: direct launches, then a CUDA graph replay
        A.for_each(a, lambda v: v * 0.5)
    print(f"n={n} ok", flush=True)
# round 2: the cross-GPU reduce combines (one GPU: 3 locales, a one-rank communicator)
for mode in ("device", "nccl", "fused"):
    with sr.Runtime(3, devices=[0], reduce_combine=mode) as rt2:
        x = rng.integers(-1000, 1000, 100_003).astype(np.int32)
        v = sr.DistributedVector.from_numpy(rt2, x)
        assert A.reduce(v, 0) == int(x.astype(np.int64).sum())
        assert A.reduce(v, 10**9, A.minimum) == int(x.min())
print("sanitize workload done")

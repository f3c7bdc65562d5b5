"""Workload for compute-sanitizer (memcheck / racecheck / synccheck): every libdrk kernel
family once on small and ragged sizes, through the public API, checked against numpy.

    compute-sanitizer --tool memcheck  python tools/sanitize.py
    compute-sanitizer --tool racecheck python tools/sanitize.py --small

Covers map (copy, fill, iota, triad, Black-Scholes, NVRTC maps), reduce (dot, sum/min/max,
NVRTC reduce), scan (single-pass tiles, the L2 two-touch kernel, chained and batched over
segments), sort (both strategies: CUB, drk_gather, drk_sort_bounds) and the readback kernel.
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
    print(f"n={n} ok", flush=True)
print("sanitize workload done")

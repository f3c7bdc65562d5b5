"""Parity at the BASELINE.json config sizes, element by element.

The golden vectors stop at 65,536 elements and the other parity tests at ~2^22, below the
tile configurations the headline numbers run (160 KB scan tiles with the first-wave
stagger at n >= 2^25, the batched 8-segment scan, the full-size STREAM / Black-Scholes
grids).  Here those exact configurations are compared with the oracle over the WHOLE
output: inputs come from the device twin of the reference's generator (repro.fill_*,
itself checked against the host generator below), are downloaded, and the reference's
algorithm runs on the host (oracle/segrange_port.py, or the numpy cumsum it reduces to
for exact data).

Tolerances: bit-exact for integer scans, the fp32 {-1,0,1} scan tier (every partial sum is
an exact integer < 2^24), STREAM copy/scale/add/triad and the generators; relative 1e-5
for the fp32 dot and Black-Scholes (against the reference's fp64-internal formula)."""

import numpy as np
import pytest

import paper_2406_00158_b200 as sr
from paper_2406_00158_b200 import algorithms as A, bench as B, repro
from oracle import segrange_port as O

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

N30 = 1 << 30


@pytest.fixture(params=["one_segment", "batched_8x2^27", "chained_8x2^27", "device_carry_8x2^27"])
def c3_schedule(request, monkeypatch):
    """C3's segment layouts on one GPU: the whole vector as one segment (the 160 KB-tile,
    staggered L2 kernel), and 8 segments of 2^27 scanned by one batched launch, by a chain of
    PDL-linked launches, or by the multi-GPU two-pass schedule (device carry fold)."""
    if request.param == "chained_8x2^27":
        monkeypatch.setattr(A, "_BATCH_SCANS", False)
    if request.param == "device_carry_8x2^27":
        monkeypatch.setattr(A, "_FORCE_MULTI_DEVICE_SCAN", True)
    return 1 if request.param == "one_segment" else 8


def _expected_scan(x, exclusive, init):
    """The reference's scan of exact data: the sequential prefix sums (int64 accumulate,
    stored into the output dtype)."""
    inc = np.cumsum(x, dtype=np.int64)
    if not exclusive:
        return inc
    exc = np.empty_like(inc)
    exc[0] = 0
    exc[1:] = inc[:-1]
    return exc + init


@pytest.mark.parametrize("dt", [np.int32, np.float32], ids=["int32_mod2001", "fp32_exact_tier"])
@pytest.mark.parametrize("exclusive", [False, True], ids=["inclusive", "exclusive"])
def test_c3_scan_2_30_whole_array(dt, exclusive, c3_schedule):
    p = c3_schedule
    with sr.Runtime(p, devices=[0]) as rt:
        x = sr.DistributedVector(rt, N30, dtype=dt)
        if dt == np.int32:
            repro.fill_mod(x, 1, 0, 2001, -1000)   # test_acceptance.py:70-74 data
        else:
            repro.fill_mod(x, 1, 0, 3, -1)         # {-1, 0, 1}: exact partial sums
        out = sr.DistributedVector(rt, N30, dtype=dt)
        if exclusive:
            A.exclusive_scan(x, out, 7)
        else:
            A.inclusive_scan(x, out)
        xs = x.to_numpy()
        got = out.to_numpy()
    assert np.array_equal(xs[:1 << 16], O.mod_ints(1, 0, 1 << 16, 2001 if dt == np.int32 else 3,
                                                   -1000 if dt == np.int32 else -1).astype(dt))
    exp = _expected_scan(xs.astype(np.int64), exclusive, 7)
    del xs
    # the fp32 tier stays exact (partial sums < 2^24); int32 never leaves its range
    assert np.abs(exp).max() < ((1 << 24) if dt == np.float32 else (1 << 31))
    assert np.array_equal(got, exp.astype(dt))


def test_c1_dot_2_24_two_segments():
    n = 1 << 24
    with sr.Runtime(2, devices=[0]) as rt:
        x = sr.DistributedVector(rt, n, dtype=np.float32)
        y = sr.DistributedVector(rt, n, dtype=np.float32)
        repro.fill_unit(x, 1, 0)          # bench_dot's scheme, bench.py:232-236
        repro.fill_unit(y, 1, n)
        got = B.dot_product(x, y)
        xs, ys = x.to_numpy(), y.to_numpy()
    assert np.array_equal(xs[:4096], O.unit_doubles(1, 0, 4096).astype(np.float32))
    exp = O.dot(xs, ys, 2)
    assert abs(got - exp) <= 1e-5 * abs(exp)
    assert abs(got - float(np.dot(xs.astype(np.float64), ys.astype(np.float64)))) <= 1e-5 * abs(exp)


@pytest.mark.parametrize("precision", ["reference", "fast"])
def test_c4_black_scholes_2_28_options(precision):
    n = 1 << 28
    cols = {}
    with sr.Runtime(1) as rt:
        vecs = []
        for k, (name, (lo, hi)) in enumerate(B.BS_RANGES.items()):
            v = sr.DistributedVector(rt, n, dtype=np.float32)
            repro.fill_uniform(v, 1, k * n, lo, hi)   # bench.py:268-273 columns
            vecs.append(v)
        out = sr.DistributedVector(rt, n, dtype=np.float32)
        B.black_scholes_prices(out, *vecs, precision=precision)
        got = out.to_numpy()
        for name, v in zip(B.BS_RANGES, vecs):
            cols[name] = v.to_numpy()
    lo, hi = B.BS_RANGES["spot"]
    assert np.array_equal(cols["spot"][:4096], O.uniform_doubles(1, 0, 4096, lo, hi).astype(np.float32))
    worst = 0.0
    ulps = 0
    chunk = 1 << 24
    for s in range(0, n, chunk):
        exp = O.black_scholes(*(cols[k][s:s + chunk] for k in B.BS_RANGES))  # fp64 internals
        g = got[s:s + chunk].astype(np.float64)
        worst = max(worst, float(np.max(np.abs(g - exp) / np.abs(exp))))
        if precision == "reference":  # the reference's fp32 result up to last-place ties
            d = np.abs(got[s:s + chunk].view(np.int32).astype(np.int64)
                       - exp.astype(np.float32).view(np.int32).astype(np.int64))
            assert d.max() <= 1
            ulps += int(np.count_nonzero(d))
    assert worst <= (1e-6 if precision == "reference" else 1e-5), worst
    assert ulps <= 1e-6 * n, ulps  # reference arithmetic: bit-identical up to rare fp64 erf/log ties


@pytest.mark.parametrize("kernel", ["copy", "scale", "add", "triad"])
def test_stream_fp32_2_26_bit_exact(kernel):
    n = 1 << 26
    with sr.Runtime(1) as rt:
        a = sr.DistributedVector(rt, n, dtype=np.float32)
        b = sr.DistributedVector(rt, n, dtype=np.float32)
        c = sr.DistributedVector(rt, n, dtype=np.float32)
        repro.fill_unit(b, 1, 0)
        repro.fill_unit(c, 1, n)
        if kernel == "copy":
            B.stream_copy(a, b)
        elif kernel == "scale":
            B.stream_scale(a, c)
        elif kernel == "add":
            B.stream_add(a, b, c)
        else:
            B.stream_triad(a, b, c)
        got, bs, cs = a.to_numpy(), b.to_numpy(), c.to_numpy()
    three = np.float32(3.0)
    exp = {"copy": bs, "scale": three * cs, "add": bs + cs, "triad": bs + three * cs}[kernel]
    assert np.array_equal(got, exp)


@pytest.mark.parametrize("dt", [np.float32, np.float64])
def test_fill_uniform_matches_host_generator(dt):
    n = (1 << 24) + 11
    with sr.Runtime(3, devices=[0]) as rt:
        v = sr.DistributedVector(rt, n, dtype=dt)
        repro.fill_uniform(v, 5, 1000, 70.0, 90.0)
        got = v.to_numpy()
        u = sr.DistributedVector(rt, n, dtype=dt)
        repro.fill_unit(u, 6, 0)
        gu = u.to_numpy()
    assert np.array_equal(got, O.uniform_doubles(5, 1000, n, 70.0, 90.0).astype(dt))
    assert np.array_equal(gu, O.unit_doubles(6, 0, n).astype(dt))

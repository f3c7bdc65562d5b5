"""Full-size and > 2^31-element runs on the GPU (64-bit indexing in every kernel family),
checked through size-independent properties: integer scan-last == reduce,
exclusive + input == inclusive at sampled indices, bit-exact triad samples regenerated on
the host, and fp32 scan accuracy against an fp64 total."""

import numpy as np
import pytest

import paper_2406_00158_b200 as sr
from paper_2406_00158_b200 import algorithms as A, bench as B, repro, views
from oracle import segrange_port as O

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


@pytest.fixture(scope="module")
def rt1():
    with sr.Runtime(1) as rt:
        yield rt


def _sample(vec, idx):
    seg = vec.segments()[0]
    return np.array([seg.get(int(i)) for i in idx])


@pytest.mark.parametrize("n", [(1 << 31) + 5])
def test_int32_scan_and_reduce_beyond_2_31(rt1, n):
    x = sr.DistributedVector(rt1, n, dtype=np.int32)
    repro.fill_mod(x, 3, 0, 3, -1)
    total = A.reduce(x, 0)
    out = sr.DistributedVector(rt1, n, dtype=np.int32)
    A.inclusive_scan(x, out)
    assert out[n - 1] == total  # int64 total of {-1,0,1}, fits int32
    idx = np.array([0, 1, 12345, (1 << 31) - 1, 1 << 31, n - 1])
    host = O.mod_ints(3, 0, 16, 3, -1)
    assert list(_sample(x, idx[:2])) == list(host[:2])
    exc = sr.DistributedVector(rt1, n, dtype=np.int32)
    A.exclusive_scan(x, exc, 0)
    e, i, v = _sample(exc, idx), _sample(out, idx), _sample(x, idx)
    assert np.array_equal(e + v, i)
    del out, exc


def test_triad_2_31_plus(rt1):
    n = (1 << 31) + 3
    b = sr.DistributedVector(rt1, n, dtype=np.float32)
    c = sr.DistributedVector(rt1, n, dtype=np.float32)
    repro.fill_unit(b, 1, 0)
    repro.fill_unit(c, 1, n)
    a = sr.DistributedVector(rt1, n, dtype=np.float32)
    B.stream_triad(a, b, c)
    for start in (0, (1 << 31) - 2, n - 4):
        bs = O.unit_doubles(1, start, 4).astype(np.float32)
        cs = O.unit_doubles(1, n + start, 4).astype(np.float32)
        got = np.array([a[start + k] for k in range(4)], dtype=np.float32)
        assert np.array_equal(got, bs + np.float32(3.0) * cs)
    d = B.dot_product(b, c)
    assert abs(d / (n / 4.0) - 1.0) < 1e-3


def test_fp32_scan_accuracy_2_30(rt1):
    # the reference's sequential fp32 scan drifts by ~50% at this size; our
    # fp64 carries keep the fp32 result within ~1e-6 of an fp64 scan
    n = 1 << 30
    x = sr.DistributedVector(rt1, n, dtype=np.float32)
    repro.fill_unit(x, 9, 0)
    out = sr.DistributedVector(rt1, n, dtype=np.float32)
    A.inclusive_scan(x, out)
    exact_total = sr.reduce(views.transform(x, lambda v: v.astype(np.float64)), 0.0)
    assert abs(out[n - 1] - exact_total) / exact_total < 1e-6

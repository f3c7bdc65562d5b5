"""Parity of the device runtime against the reference's golden vectors (GPU).

Every golden case (tests/golden, produced by the real reference) is replayed through the
public API on the GPU: the same inputs, the same segment count P (P locales on the
visible device(s)), the same call.  Tolerances (north star): bit-exact for integer work,
for element-wise float work with numpy rounding (triad, copy) and for the fp32 scan tier
whose partial sums are exact integers; relative 1e-5 for fp32 reductions/scans and
Black-Scholes (different association / fp32 internals), 1e-12 for fp64.
"""

import numpy as np
import pytest

from conftest import dec, golden

import paper_2406_00158_b200 as sr
from paper_2406_00158_b200 import algorithms as A
from paper_2406_00158_b200 import bench as B
from paper_2406_00158_b200 import views
from paper_2406_00158_b200.algorithms import _scan_aligned
from oracle import segrange_port as O

pytestmark = pytest.mark.gpu

CASES = golden().cases
REL = {"float32": 1e-5, "float64": 1e-12}


def _vec(rt, x):
    return sr.DistributedVector.from_numpy(rt, x)


def _close(got, exp, dtype, rel=None):
    rel = REL[dtype] if rel is None else rel
    if exp == 0:
        return abs(got) <= rel
    return abs(got - exp) <= rel * abs(exp)


def _sel(op):
    cs = [c for c in CASES if c["op"] == op and "raises" not in c]
    return pytest.mark.parametrize("case", cs, ids=[c["id"] for c in cs])


@_sel("dot")
def test_dot(case, rt_pool):
    dt = np.dtype(case["dtype"])
    x, y = [O.generate(d, dt) for d in case["inputs"]]
    rt = rt_pool(case["p"])
    got = B.dot_product(_vec(rt, x), _vec(rt, y))
    exp = dec(case["result"])
    assert isinstance(got, float)
    assert _close(got, exp, case["dtype"]), (got, exp)


@_sel("reduce")
def test_reduce(case, rt_pool):
    dt = np.dtype(case["dtype"])
    x = O.generate(case["inputs"][0], dt)
    rt = rt_pool(case["p"])
    got = A.reduce(_vec(rt, x), dec(case["init"]), getattr(A, case["ufunc"]))
    exp = dec(case["result"])
    assert type(got) is type(exp)
    if dt.kind == "i" or case["ufunc"] in ("minimum", "maximum"):
        assert got == exp  # exact: integer sums are exact, min/max select an element
    else:
        assert _close(got, exp, case["dtype"]), (got, exp)


@_sel("triad")
def test_triad_bit_exact(case, rt_pool, gold):
    dt = np.dtype(case["dtype"])
    b, c = [O.generate(d, dt) for d in case["inputs"]]
    rt = rt_pool(case["p"])
    a = sr.DistributedVector(rt, case["n"], dtype=dt)
    B.stream_triad(a, _vec(rt, b), _vec(rt, c), alpha=case["alpha"])
    out = a.to_numpy()
    assert O.checksum(out) == case["checksum"]
    if case.get("array"):
        assert np.array_equal(out, gold.arrays[case["id"]])


def _scan_cases():
    return [c for c in CASES if c["op"] in ("inclusive_scan", "exclusive_scan") and "raises" not in c]


@pytest.fixture(params=["single", "batched", "device_carry", "host_carry"])
def schedule(request, monkeypatch):
    """The scan schedule: one GPU's chained carries ("single": golden sizes are below the
    batching threshold), one batched launch over the GPU's segments (drk_scan_batch), or the
    multi-GPU two-pass schedule (forced onto the visible GPU) with the carry folded on the
    device (drk_carry_fold) or on the host."""
    if request.param == "batched":
        monkeypatch.setattr(A, "_BATCH_MIN", 1)
    elif request.param != "single":
        monkeypatch.setattr(A, "_FORCE_MULTI_DEVICE_SCAN", True)
        monkeypatch.setattr(A, "_FORCE_HOST_CARRY", request.param == "host_carry")
    return request.param


@pytest.mark.parametrize("case", _scan_cases(), ids=[c["id"] for c in _scan_cases()])
def test_scan(case, rt_pool, gold, schedule):
    dt = np.dtype(case["dtype"])
    x = O.generate(case["inputs"][0], dt)
    rt = rt_pool(case["p"])
    v = _vec(rt, x)
    out = sr.DistributedVector(rt, case["n"], init=0, dtype=dt)
    op = getattr(A, case.get("ufunc", "add"))
    excl = case["op"] == "exclusive_scan"
    parts = _scan_aligned(v, out, op, exclusive=excl, init=dec(case["init"]))
    got = out.to_numpy()
    exp_parts = [dec(p) for p in case["partials"]]
    exact = dt.kind == "i" or case.get("ufunc") in ("minimum", "maximum") or (
        dt == np.float32 and case.get("tier") != "accuracy")
    if exact:
        assert parts == exp_parts
        assert O.checksum(got) == case["checksum"]
        if case.get("array"):
            assert np.array_equal(got, gold.arrays[case["id"]])
    else:
        assert [p is None for p in parts] == [p is None for p in exp_parts]
        for p, e in zip(parts, exp_parts):
            if e is not None:
                assert _close(p, e, case["dtype"]), (p, e)
        if case.get("array"):
            ref = gold.arrays[case["id"]]
            np.testing.assert_allclose(got, ref, rtol=REL[case["dtype"]], atol=0)


def test_scan_int32_carry_overflow_raises(rt_pool, schedule):
    case = [c for c in CASES if "raises" in c][0]
    x = O.generate(case["inputs"][0], np.int32)
    rt = rt_pool(case["p"])
    with pytest.raises(sr.AggregateTaskError) as ei:
        A.inclusive_scan(_vec(rt, x), sr.DistributedVector(rt, case["n"], init=0, dtype=np.int32))
    assert all(isinstance(e, OverflowError) for _, e in ei.value.failures)


@pytest.mark.parametrize("init", [5, 2**31 - 1, -(2**31), 2**31, -(2**31) - 1])
def test_scan_int32_single_segment_seed_range(rt_pool, init):
    """One live segment: the int32 range check sees only the init seed (no totals read back,
    the scan stays asynchronous); in-range seeds wrap like numpy, out-of-range ones raise
    OverflowError like the reference (algorithms.py:292-308)."""
    x = ((np.arange(4099, dtype=np.int64) * 7919) % 2001 - 1000).astype(np.int32)
    rt = rt_pool(1)
    v = _vec(rt, x)
    out = sr.DistributedVector(rt, len(x), init=0, dtype=np.int32)
    try:
        exp, _ = O.scan(x, 1, exclusive=True, init=init)
    except OverflowError:
        with pytest.raises(sr.AggregateTaskError) as ei:
            A.exclusive_scan(v, out, init)
        assert all(isinstance(e, OverflowError) for _, e in ei.value.failures)
        return
    A.exclusive_scan(v, out, init)
    assert np.array_equal(out.to_numpy(), exp)
    A.inclusive_scan(v, out)
    assert np.array_equal(out.to_numpy(), O.scan(x, 1)[0])


@_sel("black_scholes")
def test_black_scholes(case, rt_pool, gold):
    dt = np.dtype(case["dtype"])
    cols = [O.generate(d, dt) for d in case["inputs"]]
    rt = rt_pool(case["p"])
    out = sr.DistributedVector(rt, case["n"], dtype=dt)
    B.black_scholes_prices(out, *[_vec(rt, c) for c in cols])
    got = out.to_numpy()
    ref = gold.arrays[case["id"]]
    if dt == np.float32:
        # the reference's arithmetic replayed (fp32 vol/discount/drift, numpy's float32 exp,
        # fp64 CDFs): bit-exact (the fast fp32 tier is checked at rel 1e-5 in test_api_gpu and
        # test_config_parity_gpu)
        assert np.array_equal(got, ref)
    else:
        np.testing.assert_allclose(got, ref, rtol=REL[case["dtype"]], atol=0)


@_sel("copy")
def test_copy_repartition(case, rt_pool, gold):
    dt = np.dtype(case["dtype"])
    x = O.generate(case["inputs"][0], dt)
    v3 = _vec(rt_pool(3), x)
    v4 = sr.DistributedVector(rt_pool(4), case["n"], dtype=dt)
    A.copy(v3, v4)
    assert np.array_equal(v4.to_numpy(), gold.arrays[case["id"]])


def test_known_answers(rt3):
    kat = golden().meta["kat"]
    x = _vec(rt3, np.array([1.0, 2.0, 3.0]))
    y = _vec(rt3, np.array([4.0, 5.0, 6.0]))
    assert B.dot_product(x, y) == dec(kat["dot_123_456"]) == 32.0
    assert abs(float(B.black_scholes_call(100.0, 100.0, 0.0, 0.2, 1.0)) - dec(kat["bs_atm"])) < 1e-12
    assert float(B.black_scholes_call(110.0, 100.0, 0.0, 0.0, 1.0)) == 10.0
    assert float(B.black_scholes_call(90.0, 100.0, 0.0, 0.0, 1.0)) == 0.0


SORT_KEYS = {"none": None, "abs": lambda x: np.abs(x), "neg": lambda x: -x}


@pytest.mark.parametrize("strategy", ["sample", "gather"])
@_sel("sort")
def test_sort(case, strategy, rt_pool, gold):
    """Both sort strategies reproduce the reference's sample sort bit-for-bit (keys: the
    stable order of equal keys is part of the result)."""
    dt = np.dtype(case["dtype"])
    x = O.generate(case["inputs"][0], dt)
    v = _vec(rt_pool(case["p"]), x)
    A.sort(v, key=SORT_KEYS[case["key"]], strategy=strategy)
    got = v.to_numpy()
    assert O.checksum(got) == case["checksum"]
    if case.get("array"):
        assert np.array_equal(got, gold.arrays[case["id"]])


@_sel("reduce_view")
def test_reduce_over_drop_take(case, rt_pool):
    dt = np.dtype(case["dtype"])
    x = O.generate(case["inputs"][0], dt)
    v = _vec(rt_pool(case["p"]), x)
    got = A.reduce(views.take(views.drop(v, case["drop"]), case["take"]), 0, A.add)
    exp = dec(case["result"])
    if dt.kind == "i":
        assert type(got) is type(exp) and got == exp
    else:
        assert _close(got, exp, case["dtype"]), (got, exp)


@_sel("dot_nonaligned")
def test_dot_over_nonaligned_zip(case, rt_pool):
    dt = np.dtype(case["dtype"])
    x, y = [O.generate(d, dt) for d in case["inputs"]]
    pa, pb = case["parts"]
    rt = rt_pool(max(len(pa), len(pb)))
    vx = sr.DistributedVector.from_numpy(rt, x, partition=pa)
    vy = sr.DistributedVector.from_numpy(rt, y, partition=pb)
    got = A.reduce(views.transform(views.zip(vx, vy), lambda t: t[0] * t[1]), 0.0, A.add)
    assert _close(got, dec(case["result"]), case["dtype"])


@_sel("scan_view")
def test_scan_of_transform_view(case, rt_pool, gold):
    x = O.generate(case["inputs"][0], np.int32)
    rt = rt_pool(case["p"])
    out = sr.DistributedVector(rt, case["n"], init=0, dtype=np.int32)
    A.inclusive_scan(views.transform(_vec(rt, x), lambda e: e * 3 - 1), out)
    got = out.to_numpy()
    assert O.checksum(got) == case["checksum"]
    assert np.array_equal(got, gold.arrays[case["id"]])


@_sel("copy_transform")
def test_copy_of_transform_view(case, rt_pool, gold):
    dt = np.dtype(case["dtype"])
    x = O.generate(case["inputs"][0], dt)
    rt = rt_pool(case["p"])
    out = sr.DistributedVector(rt, case["n"], init=0, dtype=dt)
    fn = (lambda e: e * 7 - 3) if dt.kind == "i" else (lambda e: e * 2.5 + 1)
    A.copy(views.transform(_vec(rt, x), fn), out)
    got = out.to_numpy()  # bit-exact: numpy's rounding of each operation (no FMA contraction)
    assert O.checksum(got) == case["checksum"]
    assert np.array_equal(got, gold.arrays[case["id"]])

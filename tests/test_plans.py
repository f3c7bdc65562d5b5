"""Plan cache (plans.py): structural keys of view chains, invalidation, eviction.  CPU tests
on the metadata-only runtime; the GPU tests check cached calls give the uncached results."""

import gc

import numpy as np
import pytest

import paper_2406_00158_b200 as sr
from paper_2406_00158_b200 import algorithms as A, plans, views


class _Box:
    k = 2.0


def _key(r):
    return plans.view_key(r, [])


def test_structural_keys_repeat_for_fresh_view_objects(meta_rt):
    rt = meta_rt[2]
    x = sr.DistributedVector(rt, 100, dtype=np.float32)
    y = sr.DistributedVector(rt, 100, dtype=np.float32)
    f = lambda t: t[0] * t[1]  # noqa: E731
    k1 = _key(views.transform(views.zip(x, y), f))
    k2 = _key(views.transform(views.zip(x, y), f))
    assert k1 is not None and k1 == k2
    assert _key(views.transform(views.zip(y, x), f)) != k1
    assert _key(views.take(x, 10)) == ("trim", 0, 10, ("dv", id(x)))
    assert _key(views.drop(x, 10)) == ("trim", 10, 100, ("dv", id(x)))
    assert _key(views.iota(3, 5)) == ("iota", 3, 5)
    assert _key(views.zip(x, y, mode="strict")) != _key(views.zip(x, y))


def test_uncacheable_views(meta_rt):
    rt = meta_rt[2]
    x = sr.DistributedVector(rt, 10, dtype=np.float64)
    box = _Box()
    assert _key(views.transform(x, lambda v: v * box.k)) is None  # reaches mutable state
    assert _key(views.zip(x, np.arange(10.0))) is None             # host data
    a, b = 2.0, 3.0
    assert _key(views.transform(x, lambda v: v * a)) != _key(views.transform(x, lambda v: v * b))


def test_cache_entry_dies_with_its_vector(meta_rt):
    rt = meta_rt[1]
    cache = plans.PlanCache()
    x = sr.DistributedVector(rt, 10, dtype=np.float64)
    dvs = []
    key = ("k", plans.view_key(x, dvs))
    cache.put(key, dvs, "plan")
    assert cache.get(key) == "plan" and len(cache) == 1
    del x, dvs
    gc.collect()
    assert len(cache) == 0 and cache.get(key) is None


def test_cache_entry_invalid_after_free(meta_rt):
    rt = meta_rt[1]
    cache = plans.PlanCache()
    x = sr.DistributedVector(rt, 10, dtype=np.float64)
    dvs = []
    key = ("k", plans.view_key(x, dvs))
    cache.put(key, dvs, "plan")
    x.storage[0].free()
    assert cache.get(key) is None


def test_cache_bounded(meta_rt):
    rt = meta_rt[1]
    cache = plans.PlanCache(maxsize=4)
    xs = [sr.DistributedVector(rt, 4, dtype=np.float64) for _ in range(6)]
    for i, x in enumerate(xs):
        cache.put(("k", i), [x], i)
    assert len(cache) == 4 and cache.get(("k", 0)) is None and cache.get(("k", 5)) == 5


@pytest.mark.gpu
def test_cached_calls_match_uncached(rt_pool, monkeypatch):
    rt = rt_pool(3)
    n = 100_003
    rng = np.random.default_rng(0)
    xs, ys = rng.random(n), rng.random(n)
    x, y = sr.DistributedVector.from_numpy(rt, xs), sr.DistributedVector.from_numpy(rt, ys)
    out = sr.DistributedVector(rt, n, dtype=np.float64)
    res = []
    for enabled in (False, True, True):
        monkeypatch.setattr(plans, "_ENABLED", enabled)
        d = A.reduce(views.transform(views.zip(x, y), lambda t: t[0] * t[1]), 0.0)
        A.inclusive_scan(views.transform(x, lambda v: v * 2.0), out)
        A.for_each(views.zip(out, y), lambda t: (t[0] + t[1], None), vectorized=True)
        A.copy(views.transform(out, lambda v: v - 1.0), out)
        res.append((d, out.to_numpy()))
    assert res[0][0] == res[1][0] == res[2][0]
    assert np.array_equal(res[0][1], res[1][1]) and np.array_equal(res[1][1], res[2][1])


@pytest.mark.gpu
def test_cache_follows_mutable_state(rt_pool):
    rt = rt_pool(2)
    x = sr.DistributedVector.from_numpy(rt, np.ones(1000))
    box = _Box()
    v = views.transform(x, lambda e: e * box.k)
    assert A.reduce(v, 0.0) == 2000.0
    box.k = 5.0
    assert A.reduce(v, 0.0) == 5000.0
    k = 1.0
    assert A.reduce(views.transform(x, lambda e: e * k), 0.0) == 1000.0
    k = 3.0
    assert A.reduce(views.transform(x, lambda e: e * k), 0.0) == 3000.0


@pytest.mark.gpu
def test_cache_releases_dead_vectors(rt_pool):
    rt = rt_pool(2)
    x = sr.DistributedVector.from_numpy(rt, np.arange(1000.0))
    assert A.reduce(x, 0.0) == 499500.0
    before = len(plans.CACHE)
    del x
    gc.collect()
    assert len(plans.CACHE) < before

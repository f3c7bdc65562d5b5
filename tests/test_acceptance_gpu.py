"""Acceptance criteria of the reference (pkg/tests/test_acceptance.py) replayed on the GPU
runtime: the concatenation law over random view compositions (:299-353), adversarial
sorts (:444-466), and P-independence of results (checksums identical across segment
counts, test_bench.py:237-245).  Expected values are computed with plain Python/numpy on
the host, independent of the package."""

from collections import Counter

import numpy as np
import pytest

import paper_2406_00158_b200 as sr
from paper_2406_00158_b200 import algorithms as A
from paper_2406_00158_b200 import bench as B
from paper_2406_00158_b200 import views
from oracle import segrange_port as O

pytestmark = pytest.mark.gpu


def _double_nested(x):
    if isinstance(x, tuple):
        return tuple(_double_nested(v) for v in x)
    return x * 2


def _random_composition(rng, rt, depth):
    """reference test_acceptance.py:317-346: random chains of transform/take/drop/zip over
    vectors with random partitions (and plain host arrays)."""
    if depth >= 4 or rng.random() < 0.3:
        n = int(rng.integers(0, 14))
        data = [float(x) for x in rng.integers(-9, 9, n)]
        if rng.random() < 0.25:
            return np.asarray(data), data
        parts = None
        if n > 1 and rng.random() < 0.5:
            cuts = sorted(set(int(c) for c in rng.integers(1, n, 2)))
            bounds = [0] + cuts + [n]
            parts = [bounds[i + 1] - bounds[i] for i in range(len(bounds) - 1)]
        return sr.DistributedVector.from_numpy(rt, np.asarray(data), partition=parts), data
    kind = rng.choice(["transform", "take", "drop", "zip"])
    base, expected = _random_composition(rng, rt, depth + 1)
    if kind == "transform":
        return views.transform(base, _double_nested), [_double_nested(x) for x in expected]
    if kind == "take":
        k = int(rng.integers(0, len(expected) + 3))
        return views.take(base, k), expected[:k]
    if kind == "drop":
        k = int(rng.integers(0, len(expected) + 3))
        return views.drop(base, k), expected[k:]
    other, other_expected = _random_composition(rng, rt, depth + 1)
    n = min(len(expected), len(other_expected))
    return views.zip(base, other), [(expected[i], other_expected[i]) for i in range(n)]


def _plain(x):
    if isinstance(x, tuple):
        return tuple(_plain(v) for v in x)
    return float(x)


def test_concatenation_law(rt_pool):
    """Iterating a view == the composition evaluated on host lists; for segmented views the
    concatenation of the segments' elements is the same sequence."""
    rng = np.random.default_rng(2024)
    rt = rt_pool(3)
    bad = []
    for i in range(300):
        view, expected = _random_composition(rng, rt, depth=0)
        got = [_plain(e) for e in view]
        if got != expected:
            bad.append((i, "iter"))
            continue
        if getattr(view, "is_segmented", False):
            flat = [_plain(e) for s in sr.segments_of(view) for e in s]
            if flat != expected:
                bad.append((i, "segments"))
    assert not bad, bad[:10]


@pytest.mark.parametrize("strategy", ["sample", "gather"])
def test_sort_adversarial(rt_pool, strategy):
    n = 100_000
    cases = {
        "all-equal": np.full(n, 7, dtype=np.int64),
        "pre-sorted": np.arange(n, dtype=np.int64),
        "reverse": np.arange(n, dtype=np.int64)[::-1].copy(),
        "two-valued": (O.splitmix64(5, 0, n) % 2).astype(np.int64),
        "organ-pipe": np.concatenate([np.arange(n // 2), np.arange(n - n // 2)[::-1]]).astype(np.int64),
        "sawtooth": (np.arange(n) % 97).astype(np.int64),
    }
    bad = []
    for p in (1, 4, 7):
        rt = rt_pool(p)
        for name, data in cases.items():
            v = sr.DistributedVector.from_numpy(rt, data)
            sr.sort(v, strategy=strategy)
            out = v.to_numpy()
            if not (np.diff(out) >= 0).all():
                bad.append(f"{name} P={p} not sorted")
            if Counter(out.tolist()) != Counter(data.tolist()):
                bad.append(f"{name} P={p} multiset broken")
    assert not bad, bad


def test_p_independence(rt_pool):
    """Integer results and element-wise float results do not depend on the segment count."""
    n = 100_003
    xi = O.mod_ints(3, 0, n, 2001, -1000).astype(np.int64)
    bf = O.unit_doubles(3, 0, n).astype(np.float32)
    cf = O.unit_doubles(3, n, n).astype(np.float32)
    sums, scans, triads, sorts = set(), set(), set(), set()
    for p in (1, 2, 3, 4, 7):
        rt = rt_pool(p)
        v = sr.DistributedVector.from_numpy(rt, xi)
        sums.add(A.reduce(v, 0, A.add))
        out = sr.DistributedVector(rt, n, dtype=np.int64)
        A.inclusive_scan(v, out)
        scans.add(O.checksum(out.to_numpy()))
        a = sr.DistributedVector(rt, n, dtype=np.float32)
        B.stream_triad(a, sr.DistributedVector.from_numpy(rt, bf), sr.DistributedVector.from_numpy(rt, cf))
        triads.add(O.checksum(a.to_numpy()))
        sr.sort(v)
        sorts.add(O.checksum(v.to_numpy()))
    assert len(sums) == len(scans) == len(triads) == len(sorts) == 1
    assert sums == {int(xi.sum())}
    assert scans == {O.checksum(np.cumsum(xi))}
    assert sorts == {O.checksum(np.sort(xi))}

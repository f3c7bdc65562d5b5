"""Host-side logic without a GPU: partition metadata, view segment algebra, runtime
bookkeeping (backend="meta": storage with shape and dtype but no memory; any compute
raises).  Mirrors the reference's tests/test_core.py and tests/test_views.py expectations,
computed here with independent plain-Python helpers."""

import numpy as np
import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

import paper_2406_00158_b200 as sr
from paper_2406_00158_b200 import views
from paper_2406_00158_b200.core import Distribution, SegmentDescriptor, is_aligned, rank_of, segments_of


def block_lengths(n, p):
    if n == 0:
        return []
    s = -(-n // p)
    return [min(s, max(0, n - i * s)) for i in range(p)]


def trim_pieces(lengths, ranks, f, l):
    owners = []
    for seg, (length, rank) in enumerate(zip(lengths, ranks)):
        owners.extend([(seg, rank)] * length)
    pieces = []
    for seg, rank in owners[f:l]:
        if pieces and pieces[-1][0] == seg:
            pieces[-1][2] += 1
        else:
            pieces.append([seg, rank, 1])
    return [(c, r) for _, r, c in pieces]


def boundaries(lengths):
    cuts, pos = set(), 0
    for ln in lengths[:-1]:
        pos += ln
        cuts.add(pos)
    cuts.discard(0)
    cuts.discard(sum(lengths))
    return cuts


def shape(r):
    return [(len(s), s.rank) for s in segments_of(r)]


class TestDistribution:
    @pytest.mark.parametrize("n,p", [(0, 3), (1, 3), (10, 3), (4, 8), (1000, 7), (12, 4)])
    def test_block_rule(self, n, p):
        d = Distribution.block(n, p)
        assert d.lengths() == block_lengths(n, p)
        assert [x.rank for x in d.descriptors] == list(range(len(d.descriptors)))

    def test_locale_wraps(self):
        d = Distribution.block(10, 5, 2)
        assert [x.rank for x in d.descriptors] == [0, 1, 0, 1, 0]

    def test_tiling_validation(self):
        with pytest.raises(ValueError):
            Distribution(5, (SegmentDescriptor(0, 0, 2), SegmentDescriptor(1, 3, 2)))
        with pytest.raises(ValueError):
            Distribution(5, (SegmentDescriptor(0, 0, 2),))
        with pytest.raises(ValueError):
            SegmentDescriptor(-1, 0, 1)

    def test_segment_of(self):
        d = Distribution.from_lengths([3, 0, 4], 3)
        assert d.segment_of(0) == (0, 0)
        assert d.segment_of(3) == (2, 0)
        assert d.segment_of(6) == (2, 3)
        with pytest.raises(IndexError):
            d.segment_of(7)


class TestMetaRuntime:
    def test_vector_partition(self, meta_rt):
        for p, rt in meta_rt.items():
            for n in (0, 1, 5, 23, 1000):
                v = sr.DistributedVector(rt, n, dtype=np.float32)
                assert [len(s) for s in v.segments()] == block_lengths(n, p)
                assert all(s.rank == i % p for i, s in enumerate(v.segments()))

    def test_explicit_partition(self, meta_rt):
        v = sr.DistributedVector(meta_rt[3], 10, partition=[7, 0, 3])
        assert shape(v) == [(7, 0), (0, 1), (3, 2)]
        with pytest.raises(ValueError):
            sr.DistributedVector(meta_rt[3], 10, partition=[7, 2])

    def test_meta_cannot_compute(self, meta_rt):
        v = sr.DistributedVector(meta_rt[2], 4)
        with pytest.raises(RuntimeError):
            sr.reduce(v, 0.0)
        with pytest.raises(RuntimeError):
            v.to_numpy()

    def test_live_allocations_and_free(self, meta_rt):
        rt = meta_rt[2]
        h = rt.allocate(1, 8, np.float64)
        assert rt.live_allocations(1) >= 1
        h.free()
        with pytest.raises(RuntimeError):
            h.free()
        with pytest.raises(RuntimeError):
            h.span()

    def test_submit_wait_all_errors(self, meta_rt):
        rt = meta_rt[3]

        def bad():
            raise KeyError("x")

        t = [rt.submit(0, lambda: 1), rt.submit(1, bad), rt.submit(2, lambda: sr.current_locale())]
        with pytest.raises(sr.AggregateTaskError) as ei:
            rt.wait_all(t)
        assert [i for i, _ in ei.value.failures] == [1]
        assert rt.wait_all([t[0], t[2]]) == [1, 2]
        with pytest.raises(ValueError):
            rt.submit(3, lambda: None)

    def test_default_locale_count_env(self, monkeypatch):
        monkeypatch.setenv("SEGRANGE_LOCALES", "5")
        assert sr.default_locale_count() == 5
        monkeypatch.setenv("SEGRANGE_LOCALES", "0")
        with pytest.raises(ValueError):
            sr.default_locale_count()


class TestViewsAlgebra:
    def test_transform_mirrors_segments(self, meta_rt):
        v = sr.DistributedVector(meta_rt[3], 10)
        t = views.transform(v, lambda x: x * 2)
        assert shape(t) == shape(v)
        assert t.rank is None and len(t) == 10

    @pytest.mark.parametrize("f,l", [(0, 10), (2, 9), (4, 4), (0, 1), (9, 10), (3, 7)])
    def test_trim(self, meta_rt, f, l):
        v = sr.DistributedVector(meta_rt[3], 10)
        got = [(len(s), s.rank) for s in views.trim_segments(v.segments(), f, l)]
        assert got == trim_pieces(block_lengths(10, 3), [0, 1, 2], f, l)

    def test_take_drop(self, meta_rt):
        v = sr.DistributedVector(meta_rt[4], 10)
        assert shape(views.take(v, 4)) == trim_pieces(block_lengths(10, 4), [0, 1, 2, 3], 0, 4)
        assert shape(views.drop(v, 4)) == trim_pieces(block_lengths(10, 4), [0, 1, 2, 3], 4, 10)
        assert len(views.take(v, 99)) == 10 and len(views.drop(v, 99)) == 0
        with pytest.raises(ValueError):
            views.take(v, -1)

    def test_zip_aligned_and_realigned(self, meta_rt):
        rt = meta_rt[2]
        a = sr.DistributedVector(rt, 10, partition=[6, 4])
        b = sr.DistributedVector(rt, 10, partition=[3, 7])
        z = views.zip(a, b)
        lens = [len(s) for s in z.segments()]
        assert sum(lens) == 10
        cuts = boundaries(lens)
        assert cuts == boundaries([6, 4]) | boundaries([3, 7])
        assert [s.rank for s in z.segments()] == [0, 0, 1]
        assert is_aligned(a, sr.DistributedVector(rt, 10, partition=[6, 4]))
        assert not is_aligned(a, b)

    def test_zip_truncates_and_strict(self, meta_rt):
        rt = meta_rt[3]
        a = sr.DistributedVector(rt, 10)
        b = sr.DistributedVector(rt, 7)
        assert len(views.zip(a, b)) == 7
        with pytest.raises(sr.NonAlignedZip):
            views.zip(a, sr.DistributedVector(rt, 10, partition=[1, 9, 0]), mode="strict")
        with pytest.raises(TypeError):
            views.zip(a)

    def test_enumerate_segments(self, meta_rt):
        v = sr.DistributedVector(meta_rt[3], 10)
        e = views.enumerate(v)
        assert shape(e) == shape(v)
        bases = [views.lower(s).leaves[0].base for s in e.segments()]
        assert bases == [0, 4, 8]

    def test_lowering_structure(self, meta_rt):
        v = sr.DistributedVector(meta_rt[2], 8, dtype=np.float32)
        w = sr.DistributedVector(meta_rt[2], 8, dtype=np.float32)
        z = views.transform(views.zip(v, w), lambda t: t[0] * t[1])
        lw = views.lower(z.segments()[1])
        assert lw.value.op == "multiply" and [lf.start for lf in lw.leaves] == [0, 0]
        d = views.drop(v, 5)
        lw = views.lower(d.segments()[0])
        assert lw.leaves[0].start == 1 and lw.length == 3

    def test_rank_of(self, meta_rt):
        v = sr.DistributedVector(meta_rt[3], 6)
        assert rank_of(v.segments()[2]) == 2
        with pytest.raises(TypeError):
            rank_of(v)
        with pytest.raises(sr.OffLocaleAccess):
            sr.local_view(v.segments()[0])

    @given(st.lists(st.integers(0, 9), min_size=1, max_size=5), st.lists(st.integers(0, 9), min_size=1, max_size=5))
    @settings(max_examples=60)
    def test_realign_boundary_law(self, la, lb):
        # boundary law of the reference's acceptance test (test_acceptance.py:360-409)
        rt = sr.Runtime(max(len(la), len(lb)), backend="meta")
        n = min(sum(la), sum(lb))
        if n == 0:
            return
        a = sr.DistributedVector(rt, sum(la), partition=la)
        b = sr.DistributedVector(rt, sum(lb), partition=lb)
        z = views.zip(a, b)
        lens = [len(s) for s in z.segments()]
        assert sum(lens) == n and all(lens)
        ta = [len(s) for s in views.trim_segments(a.segments(), 0, n)]
        tb = [len(s) for s in views.trim_segments(b.segments(), 0, n)]
        assert boundaries(lens) == boundaries(ta) | boundaries(tb)


def test_reduce_combine_option():
    """Runtime(reduce_combine=...) accepts the three combine modes and rejects others."""
    import paper_2406_00158_b200 as sr
    from paper_2406_00158_b200.runtime import REDUCE_COMBINES

    assert REDUCE_COMBINES == ("host", "device", "nccl", "fused")
    for mode in REDUCE_COMBINES:
        assert sr.Runtime(2, backend="meta", reduce_combine=mode).reduce_combine == mode
    assert sr.Runtime(2, backend="meta").reduce_combine in REDUCE_COMBINES
    with pytest.raises(ValueError):
        sr.Runtime(2, backend="meta", reduce_combine="allreduce")


def test_spmd_value_dtype_of_empty_view():
    """An empty rank-local view still reports its element dtype (spmd.reduce decodes the
    gathered partials in it, like the ranks that hold elements)."""
    import paper_2406_00158_b200 as sr
    from paper_2406_00158_b200 import spmd, views

    rt = sr.Runtime(2, backend="meta")
    v = sr.DistributedVector(rt, 0, dtype=np.float32)
    w = sr.DistributedVector(rt, 0, dtype=np.float32)
    assert spmd._value_dtype(v) == np.float32
    assert spmd._value_dtype(w) == np.float32
    # a view with (trailing empty) segments lowers to its element dtype
    x = sr.DistributedVector(rt, 1, dtype=np.float32)
    assert spmd._value_dtype(views.transform(views.zip(x, x), lambda t: t[0] * t[1])) == np.float32
    assert spmd._value_dtype(views.transform(x, lambda e: e * 2)) == np.float32

"""Plan cache: lowered segment work, memoised by the structure of the view it came from.

Every algorithm call walks the view chain to segments (zip realignment, trims), lowers each
segment to leaves + an expression, traces element functions and matches the kernel
catalogue — the reference rebuilds its segment objects on every call too (views.py:271-556,
"O(P) host objects per call").  On a GPU that host work is most of a small
call (dot at 2^24 over 2 segments: ~65 us of Python against a 36 us kernel).  The plan cache
keys that work by the view's *structure* —

    DistributedVector        ("dv", id)           (validity: the same live object)
    transform(base, fn)      ("tf", fn key, base)  (expr._fn_key: code + frozen state)
    zip(*bases)              ("zip", mode, n, bases)
    take / drop              ("trim", start, stop, base)
    iota(start, n)           ("iota", start, n)

— so `dot_product(x, y)`, which builds fresh zip/transform views on every call, hits the same
entry.  Anything else (host arrays, functions that reach mutable state, custom segment
types) has no key and is lowered every time, exactly as before.

An entry keeps its vectors' storage handles (the lowered leaves point into them); it is
dropped when any of its vectors is garbage-collected (weakref.finalize), when one of its
storage handles is freed, and beyond CACHE_MAX entries (oldest first).  Cached entries carry
no device state: pending transfers, stream order and scratch are resolved at every call.
"""

from __future__ import annotations

import weakref
from collections import OrderedDict

from . import expr

CACHE_MAX = 512
_ENABLED = True  # tests compare cached and uncached calls


class _Entry:
    __slots__ = ("deps", "handles", "value")

    def __init__(self, deps, handles, value):
        self.deps = deps          # weakrefs to the DistributedVectors of the key
        self.handles = handles    # their storage handles (freed -> stale)
        self.value = value

    def valid(self) -> bool:
        for ref in self.deps:
            if ref() is None:
                return False
        for h in self.handles:
            if h._freed:
                return False
        return True


class PlanCache:
    def __init__(self, maxsize=CACHE_MAX):
        self.maxsize = maxsize
        self._d: OrderedDict = OrderedDict()
        self._by_dv: dict = {}
        self.hits = 0
        self.misses = 0

    def clear(self):
        self._d.clear()
        self._by_dv.clear()

    def __len__(self):
        return len(self._d)

    def get(self, key):
        e = self._d.get(key)
        if e is None:
            self.misses += 1
            return None
        if not e.valid():
            self._drop(key)
            self.misses += 1
            return None
        self.hits += 1
        return e.value

    def put(self, key, dvs, value):
        if len(self._d) >= self.maxsize:
            old, _ = self._d.popitem(last=False)
            self._unindex(old)
        handles = [h for dv in dvs for h in dv.storage]
        self._d[key] = _Entry([weakref.ref(dv) for dv in dvs], handles, value)
        for dv in dvs:
            keys = self._by_dv.get(id(dv))
            if keys is None:
                keys = self._by_dv[id(dv)] = set()
                # drop every plan of this vector when it dies (the entry holds its storage)
                weakref.finalize(dv, _evict_dv, weakref.ref(self), id(dv))
            keys.add(key)

    def _drop(self, key):
        if self._d.pop(key, None) is not None:
            self._unindex(key)

    def _unindex(self, key):
        for keys in self._by_dv.values():
            keys.discard(key)

    def evict_dv(self, dv_id):
        for key in self._by_dv.pop(dv_id, ()):
            self._d.pop(key, None)


def _evict_dv(cache_ref, dv_id):
    cache = cache_ref()
    if cache is not None:
        cache.evict_dv(dv_id)


CACHE = PlanCache()


_TYPES = None


def _types():
    global _TYPES
    if _TYPES is None:
        from .containers import DistributedVector
        from . import views

        _TYPES = (DistributedVector, views.TransformView, views.ZipView, views.TakeView, views.DropView,
                  views.IotaView)
    return _TYPES


def view_key(r, dvs):
    """Structural key of range r (appending its DistributedVectors to dvs), or None."""
    DistributedVector, TransformView, ZipView, TakeView, DropView, IotaView = _TYPES or _types()
    t = type(r)
    if t is DistributedVector:
        dvs.append(r)
        return ("dv", id(r))
    if t is TransformView:
        fk = expr._fn_key(r.fn)
        if fk is None:
            return None
        b = view_key(r.base, dvs)
        return None if b is None else ("tf", fk, b)
    if t is ZipView:
        parts = []
        for b in r.bases:
            k = view_key(b, dvs)
            if k is None:
                return None
            parts.append(k)
        return ("zip", r.mode, r.n, tuple(parts))
    if t is TakeView or t is DropView:
        b = view_key(r.base, dvs)
        return None if b is None else ("trim", r.start, r.stop, b)
    if t is IotaView:
        return ("iota", r.start, r.n)
    return None


def lookup(kind, r, extra=()):
    """(key, dvs, cached value or None); key is None when r cannot be cached."""
    if not _ENABLED:
        return None, None, None
    dvs = []
    k = view_key(r, dvs)
    if k is None:
        return None, None, None
    key = (kind, k, extra)
    return key, dvs, CACHE.get(key)


def store(key, dvs, value):
    if key is not None:
        CACHE.put(key, dvs, value)
    return value

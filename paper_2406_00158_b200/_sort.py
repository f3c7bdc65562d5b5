"""Distributed sample sort across GPUs (reference algorithms.py:315-432, paper Alg. 5).

The reference's phases, each mapped to device work on the segments' own GPUs:

  1. local sort of every segment           LSD radix sort in place (drk_sort_keys /
                                            drk_sort_pairs for a key function), per GPU stream
  2. P-1 evenly spaced samples per segment drk_gather of the sample positions, D2H (tiny)
  3. splitters from the pooled samples     host (P·(P-1) values, like the reference's driver)
  4. counts per (segment, chunk)           drk_sort_bounds: P-1 binary searches per sorted run
  5. redistribution into per-locale chunks peer copies over NVLink, pulled by the chunk's GPU
  6. sort of every chunk                    LSD radix sort (stable: runs arrive in segment order)
  7. chunks swept back over the segments    peer copies, pulled by the segment's GPU

Ordering between GPUs is by CUDA events (a stream waits for the phase before it on every
other GPU); the host blocks only for the samples and the counts.  With a key function the
keys travel with the values, and the chunk sort is a stable pair sort, so equal keys keep
their global order exactly as the reference's `np.argsort(kind="stable")` on the chunk
assembled in segment order does.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib, expr, kernels
from .kernels import Launch, run_map
from .runtime import await_pending, torch, torch_dtype


def _sorted_positions(m: int, p: int):
    """Sample positions of a sorted run of m elements (reference algorithms.py:349-356)."""
    if m < p - 1:
        return list(range(m))
    return [(j + 1) * m // p for j in range(p - 1)]


class _Run:
    """One live segment during the sort: its values, its key buffer and its device."""

    __slots__ = ("seg", "state", "vals", "keys", "m")

    def __init__(self, seg, state, vals, keys):
        self.seg, self.state, self.vals, self.keys, self.m = seg, state, vals, keys, len(seg)


def _key_node(key, T):
    node = expr.trace_cached(key, expr.leaf(0, T), ("sortkey", T.str))
    if node is None or isinstance(node, tuple):
        raise TypeError("sort key must return one value per element")
    K = np.dtype(node.dtype)
    if K not in _lib.SORT_DTYPE_CODE:
        K2 = np.dtype(np.int32 if K.kind == "b" else np.float64)
        node, K = expr.cast(node, K2), K2
    return node, K


def _scratch(st, nbytes):
    t = torch()
    with t.cuda.stream(st.stream):
        return t.empty(max(1, int(nbytes)), dtype=t.uint8, device=st.device)


def _sort_buffer(st, code, keys, n, vals=None, vcode=None):
    """Sort `keys` (n elements on st's GPU) in place; with `vals`, stably permute them alongside
    (through an int64 index permutation).  Returns the temporaries to keep alive."""
    t = torch()
    need = ctypes.c_size_t(0)
    with t.cuda.stream(st.stream):
        kalt = t.empty_like(keys)
    if vals is None:
        _lib.call("drk_sort_keys", code, keys.data_ptr(), kalt.data_ptr(), n, None, ctypes.byref(need), st.index,
                  st.handle)
        scratch = _scratch(st, need.value)
        _lib.call("drk_sort_keys", code, keys.data_ptr(), kalt.data_ptr(), n, scratch.data_ptr(), ctypes.byref(need),
                  st.index, st.handle)
        return [kalt, scratch]
    with t.cuda.stream(st.stream):
        idx = t.empty(n, dtype=t.int64, device=st.device)
        idx_alt = t.empty(n, dtype=t.int64, device=st.device)
        valt = t.empty_like(vals)
    _lib.call("drk_iota", _lib.I64, idx.data_ptr(), n, 0, st.index, st.handle)
    _lib.call("drk_sort_pairs", code, keys.data_ptr(), kalt.data_ptr(), idx.data_ptr(), idx_alt.data_ptr(), n, None,
              ctypes.byref(need), st.index, st.handle)
    scratch = _scratch(st, need.value)
    _lib.call("drk_sort_pairs", code, keys.data_ptr(), kalt.data_ptr(), idx.data_ptr(), idx_alt.data_ptr(), n,
              scratch.data_ptr(), ctypes.byref(need), st.index, st.handle)
    _lib.call("drk_gather", vcode, valt.data_ptr(), vals.data_ptr(), idx.data_ptr(), n, st.index, st.handle)
    _lib.call("drk_memcpy_async", vals.data_ptr(), valt.data_ptr(), n * vals.element_size(), st.index, st.handle)
    return [kalt, idx, idx_alt, valt, scratch]


def _fence(states):
    """Every stream in `states` waits for the work enqueued so far on all of them."""
    t = torch()
    evs = []
    for st in states:
        ev = t.cuda.Event()
        ev.record(st.stream)
        evs.append((st, ev))
    for st in states:
        for other, ev in evs:
            if other is not st:
                st.stream.wait_event(ev)


def sample_sort(rt, segs, key=None) -> None:
    """In-place distributed sample sort of the VectorSegments `segs` (all of one dtype)."""
    t = torch()
    P = len(segs)
    live = [s for s in segs if len(s)]
    T = np.dtype(live[0].dtype)
    vcode = _lib.sort_dtype_code(T)
    for s in live:
        await_pending(rt.state_of(s.rank), [s.handle])
    states = list({rt.state_of(s.rank).index: rt.state_of(s.rank) for s in segs}.values())
    keep = []

    # views of the segment storage as device tensors
    def seg_tensor(s):
        return s.handle.span()[s.start: s.start + len(s)]

    # ---- 1. local sort (keys computed on the device when a key function is given)
    if key is not None:
        node, K = _key_node(key, T)
    else:
        node, K = None, T
    kcode = _lib.sort_dtype_code(K)
    runs = []
    for s in live:
        st = rt.state_of(s.rank)
        vals = seg_tensor(s)
        if node is None:
            keys = vals
            keep += _sort_buffer(st, kcode, keys, len(s))
        else:
            from .algorithms import _DeviceTarget

            with t.cuda.stream(st.stream):
                keys = t.empty(len(s), dtype=torch_dtype(K), device=st.device)
            run_map([(_DeviceTarget(keys, K, st.index), node)], [kernels._TensorLeaf(vals, T, len(s))], len(s),
                    Launch(st))
            keep += _sort_buffer(st, kcode, keys, len(s), vals, vcode)
        runs.append(_Run(s, st, vals, keys))

    # ---- 2./3. samples -> splitters (host, P*(P-1) keys)
    host_samples = []
    for r in runs:
        pos = _sorted_positions(r.m, P)
        if not pos:
            continue
        with t.cuda.stream(r.state.stream):
            pos_d = t.tensor(pos, dtype=t.int64).to(r.state.device, non_blocking=True)
            smp = t.empty(len(pos), dtype=torch_dtype(K), device=r.state.device)
        _lib.call("drk_gather", kcode, smp.data_ptr(), r.keys.data_ptr(), pos_d.data_ptr(), len(pos), r.state.index,
                  r.state.handle)
        host = t.empty(len(pos), dtype=torch_dtype(K), pin_memory=True)
        _lib.call("drk_memcpy_async", host.data_ptr(), smp.data_ptr(), len(pos) * K.itemsize, r.state.index,
                  r.state.handle)
        keep += [pos_d, smp]
        host_samples.append(host)
    for st in states:
        st.synchronize()
    pool = np.sort(np.concatenate([h.numpy() for h in host_samples]), kind="stable")
    m = len(pool)
    split = np.ascontiguousarray(pool[[(j + 1) * m // P for j in range(P - 1)]])

    # ---- 4. counts[k][j]: elements of run k that go to chunk j
    bounds_host = []
    for r in runs:
        with t.cuda.stream(r.state.stream):
            split_d = t.from_numpy(split).to(r.state.device, non_blocking=False)
            bnd = t.empty(P - 1, dtype=t.int64, device=r.state.device)
        _lib.call("drk_sort_bounds", kcode, r.keys.data_ptr(), r.m, split_d.data_ptr(), P - 1, bnd.data_ptr(),
                  r.state.index, r.state.handle)
        host = t.empty(P - 1, dtype=t.int64, pin_memory=True)
        _lib.call("drk_memcpy_async", host.data_ptr(), bnd.data_ptr(), (P - 1) * 8, r.state.index, r.state.handle)
        keep += [split_d, bnd]
        bounds_host.append(host)
    for st in states:
        st.synchronize()
    counts = np.zeros((len(runs), P), dtype=np.int64)
    for k, (r, h) in enumerate(zip(runs, bounds_host)):
        b = np.concatenate(([0], h.numpy(), [r.m]))
        counts[k] = np.diff(b)
    sizes = counts.sum(axis=0)
    offsets = np.zeros_like(counts)
    offsets[1:] = np.cumsum(counts, axis=0)[:-1]

    # ---- 5. redistribution: chunk j lives on segs[j]'s GPU and pulls its runs
    _fence(states)
    chunks = []
    for j in range(P):
        st = rt.state_of(segs[j].rank)
        n_j = int(sizes[j])
        with t.cuda.stream(st.stream):
            cv = t.empty(n_j, dtype=torch_dtype(T), device=st.device)
            ck = cv if node is None else t.empty(n_j, dtype=torch_dtype(K), device=st.device)
        for k, r in enumerate(runs):
            c = int(counts[k, j])
            if not c:
                continue
            lo, w = int(counts[k, :j].sum()), int(offsets[k, j])
            _lib.call("drk_memcpy_async", cv.data_ptr() + w * T.itemsize, r.vals.data_ptr() + lo * T.itemsize,
                      c * T.itemsize, st.index, st.handle)
            if node is not None:
                _lib.call("drk_memcpy_async", ck.data_ptr() + w * K.itemsize, r.keys.data_ptr() + lo * K.itemsize,
                          c * K.itemsize, st.index, st.handle)
        # ---- 6. chunk sort (stable; runs sit in segment order)
        if n_j > 1:
            keep += _sort_buffer(st, kcode, ck, n_j, None if node is None else cv, vcode)
        chunks.append((st, cv))
        keep.append(ck)

    # ---- 7. sweep the chunks back over the segments, pulled by each segment's GPU
    _fence(states)
    pos = 0
    starts = np.concatenate(([0], np.cumsum(sizes)))
    for r in runs:
        # global range [pos, pos + m) of the sorted sequence lands in this segment
        lo, hi = pos, pos + r.m
        for j in range(P):
            a, b = max(lo, int(starts[j])), min(hi, int(starts[j + 1]))
            if a >= b:
                continue
            _, cv = chunks[j]
            _lib.call("drk_memcpy_async", r.vals.data_ptr() + (a - lo) * T.itemsize,
                      cv.data_ptr() + (a - int(starts[j])) * T.itemsize, (b - a) * T.itemsize, r.state.index,
                      r.state.handle)
        pos = hi
    for st in states:
        st.synchronize()
    del keep, chunks

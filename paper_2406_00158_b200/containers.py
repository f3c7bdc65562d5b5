"""Distributed vector whose segments live in GPU memory.

Mirrors the reference DistributedVector / VectorSegment
(/root/reference/pkg/src/segrange/containers.py:28-206): block partition into ceil(n/P)
segments (or an explicit partition), one allocation per segment on its locale, O(1) index
arithmetic for uniform blocks, from_numpy / to_numpy / like_distribution, global
get/set.  Segment storage is device memory of the locale's GPU; ``eval_array`` and
``local_span`` return device tensors (views of that memory, no copy).

Host <-> device traffic (from_numpy / to_numpy) goes through pinned buffers with
asynchronous copies on the segment streams, so segments on different GPUs transfer
concurrently.
"""

from __future__ import annotations

import numpy as np

from . import _lib
from .core import Distribution
from .runtime import torch, torch_dtype
from .views import Leaf, Lowered, Target
from . import expr

_PIN_THRESHOLD = 1 << 20  # bytes; smaller transfers use pageable memory


def is_pinned(array: np.ndarray) -> bool:
    try:
        return bool(torch().from_numpy(array).is_pinned())
    except Exception:
        return False


def pinned_empty(n: int, dtype) -> np.ndarray:
    """A numpy array backed by page-locked host memory (DMA-able at full PCIe speed)."""
    t = torch().empty(int(n), dtype=torch_dtype(dtype), pin_memory=True)
    return t.numpy()


class VectorSegment:
    """Elements [start, start+length) of one storage handle (containers.py:28-83)."""

    __slots__ = ("handle", "start", "length")
    writable = True

    def __init__(self, handle, start: int, length: int):
        self.handle = handle
        self.start = start
        self.length = length

    @property
    def rank(self):
        return self.handle.locale

    @property
    def runtime(self):
        return self.handle.runtime

    @property
    def dtype(self):
        return self.handle.dtype

    def __len__(self):
        return self.length

    def _check(self, i: int) -> int:
        if not 0 <= i < self.length:
            raise IndexError(f"index {i} out of range [0, {self.length})")
        return i

    def get(self, i: int):
        return self.handle.read(self.start + self._check(i))

    def set(self, i: int, value):
        self.handle.write(self.start + self._check(i), value)

    def __iter__(self):
        host = self.to_numpy()
        for i in range(self.length):
            yield host[i].item()

    def local_span(self):
        return self.handle.span()[self.start : self.start + self.length]

    def eval_array(self):
        """The segment as a device tensor (a view of its storage).  In-flight asynchronous
        transfers of the storage are ordered before any later work on its stream."""
        rt = self.handle.runtime
        if rt.backend == "cuda":
            from .runtime import await_pending

            await_pending(rt.state_of(self.handle.locale), [self.handle])
        return self.local_span()

    def store_array(self, values):
        """Overwrite the segment from a device tensor, host array or scalar."""
        from .runtime import await_pending

        span = self.local_span()
        rt = self.handle.runtime
        rt._check_compute()
        st = rt.state_of(self.handle.locale)
        # an upload still writing, or a download still reading, this storage lands first
        await_pending(st, [self.handle])
        t = torch()
        with t.cuda.stream(st.stream):
            if isinstance(values, t.Tensor):
                span.copy_(values)
            else:
                arr = np.asarray(values)
                span.copy_(t.from_numpy(np.ascontiguousarray(arr.astype(self.handle.dtype, copy=False)))
                           if arr.ndim else t.tensor(arr.item()).to(span.dtype))

    def to_numpy(self) -> np.ndarray:
        out = np.empty(self.length, dtype=self.handle.dtype)
        if self.length:
            from .runtime import await_pending

            rt = self.handle.runtime
            rt._check_compute()
            st = rt.state_of(self.handle.locale)
            await_pending(st, [self.handle])
            _lib.call("drk_memcpy_async", out.ctypes.data, self.data_ptr(), out.nbytes, st.index, st.handle)
            st.synchronize()
        return out

    def data_ptr(self) -> int:
        return self.handle.data_ptr() + self.start * self.handle.dtype.itemsize

    def slice(self, start: int, length: int) -> "VectorSegment":
        if not (0 <= start and start + length <= self.length):
            raise IndexError(f"slice [{start}, {start + length}) outside segment of {self.length}")
        return VectorSegment(self.handle, self.start + start, length)

    def _lower(self):
        lf = Leaf("array", self.length, self.handle.dtype, handle=self.handle, start=self.start)
        tgt = Target(self.handle, self.start, self.length)
        return Lowered([lf], expr.leaf(0, self.handle.dtype), tgt, self.length, self.rank)

    def __repr__(self):
        return f"VectorSegment(rank={self.rank}, length={self.length})"


class DistributedVector:
    """A 1-D array block-partitioned over the runtime's locales (containers.py:86-206).

    ``partition`` overrides the default with a segment count or explicit lengths.  Global
    indexing and iteration are conveniences (each access is a device round trip); bulk
    work goes through segments() and the algorithms."""

    def __init__(self, runtime, n: int, init=0.0, dtype=None, partition=None):
        if n < 0:
            raise ValueError("vector length must be non-negative")
        if dtype is None:
            dtype = np.result_type(init)
        self.runtime = runtime
        self.n = n
        self.dtype = np.dtype(dtype)
        self.distribution = self._make_distribution(n, partition, runtime.locale_count)
        self.storage = [runtime.allocate(d.rank, d.length, self.dtype) for d in self.distribution.descriptors]
        if n and runtime.backend == "cuda" and np.any(np.asarray(init) != 0):
            from . import algorithms

            algorithms.fill(self, init)
        self._block = -(-n // runtime.locale_count) if (partition is None and n > 0) else None
        self._starts = np.array([d.global_offset for d in self.distribution.descriptors], dtype=np.int64)

    @staticmethod
    def _make_distribution(n, partition, locale_count) -> Distribution:
        if partition is None:
            return Distribution.block(n, locale_count, locale_count)
        if isinstance(partition, (int, np.integer)):
            return Distribution.block(n, int(partition), locale_count)
        dist = Distribution.from_lengths(partition, locale_count)
        if dist.total_length != n:
            raise ValueError(f"partition lengths sum to {dist.total_length}, expected {n}")
        return dist

    @classmethod
    def from_numpy(cls, runtime, array, partition=None) -> "DistributedVector":
        array = np.asarray(array)
        if array.ndim != 1:
            raise ValueError("from_numpy expects a 1-D array")
        vec = cls.__new__(cls)
        vec._init_empty(runtime, len(array), array.dtype, cls._make_distribution(len(array), partition,
                                                                                  runtime.locale_count),
                        partition is None)
        if runtime.backend == "cuda":
            vec.upload(array)
        return vec

    @classmethod
    def like_distribution(cls, runtime, distribution: Distribution, dtype) -> "DistributedVector":
        """A fresh zero vector with exactly this distribution."""
        vec = cls.__new__(cls)
        vec._init_empty(runtime, distribution.total_length, dtype, distribution, False)
        return vec

    def _init_empty(self, runtime, n, dtype, distribution, uniform):
        self.runtime = runtime
        self.n = n
        self.dtype = np.dtype(dtype)
        self.distribution = distribution
        self.storage = [runtime.allocate(d.rank, d.length, self.dtype) for d in distribution.descriptors]
        self._block = -(-n // runtime.locale_count) if (uniform and n > 0) else None
        self._starts = np.array([d.global_offset for d in distribution.descriptors], dtype=np.int64)

    # -- host <-> device -----------------------------------------------------------------
    def upload(self, array: np.ndarray, wait: bool = True):
        """Copy a host array of length n into the segments.

        wait=True: synchronous (returns None).  wait=False: asynchronous on each GPU's
        host->device copy stream, returning a TransferTicket; the array must stay alive and
        unchanged until then.  Kernels that later touch the vector wait for the copy on
        the device (no host sync), and the copy itself waits for work already enqueued on
        the vector, so transfers overlap compute and the opposite PCIe direction."""
        from .runtime import TransferTicket, await_pending

        array = np.asarray(array)
        if array.shape != (self.n,):
            raise ValueError(f"upload expects shape ({self.n},), got {array.shape}")
        if array.dtype != self.dtype:
            array = array.astype(self.dtype)
        rt = self.runtime
        if rt.backend != "cuda":
            raise RuntimeError("backend='meta' vectors hold no data")
        array = np.ascontiguousarray(array)
        pinned = array.nbytes >= _PIN_THRESHOLD and is_pinned(array)
        staged, events, used = [], [], {}
        for h, d in zip(self.storage, self.distribution.descriptors):
            if not d.length:
                continue
            st = rt.state_of(d.rank)
            src = array[d.global_offset : d.global_offset + d.length]
            if not pinned and src.nbytes >= _PIN_THRESHOLD:
                buf = pinned_empty(d.length, self.dtype)
                buf[...] = src
                staged.append(buf)
                src = buf
            if wait:
                await_pending(st, [h])
                _lib.call("drk_memcpy_async", h.data_ptr(), src.ctypes.data, src.nbytes, st.index, st.handle)
                used[st.index] = st
            else:
                cs = st.copy_stream("h2d")
                cs.wait_event(st.compute_event())  # earlier kernels on this vector finish first
                for ev in h._pending:
                    cs.wait_event(ev)
                _lib.call("drk_memcpy_async", h.data_ptr(), src.ctypes.data, src.nbytes, st.index,
                          int(cs.cuda_stream))
                ev = torch().cuda.Event()
                ev.record(cs)
                h._pending = [ev]
                events.append(ev)
        if wait:
            for st in used.values():
                st.synchronize()
            return None
        return TransferTicket(events, keep=(array, staged))

    def to_numpy(self, out: np.ndarray | None = None, wait: bool = True):
        """Gather all segments into a host array.

        wait=True returns the array.  wait=False enqueues the device->host copies on each
        GPU's d2h copy stream after the work already enqueued on the vector and returns
        (array, TransferTicket); the array is valid after ticket.wait().  Kernels that later
        overwrite the vector wait for the copy on the device."""
        from .runtime import TransferTicket, await_pending

        rt = self.runtime
        if out is None:
            out = np.empty(self.n, dtype=self.dtype)
        elif out.shape != (self.n,) or out.dtype != self.dtype:
            raise ValueError("to_numpy: out has the wrong shape or dtype")
        if self.n == 0:
            return out if wait else (out, TransferTicket([]))
        rt._check_compute()
        direct = out.nbytes >= _PIN_THRESHOLD and is_pinned(out)
        pending, events, used = [], [], {}
        for h, d in zip(self.storage, self.distribution.descriptors):
            if not d.length:
                continue
            st = rt.state_of(d.rank)
            dst = out[d.global_offset : d.global_offset + d.length]
            if not direct and dst.nbytes >= _PIN_THRESHOLD:
                buf = pinned_empty(d.length, self.dtype)
                pending.append((dst, buf))
                dst = buf
            if wait:
                await_pending(st, [h])
                _lib.call("drk_memcpy_async", dst.ctypes.data, h.data_ptr(), dst.nbytes, st.index, st.handle)
                used[st.index] = st
            else:
                cs = st.copy_stream("d2h")
                cs.wait_event(st.compute_event())
                for ev in h._pending:
                    cs.wait_event(ev)
                _lib.call("drk_memcpy_async", dst.ctypes.data, h.data_ptr(), dst.nbytes, st.index,
                          int(cs.cuda_stream))
                ev = torch().cuda.Event()
                ev.record(cs)
                h._pending = [ev]
                events.append(ev)

        def finish():
            for dst, buf in pending:
                dst[...] = buf

        if wait:
            for st in used.values():
                st.synchronize()
            finish()
            return out
        return out, TransferTicket(events, keep=(out,), finish=finish)

    # -- segments / indexing -----------------------------------------------------------------
    def segments(self) -> list:
        return [VectorSegment(h, 0, d.length) for h, d in zip(self.storage, self.distribution.descriptors)]

    def __len__(self):
        return self.n

    def _locate(self, i: int):
        if not 0 <= i < self.n:
            raise IndexError(f"index {i} out of range [0, {self.n})")
        if self._block is not None:
            k = i // self._block
            return k, i - k * self._block
        k = int(np.searchsorted(self._starts, i, side="right")) - 1
        return k, i - int(self._starts[k])

    def __getitem__(self, i: int):
        k, off = self._locate(i)
        return self.storage[k].read(off)

    def __setitem__(self, i: int, value):
        k, off = self._locate(i)
        self.storage[k].write(off, value)

    def __iter__(self):
        yield from self.to_numpy().tolist()

    def __repr__(self):
        return f"DistributedVector(n={self.n}, dtype={self.dtype}, segments={self.distribution.lengths()})"

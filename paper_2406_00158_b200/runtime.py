"""Single-process multi-GPU runtime: locales are CUDA devices, tasks are stream work.

Mirrors the reference Runtime (/root/reference/pkg/src/segrange/runtime.py) — allocate,
submit, wait_all, map_segments, copy, copy_async, run_transfer, close — with its one
ordering promise kept: work submitted to a locale runs in submission order.  Here each
locale maps to a CUDA device (locale i -> devices[i % len(devices)]) and each device has
one in-order stream owned by the runtime, so per-locale FIFO holds by construction and
``wait_all`` is a stream/event synchronisation (the visibility barrier).

Storage is zero-initialised device memory (torch tensors are the storage handle, so the
caching allocator and pinned host buffers come for free); every element-wise, reduce
and scan step runs in libdrk.so (include/drk.h) on the segment's stream.

``backend="meta"`` builds a runtime whose storage has shape and dtype but no memory (torch
meta tensors): all segment algebra works, any data access raises.  It exists so host
logic can be exercised on machines without a GPU; it never computes.
"""

from __future__ import annotations

import ctypes
import itertools
import os
import threading
import weakref

import numpy as np

from . import _lib
from . import core
from .core import LocaleId

LOCALES_ENV = "SEGRANGE_LOCALES"
LOCALE_CAP = 16

_torch = None


def torch():
    global _torch
    if _torch is None:
        import torch as t

        _torch = t
    return _torch


def torch_dtype(dtype):
    t = torch()
    return {
        np.dtype(np.float32): t.float32,
        np.dtype(np.float64): t.float64,
        np.dtype(np.int32): t.int32,
        np.dtype(np.int64): t.int64,
        np.dtype(np.uint8): t.uint8,
        np.dtype(np.bool_): t.bool,
        np.dtype(np.int16): t.int16,
        np.dtype(np.int8): t.int8,
        np.dtype(np.float16): t.float16,
        np.dtype(np.uint64): t.uint64,
        np.dtype(np.uint32): t.uint32,
    }[np.dtype(dtype)]


class AggregateTaskError(RuntimeError):
    """One or more tasks of a wait_all failed; ``failures`` = [(ticket index, exc)]
    (reference runtime.py:32-43)."""

    def __init__(self, failures):
        self.failures = list(failures)
        idx = ", ".join(str(i) for i, _ in self.failures)
        msgs = "; ".join(f"[{i}] {type(e).__name__}: {e}" for i, e in self.failures)
        super().__init__(f"{len(self.failures)} task(s) failed (indices {idx}): {msgs}")


# how reduce combines per-segment partials across GPUs (algorithms.py:146-149, the driver's
# ascending fold): "host" — every GPU stores its partials into mapped pinned memory and the
# host folds them; "device" — the first GPU folds them from peer memory (NVLink) and stores
# one result; "nccl" — an NCCL all-gather of the partials, then every GPU folds them in
# segment order (all-reduce semantics, the result on every GPU).  Same value every way.
# "fused" — the combine inside the reduce kernels: each segment's partial goes into a slot on
# the first GPU (NVLink peer stores), and the kernel CTA that finishes last folds them and
# stores the result into mapped host memory (drk_reduce_fused): one kernel per GPU, one wait.
REDUCE_COMBINES = ("host", "device", "nccl", "fused")

_EPOCHS = itertools.count(1)  # completion-word epochs (DeviceState.completion_flags)


def default_locale_count() -> int:
    """SEGRANGE_LOCALES if set, else the number of visible GPUs (at least 1), capped at 16."""
    env = os.environ.get(LOCALES_ENV)
    if env:
        n = int(env)
        if n < 1:
            raise ValueError(f"{LOCALES_ENV} must be at least 1, got {n}")
        return n
    try:
        g = torch().cuda.device_count()
    except Exception:  # pragma: no cover
        g = 0
    return max(1, min(g, LOCALE_CAP))


class DeviceState:
    """Per-GPU resources: the in-order stream shared by the device's locales, reduce and
    scan scratch, and device/pinned-host slots for per-segment results."""

    RESULT_BYTES = 8

    def __init__(self, index: int, backend: str):
        self.index = index
        self.backend = backend
        self._scan_scratch = None
        self._result_slots = 0
        self._results = None
        self._host_results = None
        if backend == "cuda":
            t = torch()
            self.device = t.device("cuda", index)
            self.stream = t.cuda.Stream(device=self.device)
            self.handle = int(self.stream.cuda_stream)
            with t.cuda.stream(self.stream):
                self.reduce_scratch = t.zeros(
                    int(_lib.load().drk_reduce_scratch_bytes()), dtype=t.uint8, device=self.device
                )
            self.ensure_results(64)
        else:
            self.device = None
            self.stream = None
            self.handle = 0
            self.reduce_scratch = None

    # -- scratch ---------------------------------------------------------
    def scan_scratch(self, nbytes: int, which: int = 0):
        """Scan scratch buffer `which` (0 or 1: consecutive scans of a chained launch
        alternate, kernels.run_scan)."""
        t = torch()
        if self._scan_scratch is None:
            self._scan_scratch = [None, None]
        buf = self._scan_scratch[which]
        if buf is None or buf.numel() < nbytes:
            with t.cuda.stream(self.stream):
                # zero once: tile descriptors are epoch-tagged, the ticket counter self-resets
                buf = t.zeros(int(nbytes * 1.25) + 4096, dtype=t.uint8, device=self.device)
            self._scan_scratch[which] = buf
        return buf

    def reduce_batch_scratch(self, nseg: int):
        """Scratch of a batched reduction over nseg segments (drk_reduce_batch): nseg reduce
        scratch blocks, zeroed once (their tickets reset themselves)."""
        t = torch()
        per = int(_lib.load().drk_reduce_scratch_bytes())
        buf = getattr(self, "_reduce_batch_scratch", None)
        if buf is None or buf.numel() < nseg * per:
            with t.cuda.stream(self.stream):
                buf = t.zeros(max(nseg, 4) * per, dtype=t.uint8, device=self.device)
            self._reduce_batch_scratch = buf
        return buf

    def ensure_results(self, slots: int):
        if slots <= self._result_slots:
            return
        t = torch()
        slots = max(slots, 2 * self._result_slots)
        with t.cuda.stream(self.stream):
            self._results = t.zeros(slots * self.RESULT_BYTES, dtype=t.uint8, device=self.device)
        self._host_results = t.zeros(slots * self.RESULT_BYTES, dtype=t.uint8, pin_memory=True)
        self._host_results_np = self._host_results.numpy()
        dev = ctypes.c_void_p()
        _lib.call("drk_mapped_ptr", self._host_results.data_ptr(), ctypes.byref(dev))
        self._host_results_dev = int(dev.value)
        self._result_slots = slots

    def combine_slots(self, nbytes: int):
        """Device buffer of the cross-GPU reduce combine (partials and the all-gathered
        partials, algorithms._ReducePlan.fold_on_device), kept apart from the scan's result
        slots."""
        buf = getattr(self, "_combine", None)
        if buf is None or buf.numel() < nbytes:
            t = torch()
            with t.cuda.stream(self.stream):
                buf = t.zeros(max(nbytes, 4096), dtype=t.uint8, device=self.device)
            self._combine = buf
        return buf

    def flag_ptrs(self):
        """(host address, device address) of this GPU's completion words (allocated once)."""
        if getattr(self, "_flags", None) is None:
            self.completion_flags()
        return self._flags_host, self._flags_dev

    def completion_flags(self):
        """(host address, device address) of DRK_RED_SEGS 8-byte completion words in mapped
        pinned memory, and the next epoch to wait for (drk_reduce_batch_ex / drk_wait_flags)."""
        f = getattr(self, "_flags", None)
        if f is None:
            t = torch()
            f = self._flags = t.zeros(_lib.RED_SEGS, dtype=t.int64, pin_memory=True)
            dev = ctypes.c_void_p()
            _lib.call("drk_mapped_ptr", f.data_ptr(), ctypes.byref(dev))
            self._flags_host, self._flags_dev = f.data_ptr(), int(dev.value)
        # one process-wide sequence: a completion word never sees the same epoch twice, even
        # when one launch writes the words of several GPUs with a shared epoch
        return self._flags_host, self._flags_dev, next(_EPOCHS)

    def result_ptr(self, slot: int) -> int:
        return self._results.data_ptr() + slot * self.RESULT_BYTES

    def result_dev_ptr(self, slot: int) -> int:
        return self.result_ptr(slot)

    def host_result_dev_ptr(self, slot: int) -> int:
        """Device address of host result slot `slot` (mapped pinned memory): reductions
        store their result there directly (fetch with fetch_host_results)."""
        return self._host_results_dev + slot * self.RESULT_BYTES

    def fetch_host_results(self, slots: int) -> np.ndarray:
        """Wait for the stream, then the raw bytes of host result slots [0, slots)."""
        self.synchronize()
        return self._host_results_np[: slots * self.RESULT_BYTES].copy()

    def fetch_results(self, slots: int) -> np.ndarray:
        """Copy result slots [0, slots) to pinned host memory and wait (raw bytes)."""
        nbytes = slots * self.RESULT_BYTES
        # stored by a kernel into mapped pinned memory: no copy engine, so this never waits
        # behind a bulk download running on the d2h stream
        _lib.call("drk_readback", self._host_results.data_ptr(), self._results.data_ptr(), nbytes,
                  self.index, self.handle)
        self.synchronize()
        return self._host_results.numpy()[:nbytes].copy()

    def synchronize(self):
        if self.backend == "cuda":
            _lib.call("drk_stream_synchronize", self.index, self.handle)

    def results_view(self) -> np.ndarray:
        """The mapped host result slots (valid after synchronize())."""
        return self._host_results_np

    # -- asynchronous host transfers ---------------------------------------------
    def copy_stream(self, direction: str):
        """Dedicated stream for host->device ("h2d") or device->host ("d2h") copies, so
        transfers in both PCIe directions overlap each other and the compute stream."""
        name = "_" + direction + "_stream"
        s = getattr(self, name, None)
        if s is None:
            s = torch().cuda.Stream(device=self.device)
            setattr(self, name, s)
        return s

    def compute_event(self):
        """An event recorded now on the compute stream."""
        ev = torch().cuda.Event()
        ev.record(self.stream)
        return ev


def await_pending(state, handles):
    """Make the compute stream of `state` wait for in-flight asynchronous transfers of any
    of `handles` (uploads writing them, downloads still reading them)."""
    for h in handles:
        pend = getattr(h, "_pending", None)
        if pend:
            for ev in pend:
                state.stream.wait_event(ev)
            pend.clear()


class TransferTicket:
    """Completion of an asynchronous upload / download; wait() blocks until it is done
    (and runs the host-side finisher of staged copies, if any)."""

    __slots__ = ("_events", "_keep", "_finish", "_done")

    def __init__(self, events, keep=(), finish=None):
        self._events = list(events)
        self._keep = keep
        self._finish = finish
        self._done = False

    def wait(self):
        if not self._done:
            for ev in self._events:
                ev.synchronize()
            if self._finish is not None:
                self._finish()
            self._done = True
            self._keep = ()
        return None

    def done(self) -> bool:
        return self._done or all(ev.query() for ev in self._events)


class StorageHandle:
    """Zero-initialised device storage owned by one locale (reference runtime.py:61-105).

    ``span()`` returns the 1-D device tensor; ``read``/``write`` move single elements
    between host and device (convenience only, synchronous)."""

    __slots__ = ("locale", "length", "dtype", "runtime", "_tensor", "_freed", "_pending", "__weakref__")

    def __init__(self, runtime, locale: LocaleId, length: int, dtype, tensor):
        self.runtime = runtime
        self.locale = locale
        self.length = length
        self.dtype = np.dtype(dtype)
        self._tensor = tensor
        self._freed = False
        self._pending = []  # events of in-flight async transfers touching this storage

    def span(self):
        if self._freed:
            raise RuntimeError("use after free: storage handle was released")
        return self._tensor

    @property
    def device_index(self) -> int:
        return self.runtime.device_of(self.locale)

    def data_ptr(self) -> int:
        return self.span().data_ptr()

    def read(self, i: int):
        t = self.span()
        self.runtime._check_compute()
        st = self.runtime.state_of(self.locale)
        await_pending(st, [self])
        st.synchronize()
        return t[i].item()

    def write(self, i: int, value):
        t = self.span()
        self.runtime._check_compute()
        st = self.runtime.state_of(self.locale)
        await_pending(st, [self])
        buf = np.asarray([value]).astype(self.dtype)
        host = torch().from_numpy(buf)
        with torch().cuda.stream(st.stream):
            t[i : i + 1].copy_(host)
        st.synchronize()

    def free(self):
        if self._freed:
            raise RuntimeError("double free of storage handle")
        self._freed = True
        self._tensor = self._tensor.new_zeros(0)

    @property
    def freed(self) -> bool:
        return self._freed

    def __len__(self):
        return self.length

    def __repr__(self):
        state = "freed" if self._freed else "live"
        return (f"StorageHandle(locale={self.locale}, device={self.device_index}, length={self.length}, "
                f"dtype={self.dtype}, {state})")


class TaskTicket:
    """Completion token of a submitted task (reference runtime.py:108-127): wait() waits
    for the task's device work and returns its result or re-raises its exception."""

    __slots__ = ("_result", "_exc", "_states", "_done")

    def __init__(self, result=None, exc=None, states=()):
        self._result = result
        self._exc = exc
        self._states = tuple(states)
        self._done = False

    def wait(self, timeout=None):
        if not self._done:
            for st in self._states:
                st.synchronize()
            self._done = True
        if self._exc is not None:
            raise self._exc
        return self._result

    def done(self) -> bool:
        if self._done:
            return True
        return all(st.stream is None or st.stream.query() for st in self._states)

    def exception(self, timeout=None):
        try:
            self.wait(timeout)
        except BaseException:
            pass
        return self._exc


class Runtime:
    """P locales over the process's GPUs, each with an in-order stream.

    ``worker_mode`` is accepted for API compatibility ("threads" or "inline"); both modes
    enqueue on the locale stream from the driver thread, "inline" additionally waits for
    each task.  ``devices`` picks the CUDA devices (default: all visible)."""

    def __init__(self, locale_count: int | None = None, worker_mode: str = "threads", devices=None,
                 backend: str = "cuda", reduce_combine: str | None = None):
        if locale_count is None:
            locale_count = default_locale_count()
        if locale_count < 1:
            raise ValueError(f"locale_count must be at least 1, got {locale_count}")
        if worker_mode not in ("threads", "inline"):
            raise ValueError(f"unknown worker mode {worker_mode!r}")
        if backend not in ("cuda", "meta"):
            raise ValueError(f"unknown backend {backend!r}")
        if reduce_combine is None:
            reduce_combine = os.environ.get("DRK_REDUCE_COMBINE", "host")
        if reduce_combine not in REDUCE_COMBINES:
            raise ValueError(f"unknown reduce_combine {reduce_combine!r} (one of {', '.join(REDUCE_COMBINES)})")
        self.reduce_combine = reduce_combine
        self._comm = None
        self.locale_count = int(locale_count)
        self.worker_mode = worker_mode
        self.backend = backend
        self._closed = False
        self._lock = threading.Lock()
        if backend == "cuda":
            _lib.load()
            t = torch()
            if not t.cuda.is_available():
                raise RuntimeError("no CUDA device is visible; this runtime has no CPU fallback "
                                   "(use backend='meta' for metadata-only work)")
            ndev = t.cuda.device_count()
            devices = list(range(ndev)) if devices is None else [int(d) for d in devices]
            for d in devices:
                if not 0 <= d < ndev:
                    raise ValueError(f"invalid CUDA device {d}; {ndev} visible")
        else:
            devices = [0] if devices is None else [int(d) for d in devices]
        if not devices:
            raise ValueError("need at least one device")
        self.devices = devices
        self._states = {d: DeviceState(d, backend) for d in sorted(set(devices))}
        self._registry = [weakref.WeakSet() for _ in range(self.locale_count)]
        if backend == "cuda" and len(self._states) > 1:
            self._enable_peer_access()

    def _enable_peer_access(self):
        t = torch()
        for a in self._states:
            for b in self._states:
                if a != b and t.cuda.can_device_access_peer(a, b):
                    _lib.call("drk_enable_peer_access", a, b)

    # -- placement ---------------------------------------------------------
    def device_of(self, locale: LocaleId) -> int:
        return self.devices[locale % len(self.devices)]

    def state_of(self, locale: LocaleId) -> DeviceState:
        return self._states[self.device_of(locale)]

    def device_state(self, device: int) -> DeviceState:
        return self._states[device]

    @property
    def device_states(self):
        return list(self._states.values())

    def stream_of(self, locale: LocaleId):
        return self.state_of(locale).stream

    # -- allocation ------------------------------------------------------------
    def allocate(self, locale: LocaleId, length: int, dtype=np.float64) -> StorageHandle:
        self._check_open()
        self._check_locale(locale)
        if length < 0:
            raise ValueError(f"allocation length must be non-negative, got {length}")
        dtype = np.dtype(dtype)
        t = torch()
        st = self.state_of(locale)
        if self.backend == "meta":
            tensor = t.empty(length, dtype=torch_dtype(dtype), device="meta")
        else:
            with t.cuda.stream(st.stream):
                tensor = t.empty(length, dtype=torch_dtype(dtype), device=st.device)
            if length:
                _lib.call("drk_memset_async", tensor.data_ptr(), 0, length * dtype.itemsize, st.index, st.handle)
        h = StorageHandle(self, locale, length, dtype, tensor)
        self._registry[locale].add(h)
        return h

    def live_allocations(self, locale: LocaleId) -> int:
        self._check_locale(locale)
        return len(self._registry[locale])

    # -- tasks -------------------------------------------------------------------
    def submit(self, locale: LocaleId, fn, *args, **kwargs) -> TaskTicket:
        """Run ``fn`` as a task of ``locale``: it executes on the driver thread with the
        locale's device stream current, so the device work it enqueues is ordered after
        everything submitted to that locale before it."""
        self._check_open()
        self._check_locale(locale)
        st = self.state_of(locale)
        prev = core.current_locale()
        core._set_current_locale(locale)
        result = exc = None
        try:
            if self.backend == "cuda":
                t = torch()
                with t.cuda.device(st.index), t.cuda.stream(st.stream):
                    result = fn(*args, **kwargs)
            else:
                result = fn(*args, **kwargs)
        except Exception as e:  # captured in the ticket, like a future
            exc = e
        finally:
            core._set_current_locale(prev)
        ticket = TaskTicket(result, exc, (st,))
        if self.worker_mode == "inline":
            try:
                ticket.wait()
            except Exception:
                pass
        return ticket

    def wait_all(self, tickets) -> list:
        """Results in ticket order; AggregateTaskError names every failed ticket."""
        results, failures = [], []
        for i, tk in enumerate(list(tickets)):
            try:
                results.append(tk.wait())
            except Exception as exc:
                failures.append((i, exc))
        if failures:
            raise AggregateTaskError(failures)
        return results

    def map_segments(self, pairs) -> list:
        return self.wait_all([self.submit(loc, fn) for loc, fn in pairs])

    def synchronize(self):
        for st in self._states.values():
            st.synchronize()

    # -- copies ------------------------------------------------------------------
    def copy(self, src, dst) -> None:
        """Element copy between spans/handles, possibly across devices (NVLink peer copy);
        length/dtype are checked before any write (runtime.py:253-262,324-330)."""
        self.copy_async(src, dst).wait()

    def copy_async(self, src, dst) -> TaskTicket:
        self._check_open()
        s, s_st = self._resolve(src)
        d, d_st = self._resolve(dst)
        _check_copy(s, d)
        st = d_st or s_st
        if st is None:
            d[...] = s  # host to host
            return TaskTicket(None, None, ())
        self._check_compute()
        # asynchronous uploads still writing either side, or downloads still reading the
        # destination, complete before this copy reads or overwrites them
        # (every branch below enqueues the copy on st's stream, or syncs it first)
        await_pending(st, [h for h in (src, dst) if isinstance(h, StorageHandle)])
        t = torch()
        s_t = t.from_numpy(np.ascontiguousarray(s)) if isinstance(s, np.ndarray) else s
        if isinstance(d, np.ndarray):
            host = t.from_numpy(d)
            s_st.synchronize() if s_st else None
            with t.cuda.stream((s_st or st).stream):
                host.copy_(s_t, non_blocking=False)
            return TaskTicket(None, None, ())
        if s_st is not None and s_st is not d_st:
            s_st.synchronize()  # the source's pending writes land before the peer copy
        nbytes = d.numel() * d.element_size()
        if nbytes:
            if isinstance(s, np.ndarray):
                with t.cuda.stream(st.stream):
                    d.copy_(s_t.pin_memory() if nbytes > (1 << 20) else s_t, non_blocking=True)
            else:
                _lib.call("drk_memcpy_async", d.data_ptr(), s_t.data_ptr(), nbytes, st.index, st.handle)
        return TaskTicket(None, None, (st,))

    def run_transfer(self, fn, *args) -> TaskTicket:
        self._check_open()
        try:
            return TaskTicket(fn(*args), None, tuple(self._states.values()))
        except Exception as exc:
            return TaskTicket(None, exc, ())

    def _resolve(self, obj):
        if isinstance(obj, StorageHandle):
            return obj.span(), self.state_of(obj.locale)
        if isinstance(obj, np.ndarray):
            return obj, None
        t = torch()
        if isinstance(obj, t.Tensor):
            if obj.device.type == "cuda":
                return obj, self._states.get(obj.device.index)
            return obj.numpy(), None
        raise TypeError(f"cannot copy {type(obj).__name__}; expected ndarray, tensor or StorageHandle")

    # -- lifecycle -----------------------------------------------------------------
    def comm(self):
        """The runtime's single-process NCCL communicator over its GPUs (ncclCommInitAll,
        created on first use; drk_comm_create), for reduce_combine="nccl"."""
        self._check_open()
        if self._comm is None:
            devs = sorted(self._states)
            arr = (ctypes.c_int * len(devs))(*devs)
            h = ctypes.c_void_p()
            _lib.call("drk_comm_create", len(devs), arr, ctypes.byref(h))
            self._comm = h.value
        return self._comm

    def close(self):
        with self._lock:
            if self._closed:
                return
            self._closed = True
        if self.backend == "cuda":
            for st in self._states.values():
                try:
                    st.synchronize()
                except Exception:  # pragma: no cover - teardown
                    pass
            if self._comm is not None:
                try:
                    _lib.call("drk_comm_destroy", self._comm)
                except Exception:  # pragma: no cover - teardown
                    pass
                self._comm = None

    def __enter__(self):
        return self

    def __exit__(self, *exc):
        self.close()
        return False

    def __repr__(self):
        return (f"Runtime(locale_count={self.locale_count}, worker_mode={self.worker_mode!r}, "
                f"devices={self.devices}, backend={self.backend!r})")

    def _check_open(self):
        if self._closed:
            raise RuntimeError("runtime is closed")

    def _check_locale(self, locale):
        if not 0 <= locale < self.locale_count:
            raise ValueError(f"invalid locale {locale}: runtime has locales 0..{self.locale_count - 1}")

    def _check_compute(self):
        if self.backend != "cuda":
            raise RuntimeError("this runtime has backend='meta': it holds no data and cannot compute")


def _shape_dtype(x):
    if isinstance(x, np.ndarray):
        return tuple(x.shape), x.dtype
    return tuple(x.shape), _np_dtype_of(x)


def _np_dtype_of(tensor):
    t = torch()
    return np.dtype({t.float32: np.float32, t.float64: np.float64, t.int32: np.int32, t.int64: np.int64,
                     t.uint8: np.uint8, t.bool: np.bool_, t.int16: np.int16, t.int8: np.int8,
                     t.float16: np.float16, t.uint64: np.uint64, t.uint32: np.uint32}[tensor.dtype])


def _check_copy(src, dst):
    (ss, sd), (ds, dd) = _shape_dtype(src), _shape_dtype(dst)
    if ss != ds:
        raise ValueError(f"copy length mismatch: source {ss}, destination {ds}")
    if sd != dd:
        raise ValueError(f"copy dtype mismatch: source {sd}, destination {dd}")
    if isinstance(dst, np.ndarray) and not dst.flags.writeable:
        raise ValueError("copy destination is read-only")

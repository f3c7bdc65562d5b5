"""Segment-parallel algorithms on the device runtime.

Same collective driver-side calls as the reference
(/root/reference/pkg/src/segrange/algorithms.py): for_each (:86-128), reduce (:135-162),
inclusive/exclusive_scan (:169-308, incl. the white-box ``_scan_aligned``), copy
(:468-503), plus ``fill`` and ``transform`` from the north star.  The driver decomposes
the input into segments, lowers each to a fused device expression (views.lower), and
enqueues one kernel per segment on the segment's GPU stream; the combine steps that the
reference runs on the driver (ascending fold of partials, scan of segment totals) stay
on the host over P scalars, with identical numpy scalar semantics.

Element functions are traced once on symbols (expr.py) instead of being executed per
element; functions that cannot be traced raise TypeError rather than running on the
host.
"""

from __future__ import annotations

import ctypes
import operator
import struct
from dataclasses import dataclass

import numpy as np

from . import _lib, expr, kernels, plans
from . import views as _views
from .containers import DistributedVector
from .core import has_segments, is_aligned, runtime_of, segments_of
from .kernels import OPCODES, Launch, run_map, run_reduce, run_scan
from .runtime import AggregateTaskError
from .views import ReadOnly, Target, ZipView, lower


# Tracing: DRK_NVTX=1 wraps every public algorithm in an NVTX range named after
# it, so an nsys / Nsight timeline shows the algorithm calls above their kernels.  Off by
# default (no cost beyond one flag test).
import functools
import os as _os

_NVTX = _os.environ.get("DRK_NVTX") == "1"


def _traced(fn):
    @functools.wraps(fn)
    def wrapper(*args, **kwargs):
        if not _NVTX:
            return fn(*args, **kwargs)
        from .runtime import torch

        nvtx = torch().cuda.nvtx
        nvtx.range_push("drk." + fn.__name__)
        try:
            return fn(*args, **kwargs)
        finally:
            nvtx.range_pop()

    return wrapper


@dataclass(frozen=True)
class BinaryOp:
    """A binary operator with optional identity and numpy ufunc (algorithms.py:34-44)."""

    fn: callable
    identity: object = None
    ufunc: object = None
    name: str = ""

    def __call__(self, a, b):
        return self.fn(a, b)


add = BinaryOp(operator.add, 0, np.add, "add")
multiply = BinaryOp(operator.mul, 1, np.multiply, "multiply")
minimum = BinaryOp(min, None, np.minimum, "minimum")
maximum = BinaryOp(max, None, np.maximum, "maximum")


def as_binary_op(op) -> BinaryOp:
    if isinstance(op, BinaryOp):
        return op
    if callable(op):
        return BinaryOp(op)
    raise TypeError(f"expected a BinaryOp or callable, got {type(op).__name__}")


def _opcode(op: BinaryOp):
    if op.ufunc is None:
        return None
    return OPCODES.get(getattr(op.ufunc, "__name__", ""))


def _pieces(r) -> list:
    """Non-empty segment pieces of r (algorithms.py:61-71)."""
    if has_segments(r) or isinstance(r, ZipView):
        segs = r.segments() if isinstance(r, ZipView) else segments_of(r)
    else:
        segs = [_views._as_piece(r, len(r))]
    return [s for s in segs if len(s)]


def _require_runtime(rt, what):
    if rt is None:
        raise TypeError(f"{what}: input has no device runtime (plain host data); build a DistributedVector")
    rt._check_compute()
    return rt


def _launch_for(rt, rank):
    return Launch(rt.state_of(rank if rank is not None else 0))


def _promote_python(value):
    """Element-wise (non-vectorised) functions see Python scalars in the reference
    (`seg.get(i)` -> .item()): float32 -> float, int32 -> int."""
    if value is None:
        return None
    if isinstance(value, tuple):
        return tuple(_promote_python(v) for v in value)
    dt = value.dtype
    if dt.kind == "f" and dt != np.float64:
        return expr.cast(value, np.float64)
    if dt.kind in "iu" and dt != np.int64:
        return expr.cast(value, np.int64)
    return value


# ----------------------------------------------------------------------------------------
# for_each


@_traced
def for_each(r, fn, vectorized: bool = False) -> None:
    """Apply fn to every element; its non-None result replaces the element (a tuple for
    zips, None components skipped).  Effects are visible on return (algorithms.py:86-98)."""
    fk = expr._fn_key(fn)
    key, dvs, plan = plans.lookup("for_each", r, (fk, vectorized)) if fk is not None else (None, None, None)
    if plan is None:
        pieces = _pieces(r)
        if not pieces:
            return
        rt = _require_runtime(runtime_of(r), "for_each")
        cache = {}
        work = []
        for piece in pieces:
            lw = lower(piece)
            value = lw.value if vectorized else _promote_python(lw.value)
            vkey = _views._value_key(value)
            if vkey not in cache:
                cache[vkey] = expr.trace_cached(fn, value, vkey)
            result = cache[vkey]
            if result is None:
                raise TypeError(
                    "for_each function returned None for every element: it only has side effects, which "
                    "cannot run inside a device kernel"
                )
            writes = []
            _collect_writes(result, lw.target, writes)
            if writes:
                work.append((rt.state_of(writes[0][0].handle.locale), writes, lw.leaves, lw.length))
        plan = plans.store(key, dvs, [rt, work, None])
    _run_map_plan(plan, key is not None)


def _run_map_plan(plan, cached=True):
    """Run a cached map plan [rt, work, bound]: after the first run every launch whose
    arguments are fixed is re-issued as one direct call (kernels.BoundMap)."""
    rt, work, bound = plan
    if bound and kernels._PROFILE is None:
        for b in bound:
            b()
        if _SYNC_ALGORITHMS:
            rt.synchronize()
        return
    launches = []
    for st, writes, leaves, length in work:
        launch = Launch(st)
        run_map(writes, leaves, length, launch)
        launches.append(launch)
    _finish(rt, launches)
    if bound is None and cached:
        bs = [kernels.bind_map(writes, leaves, length, st) for st, writes, leaves, length in work]
        plan[2] = _bind_launches(bs)


def _bind_launches(bs):
    """The fixed-argument launches of a plan: one CUDA graph when several go to one stream,
    else the BoundMaps; () when any launch needs per-call work (then run_map every time)."""
    if not bs or not all(b is not None for b in bs):
        return ()
    g = kernels.capture(bs) if len(bs) > 1 else None
    return [g] if g is not None else bs


def _collect_writes(result, target, writes):
    if result is None:
        return
    if isinstance(target, ReadOnly):
        raise TypeError(f"cannot write through read-only {target.what}")
    if isinstance(target, tuple):
        if not isinstance(result, tuple) or len(result) != len(target):
            n = len(target)
            raise ValueError(f"expected a {n}-tuple, got {len(result) if isinstance(result, tuple) else 1} values")
        for r, t in zip(result, target):
            _collect_writes(r, t, writes)
        return
    if isinstance(result, tuple):
        raise TypeError("element function returned a tuple for a non-zip range")
    writes.append((target, result))


# Element-wise algorithms (for_each, copy, fill, transform) return once their kernels are
# enqueued.  Everything that reads the results is ordered after them: later work on the same
# GPU by stream order, kernels on other GPUs by an event wait (kernels.stage_leaves), host
# reads (to_numpy, element access, copies to host) by a stream sync, peer copies and sort by
# an explicit sync of the source GPU.  Device temporaries are stream-ordered allocations, so
# dropping them here is safe.  _SYNC_ALGORITHMS = True restores wait-on-return.
_SYNC_ALGORITHMS = False


def _finish(rt, launches):
    if not _SYNC_ALGORITHMS:
        return
    devs = {id(l.state): l.state for l in launches}
    for st in devs.values():
        st.synchronize()


# ----------------------------------------------------------------------------------------
# reduce


_PARTIAL_DTYPE = {}


def _partial_dtype(op: BinaryOp, dtype):
    """numpy's reduce result dtype (int32 add/mul -> int64, float32 stays float32)."""
    if op.ufunc is None:
        return np.dtype(dtype)
    key = (op.ufunc, np.dtype(dtype))
    r = _PARTIAL_DTYPE.get(key)
    if r is None:
        r = _PARTIAL_DTYPE[key] = op.ufunc.reduce(np.zeros(1, dtype=dtype)).dtype
    return r


@_traced
def reduce(r, init=0, op=add):
    """Fold all elements onto init: per-segment device partials, then an ascending fold on
    the driver (algorithms.py:135-150), so exact types give identical results for every
    segment count.  The lowered plan of r is memoised by r's structure (plans.py)."""
    op = as_binary_op(op)
    opk = _op_key(op)
    key, dvs, plan = plans.lookup("reduce", r, opk) if opk is not None else (None, None, None)
    if plan is None:
        pieces = _pieces(r)
        if not pieces:
            return init.item() if isinstance(init, np.generic) else init
        plan = plans.store(key, dvs, _ReducePlan(_require_runtime(runtime_of(r), "reduce"), pieces, op))
    if plan.rt.reduce_combine != "host":
        r = plan.fold_on_device(init)
        if r is not None:
            return r
    partials = plan.run()
    acc = init
    for p in partials:
        acc = op.fn(acc, p)
    return acc.item() if isinstance(acc, np.generic) else acc


def _op_key(op: BinaryOp):
    """Cache identity of a binary operator: the ufunc and the function (by behaviour for
    traced Python functions), or None if the function can reach mutable state."""
    fn = op.fn
    if isinstance(fn, (type(min), type(operator.add))) or fn in (min, max):
        fk = ("builtin", fn)
    else:
        fk = expr._fn_key(fn)
        if fk is None:
            return None
    return (getattr(op.ufunc, "__name__", None), fk)


class _ReducePlan:
    """A reduce over fixed segments: lowered pieces, their launch plan (one batched launch when
    a single GPU holds every piece and the catalogue covers them), and the result decoding."""

    __slots__ = ("rt", "lowered", "op", "opcode", "combiner", "batch", "order", "need", "fused", "dinit")

    def __init__(self, rt, pieces, op):
        self.rt = rt
        self.op = op
        self.opcode = _opcode(op)
        self.combiner = op if self.opcode is None else None
        lowered = []
        for piece in pieces:
            lw = lower(piece)
            if isinstance(lw.value, tuple):
                raise TypeError("reduce needs scalar elements; apply a transform to the zip first")
            lowered.append(lw)
        self.lowered = lowered
        need = {}
        for lw in lowered:
            st = rt.state_of(lw.rank if lw.rank is not None else 0)
            need[id(st)] = (st, need.get(id(st), (st, 0))[1] + 1)
        self.need = list(need.values())
        self.batch = _batch_reduce_plan(rt, lowered, self.opcode) if self.opcode is not None else None
        self.fused = None  # _FusedReduce, built on first use (reduce_combine="fused")
        self.dinit = {}    # init -> (P, init as P) of the device folds

    def run(self):
        for st, k in self.need:
            st.ensure_results(k)  # before any launch: growing the slot buffer reallocates it
        if self.batch is not None:
            return self.batch.run()
        else:
            order, launches, slots = [], {}, {}
            for lw in self.lowered:
                st = self.rt.state_of(lw.rank if lw.rank is not None else 0)
                launch = launches.setdefault(id(st), Launch(st))
                slot = slots.get(id(st), 0)
                slots[id(st)] = slot + 1
                node = lw.value if self.opcode is not None else _promote_python(lw.value)
                run_reduce(node, lw.leaves, lw.length, self.opcode, self.combiner, launch, slot)
                order.append((st, slot, node.dtype))
        raw = {id(l.state): l.state.fetch_host_results(slots[id(l.state)]) for l in launches.values()}
        out = []
        op = self.op
        for st, slot, vdt in order:
            if self.opcode is not None:
                A = _lib.acc_dtype(vdt, self.opcode)
                a = np.frombuffer(raw[id(st)][slot * 8 : slot * 8 + A.itemsize].tobytes(), dtype=A)[0]
                out.append(a.astype(_partial_dtype(op, vdt)))
            else:
                a = np.frombuffer(raw[id(st)][slot * 8 : slot * 8 + vdt.itemsize].tobytes(), dtype=vdt)[0]
                out.append(a.item())
        return out


    def _device_init(self, init):
        """init as a scalar of the partial dtype P when the host fold `op.fn(init, p)` stays
        in P (numpy promotion of a Python or same-dtype scalar), else None (host fold)."""
        if self.opcode is None or not self.lowered:
            return None
        vdts = {lw.value.dtype for lw in self.lowered}
        if len(vdts) != 1:
            return None
        P = _partial_dtype(self.op, vdts.pop())
        if P not in _lib.DTYPE_CODE:
            return None
        try:
            with np.errstate(all="ignore"):
                probe = self.op.fn(init, P.type(0))
                iv = P.type(init)
        except (OverflowError, TypeError, ValueError):
            return None
        if np.asarray(probe).dtype != P:
            return None
        return P, iv

    def fold_on_device(self, init):
        """The reduce folded on the device (rt.reduce_combine "device" or "nccl"): every
        segment's partial is reduced into a device slot of its GPU, then
          device: the first GPU waits for the others (CUDA events) and folds the partials
                  from their memory over NVLink (drk_reduce_fold);
          nccl:   one drk_comm_reduce — an NCCL all-gather of every GPU's partial slots, then
                  every GPU folds them in segment order (the result on every GPU);
        and one mapped-memory read of the result.  The fold is the reference driver's
        ascending fold in numpy's reduce dtype (algorithms.py:146-149), so the value is the
        host fold's bit for bit.  None when the host must fold (see _device_init)."""
        from .runtime import torch

        k = (type(init), repr(init))
        di = self.dinit.get(k, 0)
        if di == 0:
            di = self._device_init(init)
            if di is not None:
                di = (*di, _lib.scalar_buffer(di[1], di[0]))
            self.dinit[k] = di
        if di is None or len(self.lowered) > _lib.FOLD_MAX:
            return None
        P, iv, initbuf = di
        rt = self.rt
        mode = rt.reduce_combine
        if mode == "fused":
            return self._fused(P, iv, initbuf)
        for st, k in self.need:
            st.ensure_results(k)
        states = sorted(rt.device_states, key=lambda s: s.index)
        pos = {id(s): i for i, s in enumerate(states)}
        cnt = {}
        place = []  # (state, slot) of each segment, in segment order
        for lw in self.lowered:
            st = rt.state_of(lw.rank if lw.rank is not None else 0)
            j = cnt.get(id(st), 0)
            cnt[id(st)] = j + 1
            place.append((st, j))
        words = max(cnt.values())
        ndev = len(states)
        for st in states:
            st.combine_slots(8 * words * (ndev + 1))
        if isinstance(self.batch, _BatchReduce):
            self.batch.launch(result_ptr=self.batch.st.combine_slots(0).data_ptr())
        else:
            launches = {}
            for lw, (st, j) in zip(self.lowered, place):
                launch = launches.setdefault(id(st), Launch(st))
                node = lw.value
                run_reduce(node, lw.leaves, lw.length, self.opcode, None, launch, j,
                           result_ptr=st.combine_slots(0).data_ptr() + 8 * j)
        code = _lib.DTYPE_CODE[self.lowered[0].value.dtype]
        initbuf = _lib.scalar_buffer(iv, P)
        st0 = states[0]
        host = st0.host_result_dev_ptr(0)
        if mode == "nccl":
            comm = rt.comm()
            vp = ctypes.c_void_p
            send = (vp * ndev)(*[s.combine_slots(0).data_ptr() for s in states])
            recv = (vp * ndev)(*[s.combine_slots(0).data_ptr() + 8 * words for s in states])
            streams = (vp * ndev)(*[s.handle for s in states])
            order = (ctypes.c_int * len(place))(*[pos[id(s)] * words + j for s, j in place])
            _lib.call("drk_comm_reduce", comm, code, self.opcode, send, recv, words, order, len(place),
                      ctypes.addressof(initbuf), None, host, streams)
        else:
            t = torch()
            for s in states[1:]:
                if s is not st0 and id(s) in cnt:
                    ev = t.cuda.Event()
                    ev.record(s.stream)
                    st0.stream.wait_event(ev)
            parts = (ctypes.c_void_p * len(place))(*[s.combine_slots(0).data_ptr() + 8 * j for s, j in place])
            _lib.call("drk_reduce_fold", code, self.opcode, parts, len(place), ctypes.addressof(initbuf), None, host,
                      st0.index, st0.handle)
        raw = st0.fetch_host_results(1)
        r = np.frombuffer(raw[: P.itemsize].tobytes(), dtype=P)[0]
        return r.item()


    def _fused(self, P, iv, initbuf):
        """reduce_combine="fused": one drk_reduce_fused call — every GPU's batched kernel stores
        its segments' partials into slots on the first GPU and the last CTA of the call folds
        them (segment order, numpy's reduce dtype) straight into mapped host memory.  None
        (another mode runs) when the pieces are not a catalogue batch."""
        fp = self.fused
        if fp is None:
            fp = self.fused = _FusedReduce.build(self) or False
        if fp is False:
            return None
        return fp.run(P, iv, initbuf)


class _FusedReduce:
    """The fixed arguments of a drk_reduce_fused call for one reduce plan (built once)."""

    __slots__ = ("home", "states", "handles", "args_head", "args_tail", "total", "scratch")

    @staticmethod
    def build(plan):
        rt = plan.rt
        st_of = [rt.state_of(lw.rank if lw.rank is not None else 0) for lw in plan.lowered]
        groups = {}
        for j, st in enumerate(st_of):
            groups.setdefault(id(st), (st, []))[1].append(j)
        gs = sorted(groups.values(), key=lambda g: g[0].index)
        if any(len(ix) > _lib.RED_SEGS for _, ix in gs) or len(plan.lowered) > _lib.FOLD_MAX:
            return None
        plans_ = [kernels.catalogue_reduce(lw.value, lw.leaves, plan.opcode, st.index)
                  for lw, st in zip(plan.lowered, st_of)]
        if any(p is None for p in plans_) or len({(p[0], p[1]) for p in plans_}) != 1:
            return None
        f = _FusedReduce()
        f.home = gs[0][0]
        f.states = [st for st, _ in gs]
        f.handles = [(st, [lf.handle for j in ix for lf in plan.lowered[j].leaves if lf.handle is not None])
                     for st, ix in gs]
        total = f.total = len(plan.lowered)
        flat = [j for _, ix in gs for j in ix]
        nd, vp = len(gs), ctypes.c_void_p
        kind, code = plans_[0][0], plans_[0][1]
        buf = f.home.combine_slots(8 * _lib.FOLD_MAX + 64)
        f.args_head = (0 if kind == "reduce" else 1, code, plan.opcode, nd,
                       (ctypes.c_int * nd)(*[st.index for st in f.states]),
                       (vp * nd)(*[st.handle for st in f.states]),
                       (ctypes.c_int * nd)(*[len(ix) for _, ix in gs]),
                       (vp * total)(*[plans_[j][2] for j in flat]),
                       (vp * total)(*[plans_[j][3] for j in flat]) if kind == "dot" else None,
                       (ctypes.c_int64 * total)(*[plan.lowered[j].length for j in flat]),
                       (ctypes.c_int * total)(*flat), buf.data_ptr(), buf.data_ptr() + 8 * _lib.FOLD_MAX)
        f.args_tail = [len(ix) for _, ix in gs]
        f.scratch = None
        return f

    def run(self, P, iv, initbuf):
        from .runtime import _EPOCHS, await_pending

        for st, hs in self.handles:
            for h in hs:
                if h._pending:
                    await_pending(st, hs)
                    break
        home = self.home
        fh, fd = home.flag_ptrs()
        epoch = next(_EPOCHS)
        bufs = [st.reduce_batch_scratch(c) for st, c in zip(self.states, self.args_tail)]
        if self.scratch is None or any(a is not b for a, b in zip(bufs, self.scratch[0])):
            self.scratch = (bufs, (ctypes.c_void_p * len(bufs))(*[b.data_ptr() for b in bufs]))
        rc = _lib.fn("drk_reduce_fused")(*self.args_head, ctypes.addressof(initbuf), home.host_result_dev_ptr(0),
                                         fd, epoch, self.scratch[1])
        if rc:
            _lib.check(rc, "drk_reduce_fused")
        rc = _lib.fn("drk_wait_flags")(fh, 1, epoch, home.index, home.handle)
        if rc:
            _lib.check(rc, "drk_wait_flags")
        return np.frombuffer(home._host_results_np, dtype=P, count=1)[0].item()


def _segment_partials(rt, pieces, op):
    return _ReducePlan(rt, pieces, op).run()


class _BatchReduce:
    """Several segments on one GPU, each a catalogue reduction (a plain device array, or the
    product of two for dot): one drk_reduce_batch / drk_dot_batch launch, its argument arrays
    built once."""

    __slots__ = ("st", "kind", "code", "opcode", "m", "xs", "ys", "ns", "handles", "dtypes", "total", "decode",
                 "fmt", "op")

    def run(self):
        """Launch, wait, and the partials in numpy's reduce dtype (the C1 hot path: argument
        arrays, the result layout and the decoding are fixed at plan time).  The kernel marks
        each result final with a completion word in mapped memory, and the host waits on
        those words (drk_wait_flags) rather than synchronising the whole stream."""
        st = self.st
        if kernels._PROFILE is not None:
            self.launch()
            st.synchronize()
        else:
            for h in self.handles:
                if h._pending:
                    from .runtime import await_pending

                    await_pending(st, self.handles)
                    break
            fh, fd, epoch = st.completion_flags()
            scratch = st.reduce_batch_scratch(self.m).data_ptr()
            res = st.host_result_dev_ptr(0)
            if self.kind == "reduce":
                rc = _lib.fn("drk_reduce_batch_ex")(self.code, self.opcode, self.m, self.xs, self.ns, res, fd, epoch,
                                                    scratch, st.index, st.handle)
            else:
                rc = _lib.fn("drk_dot_batch_ex")(self.code, self.m, self.xs, self.ys, self.ns, res, fd, epoch,
                                                 scratch, st.index, st.handle)
            if rc:
                _lib.check(rc, "drk_reduce_batch" if self.kind == "reduce" else "drk_dot_batch")
            rc = _lib.fn("drk_wait_flags")(fh, self.m, epoch, st.index, st.handle)
            if rc:
                _lib.check(rc, "drk_wait_flags")
        vals = struct.unpack_from(self.fmt, st._host_results_np)
        return [cast(v) for cast, v in zip(self.decode, vals)]

    def launch(self, result_ptr=None):
        """Enqueue the batched kernel; results into the mapped host slots [0, m) of the
        GPU, or into device memory at result_ptr (8-byte slots)."""
        st = self.st
        for h in self.handles:
            if h._pending:
                from .runtime import await_pending

                await_pending(st, self.handles)
                break
        scratch = st.reduce_batch_scratch(self.m)
        res = st.host_result_dev_ptr(0) if result_ptr is None else result_ptr
        if kernels._PROFILE is None:  # the common case: one direct call
            if self.kind == "reduce":
                rc = _lib.fn("drk_reduce_batch")(self.code, self.opcode, self.m, self.xs, self.ns, res,
                                                 scratch.data_ptr(), st.index, st.handle)
            else:
                rc = _lib.fn("drk_dot_batch")(self.code, self.m, self.xs, self.ys, self.ns, res, scratch.data_ptr(),
                                              st.index, st.handle)
            if rc:
                _lib.check(rc, "drk_reduce_batch" if self.kind == "reduce" else "drk_dot_batch")
            return None
        launch = Launch(st)
        if self.kind == "reduce":
            kernels.launch_kernel("drk_reduce_batch", launch, self.total, self.code, self.opcode, self.m, self.xs,
                                  self.ns, res, scratch.data_ptr())
        else:
            kernels.launch_kernel("drk_dot_batch", launch, self.total, self.code, self.m, self.xs, self.ys, self.ns,
                                  res, scratch.data_ptr())
        order = [(st, j, dt) for j, dt in enumerate(self.dtypes)]
        return order, {id(st): launch}, {id(st): self.m}


class _MultiReduce:
    """The segments of a reduce spread over several GPUs, each GPU's share a catalogue batch:
    one drk_reduce_multi call enqueues every GPU's batched kernel (the multi-device variant of
    the C ABI), the host waits on every GPU's completion words, and the partials come back in
    segment order for the driver fold."""

    __slots__ = ("states", "kind", "code", "opcode", "counts", "devices", "streams", "xs", "ys", "ns", "handles",
                 "order", "fmts", "decode")

    def run(self):
        from .runtime import _EPOCHS, await_pending

        for st, hs in self.handles:
            for h in hs:
                if h._pending:
                    await_pending(st, hs)
                    break
        nd = len(self.states)
        vp = ctypes.c_void_p
        results = (vp * nd)(*[st.host_result_dev_ptr(0) for st in self.states])
        ptrs = [st.flag_ptrs() for st in self.states]
        flags = (vp * nd)(*[p[1] for p in ptrs])
        scratch = (vp * nd)(*[st.reduce_batch_scratch(c).data_ptr() for st, c in zip(self.states, self.counts)])
        epoch = next(_EPOCHS)
        if kernels._PROFILE is None:
            _lib.call("drk_reduce_multi", 0 if self.kind == "reduce" else 1, self.code, self.opcode, nd, self.devices,
                      self.streams, (ctypes.c_int * nd)(*self.counts), self.xs, self.ys, self.ns, results, flags,
                      epoch, scratch)
        else:  # profiled runs (bench.py): each GPU's batched launch, timed on its own stream
            off = 0
            for d, (st, c) in enumerate(zip(self.states, self.counts)):
                xs = (vp * c)(*self.xs[off:off + c])
                ns = (ctypes.c_int64 * c)(*self.ns[off:off + c])
                if self.kind == "reduce":
                    kernels.launch_kernel("drk_reduce_batch_ex", Launch(st), sum(ns), self.code, self.opcode, c, xs,
                                          ns, results[d], flags[d], epoch, scratch[d])
                else:
                    ys = (vp * c)(*self.ys[off:off + c])
                    kernels.launch_kernel("drk_dot_batch_ex", Launch(st), sum(ns), self.code, c, xs, ys, ns,
                                          results[d], flags[d], epoch, scratch[d])
                off += c
        out = [None] * sum(self.counts)
        for st, c, (fh, _), fmt, dec, ix in zip(self.states, self.counts, ptrs, self.fmts, self.decode, self.order):
            _lib.call("drk_wait_flags", fh, c, epoch, st.index, st.handle)
            for j, cast, v in zip(ix, dec, struct.unpack_from(fmt, st._host_results_np)):
                out[j] = cast(v)
        return out


def _batch_reduce_plan(rt, lowered, opcode):
    """A _BatchReduce (one GPU) or _MultiReduce (several) for the pieces, or None when they do
    not qualify (more than DRK_RED_SEGS pieces on one GPU, or an expression outside the
    catalogue)."""
    m = len(lowered)
    if m < 1 or opcode is None:
        return None
    groups = {}
    for j, lw in enumerate(lowered):
        st = rt.state_of(lw.rank if lw.rank is not None else 0)
        groups.setdefault(id(st), (st, []))[1].append(j)
    if any(len(ix) > _lib.RED_SEGS for _, ix in groups.values()):
        return None
    st_of = [rt.state_of(lw.rank if lw.rank is not None else 0) for lw in lowered]
    plans_ = [kernels.catalogue_reduce(lw.value, lw.leaves, opcode, st.index) for lw, st in zip(lowered, st_of)]
    if any(p is None for p in plans_) or len({(p[0], p[1]) for p in plans_}) != 1:
        return None
    if len(groups) > 1:
        mb = _MultiReduce()
        gs = sorted(groups.values(), key=lambda g: g[0].index)
        mb.states = [g[0] for g in gs]
        mb.order = [g[1] for g in gs]
        mb.counts = [len(ix) for ix in mb.order]
        mb.kind, mb.code, mb.opcode = plans_[0][0], plans_[0][1], opcode
        flat = [j for ix in mb.order for j in ix]
        nd, m_ = len(gs), len(flat)
        mb.devices = (ctypes.c_int * nd)(*[st.index for st in mb.states])
        mb.streams = (ctypes.c_void_p * nd)(*[st.handle for st in mb.states])
        mb.xs = (ctypes.c_void_p * m_)(*[plans_[j][2] for j in flat])
        mb.ys = (ctypes.c_void_p * m_)(*[plans_[j][3] for j in flat]) if mb.kind == "dot" else None
        mb.ns = (ctypes.c_int64 * m_)(*[lowered[j].length for j in flat])
        mb.handles = [(st, [lf.handle for j in ix for lf in lowered[j].leaves if lf.handle is not None])
                      for st, ix in zip(mb.states, mb.order)]
        mb.fmts, mb.decode = [], []
        for ix in mb.order:
            fmt, dec = _decode_of([lowered[j].value.dtype for j in ix], opcode)
            mb.fmts.append(fmt)
            mb.decode.append(dec)
        return mb
    st = st_of[0]
    b = _BatchReduce()
    b.st = st
    b.kind, b.code = plans_[0][0], plans_[0][1]
    b.opcode = opcode
    b.m = m
    b.ns = (ctypes.c_int64 * m)(*[lw.length for lw in lowered])
    b.total = sum(lw.length for lw in lowered)
    b.xs = (ctypes.c_void_p * m)(*[p[2] for p in plans_])
    b.ys = (ctypes.c_void_p * m)(*[p[3] for p in plans_]) if b.kind == "dot" else None
    b.handles = [lf.handle for lw in lowered for lf in lw.leaves if lf.handle is not None]
    b.dtypes = [lw.value.dtype for lw in lowered]
    b.fmt, b.decode = _decode_of(b.dtypes, opcode)
    return b


def _decode_of(dtypes, opcode):
    """struct format and casts of consecutive result slots: slot j holds the accumulator
    (drk_acc_dtype) of segment j; the reference's partial is that value in numpy's reduce
    dtype (float32 sums are accumulated in fp64, then rounded)."""
    fmt, decode = "<", []
    for dt in dtypes:
        A = _lib.acc_dtype(dt, opcode)
        fmt += {"f8": "d", "f4": "f4x", "i8": "q", "i4": "i4x"}[A.kind + str(A.itemsize)]
        decode.append(_PARTIAL_OF[(opcode, np.dtype(dt))])
    return fmt, decode


def _partial_caster(opcode, dt):
    ufunc = {_lib.ADD: np.add, _lib.MUL: np.multiply, _lib.MIN: np.minimum, _lib.MAX: np.maximum}[opcode]
    return _partial_dtype(BinaryOp(ufunc, None, ufunc), dt).type


class _PartialOf(dict):
    def __missing__(self, key):
        v = self[key] = _partial_caster(*key)
        return v


_PARTIAL_OF = _PartialOf()


# ----------------------------------------------------------------------------------------
# scans


@_traced
def inclusive_scan(r, out, op=add) -> None:
    """out[i] = fold of r[0..i] (algorithms.py:169-177)."""
    _scan_entry(r, out, as_binary_op(op), exclusive=False, init=None)


@_traced
def exclusive_scan(r, out, init, op=add) -> None:
    """out[0] = init, out[i] = init ⊕ fold of r[0..i) (algorithms.py:180-182)."""
    _scan_entry(r, out, as_binary_op(op), exclusive=True, init=init)


def _scan_entry(r, out, op, exclusive, init):
    if len(r) != len(out):
        raise ValueError(f"scan length mismatch: input {len(r)}, output {len(out)}")
    r_seg, o_seg = has_segments(r), has_segments(out)
    if not o_seg:
        raise TypeError("scan output must be a segmented device range")
    if r is out or (r_seg and _aligned(r, out)):
        _scan_impl(r, out, op, exclusive, init, want_partials=False)
        return
    if not isinstance(out, DistributedVector):
        raise TypeError("non-aligned scan needs a DistributedVector output")
    temp = DistributedVector.like_distribution(out.runtime, out.distribution, out.dtype)
    copy(r, temp)
    _scan_impl(temp, out, op, exclusive, init, want_partials=False)


def _aligned(r, out) -> bool:
    """core.is_aligned, memoised by the structure of both ranges (plans.py)."""
    key = None
    if plans._ENABLED:
        dvs = []
        kr, ko = plans.view_key(r, dvs), plans.view_key(out, dvs)
        if kr is not None and ko is not None:
            key = ("aligned", kr, ko)
            hit = plans.CACHE.get(key)
            if hit is not None:
                return hit[0]
    value = is_aligned(r, out)
    if key is not None:
        plans.CACHE.put(key, dvs, (value,))
    return value


def _scan_aligned(r, out, op, exclusive, init) -> list:
    """Aligned scan; returns the per-segment input totals (None for empty segments), the
    white-box intermediate of the reference (algorithms.py:234-274)."""
    return _scan_impl(r, out, op, exclusive, init)


def _scan_impl(r, out, op, exclusive, init, carry=None, carry_hook=None, want_partials=True) -> list:
    """Aligned scan with an optional incoming carry (the fold of everything before r,
    in the accumulator type; used when r is one rank's block of a larger vector).

    carry_hook(total_ptrs, state) -> (carry_dev_ptr or None, carry_host_fn): the incoming
    carry produced on the device between the two passes of the multi-device schedule (the
    one-process-per-GPU scan, spmd.py); carry_host_fn() gives its value on the host after
    the scan (for the int32 range check).

    want_partials=False (the public inclusive/exclusive_scan, which return nothing): on one
    GPU, when no int32 carry-range check is due, the scan is left running on the stream —
    the host does not wait for the totals, later work on the stream is ordered after it,
    and kernels on other GPUs that read its output wait for it (kernels.stage_leaves)."""
    op = as_binary_op(op)
    opcode = _opcode(op)
    if opcode is None:
        from . import codegen

        in_segs = segments_of(r)
        out_segs = segments_of(out)
        live = [k for k, s in enumerate(in_segs) if len(s)]
        if not live:
            return [None] * len(in_segs)
        rt = _require_runtime(runtime_of(out, r), "scan")
        return codegen.custom_scan(rt, in_segs, out_segs, live, op, exclusive, init, carry)
    rt, nseg, live, lowered = _scan_lowered(r, out)
    partials = [None] * nseg
    if not live:
        return partials

    # 1. what each live segment scan reads: a plain device array in the output dtype, or a
    #    view — fused into the scan kernel (its leaves are read, nothing is materialised;
    #    the reference materialises f's result, views.py:164-181, then accumulates it)
    work = []
    launches = {}
    for k, lw, tgt, st in lowered:
        launch = launches.setdefault(id(st), Launch(st))
        node = lw.value
        if isinstance(node, tuple):
            raise TypeError("scan needs scalar elements; apply a transform to the zip first")
        plain = node.op == "leaf" and lw.leaves[node.value].kind == "array" and node.dtype == tgt.dtype
        if plain and lw.leaves[node.value].device == st.index:
            from .runtime import await_pending

            await_pending(st, [lw.leaves[node.value].handle, tgt.handle])
            src = lw.leaves[node.value].ptr()
        else:
            src = _fused_scan_source(node, lw, tgt, opcode, launch)
            if src is None:
                run_map([(tgt, node)], lw.leaves, lw.length, launch)
                src = tgt.ptr()
        work.append((k, st, launch, src, tgt))

    T = np.dtype(out.dtype if hasattr(out, "dtype") else work[0][4].dtype)
    A = _lib.acc_dtype(T, opcode)
    L = _partial_dtype(op, T)
    devices = {id(w[1]) for w in work}
    init_a = None
    if exclusive:
        init_a = _to_acc(init, A)

    if len(devices) == 1 and not _FORCE_MULTI_DEVICE_SCAN and carry_hook is None:
        st = work[0][1]
        m = len(work)
        if (_BATCH_SCANS and 1 < m <= _lib.SCAN_SEGS and sum(w[4].length for w in work) >= _BATCH_MIN
                and all(isinstance(w[3], int) and w[3] % 16 == 0 and w[4].ptr() % 16 == 0 for w in work)):
            # single device, several segments: one batched launch scans them as one sequence
            return _scan_batched(work, partials, live, st, op, opcode, T, A, L, exclusive, init, init_a, carry,
                                 want_partials)
        # single device: chain the carry on the device, one pass per segment
        st.ensure_results(2 * len(work) + 2)
        prev_carry = None
        for j, (k, _, launch, in_ptr, tgt) in enumerate(work):
            first_carry = _to_acc(carry, A) if (j == 0 and carry is not None) else None
            # segment j's carry is written by segment j-1's scan, enqueued just before: chain
            # them (programmatic dependent launch) so j's tiles reduce while j-1 drains
            _run_segment_scan(T, opcode, exclusive, in_ptr, tgt, launch, init=init_a,
                              carry_value=first_carry,
                              carry_dev=st.result_dev_ptr(prev_carry) if prev_carry is not None else None,
                              seg_total_slot=2 * j, carry_out_slot=2 * j + 1,
                              chained=prev_carry is not None and _CHAIN_SCANS, scratch_index=j % 2)
            prev_carry = 2 * j + 1
        if not want_partials and (not _needs_range_check(T) or len(work) == 1):
            # nothing to read back: the scan stays asynchronous on its stream.  With one live
            # segment the int32 range check sees only host values (the carry / init seed its
            # one segment; no device total is added to anything)
            if len(work) == 1:
                _check_carry_range(op, partials, live, exclusive, init, T, carry)
            return partials
        raw = st.fetch_results(2 * len(work))
        for j, (k, *_rest) in enumerate(work):
            total = np.frombuffer(raw[16 * j : 16 * j + A.itemsize].tobytes(), dtype=A)[0]
            partials[k] = total.astype(L).item()
        _check_carry_range(op, partials, live, exclusive, init, T, carry)
        return partials

    if carry_hook is not None or (len(work) <= _lib.CARRY_MAX + 1 and not _FORCE_HOST_CARRY):
        return _scan_device_carry(work, partials, live, op, opcode, T, A, L, exclusive, init, init_a, carry,
                                  launches, carry_hook, want_partials)
    # several devices, host carry (more segments than drk_carry_fold takes): totals first
    # (all GPUs in parallel), carries on the host exactly as the reference's driver loop,
    # then one carried scan per segment.
    per_dev_slot = {}
    for k, st, launch, in_ptr, tgt in work:
        per_dev_slot[id(st)] = per_dev_slot.get(id(st), 0) + 1
    for k, st, *_ in work:
        st.ensure_results(per_dev_slot[id(st)])
    per_dev_slot = {}
    for k, st, launch, in_ptr, tgt in work:
        slot = per_dev_slot.get(id(st), 0)
        per_dev_slot[id(st)] = slot + 1
        _segment_total(T, opcode, in_ptr, tgt, launch, st.host_result_dev_ptr(slot))
    fetched = {id(w[1]): w[1].fetch_host_results(per_dev_slot[id(w[1])]) for w in work}
    counter = {}
    for k, st, *_ in work:
        slot = counter.get(id(st), 0)
        counter[id(st)] = slot + 1
        total = np.frombuffer(fetched[id(st)][8 * slot : 8 * slot + A.itemsize].tobytes(), dtype=A)[0]
        partials[k] = total.astype(L).item()
    offsets = _offsets(op, partials, carry)
    _check_carry_range(op, partials, live, exclusive, init, T, carry)
    for k, st, launch, in_ptr, tgt in work:
        off = offsets[k]
        _run_segment_scan(T, opcode, exclusive, in_ptr, tgt, launch, init=init_a,
                          carry_value=_to_acc(off, A) if off is not None else None)
    for l in launches.values():
        l.state.synchronize()
    return partials


# Test hooks: take the multi-device scan schedule even when every segment shares one GPU
# (_FORCE_MULTI_DEVICE_SCAN), or fold its carries on the host (_FORCE_HOST_CARRY).
_FORCE_MULTI_DEVICE_SCAN = False
_FORCE_HOST_CARRY = False
_CHAIN_SCANS = True  # programmatic dependent launches for consecutive segment scans on one GPU
_BATCH_SCANS = True  # one drk_scan_batch launch for the segments a GPU holds (up to SCAN_SEGS)
_BATCH_MIN = 1 << 20  # below this many elements the chained single-pass scans are cheaper


def _needs_range_check(T):
    """int32 scans check the carry range on the host (the reference's OverflowError)."""
    T = np.dtype(T)
    return T.kind in "iu" and T.itemsize < 8


def _scan_batched(work, partials, live, st, op, opcode, T, A, L, exclusive, init, init_a, carry,
                  want_partials=True):
    """The segments on one GPU scanned by one drk_scan_batch launch: the L2 scan runs over
    their concatenation, so the look-back carries the prefix from segment to segment
    (algorithms.py:256-262 without a pass per segment), and the per-segment totals — the
    reference's partials — are folded from the tile aggregates afterwards."""
    code = _lib.dtype_code(T)
    m = len(work)
    ins = (ctypes.c_void_p * m)(*[w[3] for w in work])
    outs = (ctypes.c_void_p * m)(*[w[4].ptr() for w in work])
    ns = (ctypes.c_int64 * m)(*[w[4].length for w in work])
    nbytes = int(_lib.load().drk_scan_batch_scratch_bytes(code, opcode, m, ns))
    scratch = st.scan_scratch(nbytes, 0)
    st.ensure_results(m)
    launch = work[0][2]
    init_buf = _lib.scalar_buffer(init_a, A) if init_a is not None else None
    carry_buf = _lib.scalar_buffer(_to_acc(carry, A), A) if carry is not None else None
    kernels.launch_kernel("drk_scan_batch", launch, sum(ns), code, opcode, 1 if exclusive else 0, m, ins, outs, ns,
                          ctypes.addressof(init_buf) if init_buf is not None else None,
                          ctypes.addressof(carry_buf) if carry_buf is not None else None, None,
                          st.result_dev_ptr(0), None, scratch.data_ptr(), scratch.numel())
    if not want_partials and not _needs_range_check(T):
        return partials  # nothing to read back: the scan stays asynchronous on its stream
    raw = st.fetch_results(m)
    for j, (k, *_rest) in enumerate(work):
        total = np.frombuffer(raw[8 * j: 8 * j + A.itemsize].tobytes(), dtype=A)[0]
        partials[k] = total.astype(L).item()
    _check_carry_range(op, partials, live, exclusive, init, T, carry)
    return partials


def _scan_device_carry(work, partials, live, op, opcode, T, A, L, exclusive, init, init_a, carry, launches,
                       carry_hook=None, want_partials=True):
    """Scan of segments spread over several GPUs with the carry folded on the devices.

    1. Every segment's total is reduced on its own GPU (all GPUs in parallel).
    2. Each segment's stream waits (CUDA events) for the GPUs that hold earlier segments,
       folds their totals straight from peer memory over NVLink (drk_carry_fold: the
       reference's driver loop, algorithms.py:256-262, on the device), and scans with it.
    The host reads the totals only afterwards (the white-box partials, the int32 carry
    range check), so nothing between the two passes waits for the host."""
    from .runtime import torch

    t = torch()
    code = _lib.dtype_code(T)
    count = {}
    for k, st, *_ in work:
        count[id(st)] = count.get(id(st), 0) + 1
    for k, st, *_ in work:
        st.ensure_results(2 * count[id(st)])  # totals, then carries
    tot_ptr, used = {}, {}
    for k, st, launch, in_ptr, tgt in work:
        slot = used.get(id(st), 0)
        used[id(st)] = slot + 1
        tot_ptr[k] = st.result_dev_ptr(slot)
        _segment_total(T, opcode, in_ptr, tgt, launch, tot_ptr[k])
    reduced = {}
    for k, st, *_ in work:
        if id(st) not in reduced:
            ev = t.cuda.Event()
            ev.record(st.stream)
            reduced[id(st)] = ev
    in_dev, carry_host_fn = None, None
    if carry_hook is not None:
        st0 = work[0][1]
        for k, st, *_ in work:
            if st is not st0:
                st0.stream.wait_event(reduced[id(st)])
        in_dev, carry_host_fn = carry_hook([tot_ptr[w[0]] for w in work], st0)
        if any(w[1] is not st0 for w in work):
            ev = t.cuda.Event()
            ev.record(st0.stream)
            for k, st, *_ in work:
                if st is not st0:
                    st.stream.wait_event(ev)
    carry_buf = _lib.scalar_buffer(carry, A) if carry is not None else None
    waited, carries = set(), {}
    for i, (k, st, launch, in_ptr, tgt) in enumerate(work):
        before = [w[0] for w in work[:i]]
        for _, st2, *_rest in work[:i]:
            if st2 is not st and (id(st), id(st2)) not in waited:
                st.stream.wait_event(reduced[id(st2)])
                waited.add((id(st), id(st2)))
        carry_dev = None
        if not before and carry_buf is None and in_dev is not None:
            carry_dev = in_dev
        elif before or carry_buf is not None:
            cslot = count[id(st)] + carries.get(id(st), 0)
            carries[id(st)] = carries.get(id(st), 0) + 1
            vals = (ctypes.c_void_p * max(1, len(before)))(*[tot_ptr[j] for j in before])
            carry_dev = st.result_dev_ptr(cslot)
            kernels.launch_kernel("drk_carry_fold", launch, 1, code, opcode, vals, None, len(before),
                                  ctypes.addressof(carry_buf) if carry_buf is not None else None, in_dev, carry_dev)
        _run_segment_scan(T, opcode, exclusive, in_ptr, tgt, launch, init=init_a, carry_dev=carry_dev)
    if not want_partials and not _needs_range_check(T):
        return partials  # nothing to read back: the scans stay asynchronous on their streams
    raw = {}
    for k, st, *_ in work:
        if id(st) not in raw:
            raw[id(st)] = st.fetch_results(count[id(st)])  # waits for the device's scans too
    seen = {}
    for k, st, *_ in work:
        slot = seen.get(id(st), 0)
        seen[id(st)] = slot + 1
        total = np.frombuffer(raw[id(st)][8 * slot : 8 * slot + A.itemsize].tobytes(), dtype=A)[0]
        partials[k] = total.astype(L).item()
    for l in launches.values():
        l.state.synchronize()
    if carry_host_fn is not None:
        carry = carry_host_fn()
    _check_carry_range(op, partials, live, exclusive, init, T, carry)
    return partials


def _scan_lowered(r, out):
    """(runtime, segment count, live segment indices, [(k, lowered input, output Target,
    device state)]) of an aligned scan r -> out, memoised by the structure of both
    (plans.py); device state (pending transfers, staging) is resolved per call."""
    key = None
    if plans._ENABLED:
        dvs = []
        kr, ko = plans.view_key(r, dvs), plans.view_key(out, dvs)
        if kr is not None and ko is not None:
            key = ("scan", kr, ko)
            hit = plans.CACHE.get(key)
            if hit is not None:
                return hit
    in_segs = segments_of(r)
    out_segs = segments_of(out)
    live = [k for k, s in enumerate(in_segs) if len(s)]
    if not live:
        return None, len(in_segs), live, []
    rt = _require_runtime(runtime_of(out, r), "scan")
    lowered = []
    for k in live:
        lw = lower(in_segs[k])
        tgt = lower(out_segs[k]).target
        if not isinstance(tgt, Target):
            raise TypeError("scan output segments must be writable vector storage")
        lowered.append((k, lw, tgt, rt.state_of(out_segs[k].rank)))
    value = (rt, len(in_segs), live, lowered)
    if key is not None:
        plans.CACHE.put(key, dvs, value)
    return value


# Views scanned in a fused kernel (kernels.run_scan_view); False materialises them first.
_FUSE_SCAN_VIEWS = True


def _fused_scan_source(node, lw, tgt, opcode, launch):
    """A view input of a segment scan as a kernels.ScanView (its value cast to the output
    dtype, like store_array's cast, then scanned), or None to materialise it instead (fusion
    off, or an expression the fused loader cannot take)."""
    if not _FUSE_SCAN_VIEWS or tgt.dtype not in _lib.DTYPE_CODE:
        return None
    from . import codegen

    node_t = expr.cast(node, tgt.dtype)
    leaves = kernels._dealias([(tgt, node_t)], lw.leaves, lw.length, launch)
    if kernels.match_scan_view(node_t, leaves, opcode, tgt.dtype) is None:
        try:  # compile (or fetch) the NVRTC loader now, so a failure can fall back
            probe = kernels.ScanView(node_t, leaves, [0] * len(leaves), lw.length)
            codegen.scan_view_plan(probe, tgt.dtype, opcode)
        except codegen.JitError:
            return None
    from .runtime import await_pending

    await_pending(launch.state, [tgt.handle])
    ptrs = kernels.stage_leaves(leaves, launch)
    return kernels.ScanView(node_t, leaves, ptrs, lw.length)


def _run_segment_scan(T, opcode, exclusive, src, tgt, launch, **kw):
    if isinstance(src, kernels.ScanView):
        kernels.run_scan_view(T, opcode, exclusive, src, tgt.ptr(), tgt.length, launch, **kw)
    else:
        run_scan(T, opcode, exclusive, src, tgt.ptr(), tgt.length, launch, **kw)


def _segment_total(T, opcode, src, tgt, launch, result_ptr):
    """The total of one segment's input (the first pass of the multi-device scan) into the
    device address result_ptr, in the scan's accumulator type."""
    if isinstance(src, kernels.ScanView):
        kernels.run_reduce(src.node, src.leaves, src.n, opcode, None, launch, 0, ptrs=src.ptrs,
                           result_ptr=result_ptr)
    else:
        kernels.launch_kernel("drk_reduce", launch, tgt.length, _lib.dtype_code(T), opcode, src, tgt.length,
                              result_ptr, launch.state.reduce_scratch.data_ptr())


def _to_acc(v, A):
    return np.asarray(v).astype(A).item() if np.asarray(v).dtype != A else np.asarray(v).item()


def _offsets(op, partials, carry=None):
    offsets, prefix = [], carry
    for p in partials:
        offsets.append(prefix)
        if p is not None:
            prefix = p if prefix is None else op.fn(prefix, p)
    return offsets


def _check_carry_range(op, partials, live, exclusive, init, T, carry=None):
    """The reference adds the (Python int) carry to an int32 segment with np.add, which
    raises OverflowError once the carry leaves the int32 range (algorithms.py:292-308)."""
    if T.kind not in "iu" or T.itemsize >= 8:
        return
    info = np.iinfo(T)
    offsets = _offsets(op, partials, carry)
    failures = []
    for j, k in enumerate(live):
        off = offsets[k]
        seed = off
        if exclusive:
            seed = init if off is None else op.fn(init, off)
        if seed is None:
            continue
        if not info.min <= int(seed) <= info.max:
            failures.append((j, OverflowError(f"Python integer {int(seed)} out of bounds for {T}")))
    if failures:
        raise AggregateTaskError(failures)


# ----------------------------------------------------------------------------------------
# sort


@_traced
def sort(r, key=None, *, strategy: str | None = None) -> None:
    """In-place ascending sort of a distributed vector (algorithms.py:315-432); with `key`,
    a stable sort by key(x) (the key function is traced like any element function).

    strategy "sample" (the default when the segments live on more than one GPU): the
    reference's distributed sample sort — local sorts, splitters, redistribution into
    per-locale chunks over NVLink, chunk sorts, sweep back (_sort.py).
    strategy "gather" (the default on one GPU): the segments are concatenated in one buffer,
    radix-sorted once and written back in segment order — one sort instead of two when
    there is no second GPU to share the work.  Both give the reference's result."""
    from .containers import VectorSegment
    from .runtime import torch, torch_dtype

    segs = segments_of(r)
    for s_ in segs:
        if not isinstance(s_, VectorSegment):
            raise TypeError("sort needs raw writable storage segments")
    if strategy not in (None, "auto", "gather", "sample"):
        raise ValueError(f"unknown sort strategy {strategy!r}")
    live = [s_ for s_ in segs if len(s_)]
    total = sum(len(s_) for s_ in live)
    if total <= 1:
        return
    rt = _require_runtime(runtime_of(r), "sort")
    if len({s_.dtype for s_ in live}) > 1:
        raise TypeError("sort needs segments of one dtype")
    if strategy in (None, "auto"):
        strategy = "sample" if len({rt.device_of(s_.rank) for s_ in live}) > 1 else "gather"
    if strategy == "sample" and len(segs) > 1:
        from ._sort import sample_sort

        sample_sort(rt, segs, key)
        return
    T = np.dtype(live[0].dtype)
    code = _lib.sort_dtype_code(T)
    states = {rt.state_of(s_.rank).index: rt.state_of(s_.rank) for s_ in live}
    from .runtime import await_pending

    for s_ in live:
        await_pending(rt.state_of(s_.rank), [s_.handle])
    for st in states.values():
        st.synchronize()  # pending writes of every segment land before the gather
    st0 = rt.state_of(live[0].rank)
    t = torch()
    with t.cuda.stream(st0.stream):
        buf = t.empty(total, dtype=torch_dtype(T), device=st0.device)
        alt = t.empty(total, dtype=torch_dtype(T), device=st0.device)
    off = 0
    for s_ in live:
        _lib.call("drk_memcpy_async", buf.data_ptr() + off * T.itemsize, s_.data_ptr(), len(s_) * T.itemsize,
                  st0.index, st0.handle)
        off += len(s_)
    launch = Launch(st0)
    need = ctypes.c_size_t(0)
    if key is None:
        _lib.call("drk_sort_keys", code, buf.data_ptr(), alt.data_ptr(), total, None, ctypes.byref(need),
                  st0.index, st0.handle)
        with t.cuda.stream(st0.stream):
            scratch = t.empty(max(1, need.value), dtype=t.uint8, device=st0.device)
        _lib.call("drk_sort_keys", code, buf.data_ptr(), alt.data_ptr(), total, scratch.data_ptr(),
                  ctypes.byref(need), st0.index, st0.handle)
        result = buf
    else:
        node = expr.trace_cached(key, expr.leaf(0, T), ("sortkey", T.str))
        if node is None or isinstance(node, tuple):
            raise TypeError("sort key must return one value per element")
        K = np.dtype(node.dtype)
        if K not in _lib.SORT_DTYPE_CODE:
            node, K = expr.cast(node, np.int32 if K.kind == "b" else np.float64), np.dtype(
                np.int32 if K.kind == "b" else np.float64)
        with t.cuda.stream(st0.stream):
            kbuf = t.empty(total, dtype=torch_dtype(K), device=st0.device)
            kalt = t.empty(total, dtype=torch_dtype(K), device=st0.device)
            idx = t.empty(total, dtype=t.int64, device=st0.device)
            idx_alt = t.empty(total, dtype=t.int64, device=st0.device)
        tgt = _DeviceTarget(kbuf, K, st0.index)
        run_map([(tgt, node)], [kernels._TensorLeaf(buf, T, total)], total, launch)
        _lib.call("drk_iota", _lib.I64, idx.data_ptr(), total, 0, st0.index, st0.handle)
        _lib.call("drk_sort_pairs", _lib.sort_dtype_code(K), kbuf.data_ptr(), kalt.data_ptr(), idx.data_ptr(),
                  idx_alt.data_ptr(), total, None, ctypes.byref(need), st0.index, st0.handle)
        with t.cuda.stream(st0.stream):
            scratch = t.empty(max(1, need.value), dtype=t.uint8, device=st0.device)
        _lib.call("drk_sort_pairs", _lib.sort_dtype_code(K), kbuf.data_ptr(), kalt.data_ptr(), idx.data_ptr(),
                  idx_alt.data_ptr(), total, scratch.data_ptr(), ctypes.byref(need), st0.index, st0.handle)
        _lib.call("drk_gather", code, alt.data_ptr(), buf.data_ptr(), idx.data_ptr(), total, st0.index, st0.handle)
        result = alt
    off = 0
    for s_ in live:
        _lib.call("drk_memcpy_async", s_.data_ptr(), result.data_ptr() + off * T.itemsize, len(s_) * T.itemsize,
                  st0.index, st0.handle)
        off += len(s_)
    st0.synchronize()


class _DeviceTarget(Target):
    """A write target over a raw device tensor (temporaries of sort)."""

    def __init__(self, tensor, dtype, device):
        self.handle = None
        self.start = 0
        self.length = tensor.numel()
        self.dtype = np.dtype(dtype)
        self._t = tensor
        self._device = device

    def ptr(self):
        return self._t.data_ptr()

    @property
    def device(self):
        return self._device


# ----------------------------------------------------------------------------------------
# copy / fill / transform


@_traced
def copy(src, dst) -> None:
    """Element copy between equal-length ranges: aligned pairs segment by segment, else
    chunks at the union of both sides' boundaries (algorithms.py:468-503).  Sources may
    be lazy views (fused into the copy kernel); host arrays on either side are
    transferred over PCIe."""
    if len(src) != len(dst):
        raise ValueError(f"copy length mismatch: source {len(src)}, destination {len(dst)}")
    if len(src) == 0:
        return
    key = None
    if plans._ENABLED:
        dvs = []
        ks, kd = plans.view_key(src, dvs), plans.view_key(dst, dvs)
        if ks is not None and kd is not None:
            key = ("copy", ks, kd)
    plan = plans.CACHE.get(key) if key is not None else None
    if plan is None:
        rt = runtime_of(dst, src)
        s_seg, d_seg = has_segments(src), has_segments(dst)
        if s_seg and d_seg and is_aligned(src, dst):
            pairs = [(s, d) for s, d in zip(segments_of(src), segments_of(dst)) if len(s)]
        else:
            src_list = segments_of(src) if s_seg else [_views._as_piece(src, len(src))]
            dst_list = segments_of(dst) if d_seg else [_views._as_piece(dst, len(dst))]
            pairs = [tuple(ch.components) for ch in _views.realign_segments([src_list, dst_list])]
        rt = _require_runtime(rt, "copy")
        work = []
        for s, d in pairs:
            ls = lower(s)
            if isinstance(ls.value, tuple):
                raise TypeError("copy source elements must be scalars")
            if isinstance(d, _views.LocalPiece):
                work.append((ls, d, None))
                continue
            tgt = lower(d).target
            if isinstance(tgt, ReadOnly):
                raise TypeError(f"cannot write through read-only {tgt.what}")
            work.append((ls, tgt, rt.state_of(d.rank)))
        plan = [rt, work, None]
        if key is not None:
            plans.CACHE.put(key, dvs, plan)
    rt, work, bound = plan
    if bound and kernels._PROFILE is None:
        for b in bound:
            b()
        if _SYNC_ALGORITHMS:
            rt.synchronize()
        return
    launches = []
    for ls, d, st in work:
        if st is None:
            _copy_to_host(rt, ls, d, launches)
            continue
        launch = Launch(st)
        run_map([(d, ls.value)], ls.leaves, ls.length, launch)
        launches.append(launch)
    _finish(rt, launches)
    if bound is None and key is not None:
        bs = [kernels.bind_map([(d, ls.value)], ls.leaves, ls.length, st) if st is not None else None
              for ls, d, st in work]
        plan[2] = _bind_launches(bs)


def _copy_to_host(rt, ls, piece, launches):
    if not piece.writable:
        raise TypeError("cannot write through a sequence converted to a local piece")
    node = ls.value
    rank = ls.rank if ls.rank is not None else 0
    st = rt.state_of(rank)
    launch = Launch(st)
    host = piece.array
    if node.op == "leaf" and ls.leaves[node.value].kind == "array" and node.dtype == host.dtype \
            and host.flags.c_contiguous:
        _lib.call("drk_memcpy_async", host.ctypes.data, ls.leaves[node.value].ptr(), host.nbytes, st.index,
                  st.handle)
        st.synchronize()
        return
    from .runtime import torch, torch_dtype

    t = torch()
    with t.cuda.stream(st.stream):
        tmp = t.empty(ls.length, dtype=torch_dtype(host.dtype), device=st.device)
    run_map([(_DeviceTarget(tmp, host.dtype, st.index), node)], ls.leaves, ls.length, launch)
    st.synchronize()
    host[...] = tmp.cpu().numpy()


@_traced
def fill(r, value) -> None:
    """Set every element of a writable range to value."""
    for_each(r, lambda _x: value, vectorized=True)


@_traced
def transform(src, dst, fn) -> None:
    """dst[i] = fn(src[i]) — the reference spells this copy(views.transform(src, fn), dst)
    (algorithms.py:468-503, tests/test_algorithms.py:376-381)."""
    copy(_views.transform(src, fn), dst)

"""Lowered segment work -> libdrk launches.

Each algorithm hands this module per-segment work already lowered by views.py: a list
of leaves (device buffers, index ranges, host slices) and an expression over them.  The
expression is first matched against the ahead-of-time catalogue of hand-written sm_100a
kernels in libdrk.so — copy, fill, iota, scale, add, triad, Black-Scholes, reduce,
dot, scan — which cover the benchmarked paths (bench.py:87-126 of the reference).  Any
other expression is compiled once by NVRTC from generated CUDA (codegen.py) and cached.
There is no host evaluation path.
"""

from __future__ import annotations

import ctypes

import numpy as np

from . import _lib
from .views import Leaf

OPCODES = {"add": _lib.ADD, "multiply": _lib.MUL, "minimum": _lib.MIN, "maximum": _lib.MAX}

# Optional live kernel timing: when enabled, every launch is bracketed by CUDA events on
# the stream it is launched on (bench.py uses this inside its timed region).
_PROFILE = None


class profile:
    """Context manager collecting {kernel name: [(start_event, end_event, elements)]}."""

    def __enter__(self):
        global _PROFILE
        self.records = {}
        _PROFILE = self.records
        return self

    def __exit__(self, *exc):
        global _PROFILE
        _PROFILE = None
        return False

    def summary(self):
        """{name: (launches, total_ms, total_elements)} — call after synchronising."""
        out = {}
        for name, recs in self.records.items():
            ms = sum(s.elapsed_time(e) for s, e, _ in recs)
            out[name] = (len(recs), ms, sum(n for _, _, n in recs))
        return out


def launch_kernel(name, launch_ctx, n, *args, key=None):
    """Call libdrk entry `name` (device and stream appended) on launch_ctx; `key` names the
    launch in kernels.profile (default: the entry point, drk_*_ex reported without _ex)."""
    if _PROFILE is None:
        _lib.call(name, *args, launch_ctx.device, launch_ctx.stream)
        return
    from .runtime import torch

    t = torch()
    s, e = t.cuda.Event(enable_timing=True), t.cuda.Event(enable_timing=True)
    s.record(launch_ctx.state.stream)
    _lib.call(name, *args, launch_ctx.device, launch_ctx.stream)
    e.record(launch_ctx.state.stream)
    if key is None:
        key = name[:-3] if name.endswith("_ex") else name  # drk_scan_ex is reported as drk_scan
        if name == "drk_black_scholes_ex" and args[1] & _lib.BS_FAST:
            key = "drk_black_scholes:fast"
    _PROFILE.setdefault(key, []).append((s, e, n))


def launch_jit(mod, kernel, grid, block, smem, buf, nbytes, lctx, n):
    """Launch an NVRTC kernel (single packed-struct argument) on lctx's stream."""
    args = (mod.handle, kernel.encode(), grid, block, smem, buf, nbytes, lctx.device, lctx.stream)
    if _PROFILE is None:
        _lib.call("drk_jit_launch", *args)
        return
    from .runtime import torch

    t = torch()
    s, e = t.cuda.Event(enable_timing=True), t.cuda.Event(enable_timing=True)
    s.record(lctx.state.stream)
    _lib.call("drk_jit_launch", *args)
    e.record(lctx.state.stream)
    _PROFILE.setdefault("jit:" + kernel, []).append((s, e, n))


class Launch:
    """Execution context of one segment: device, stream, device state, keep-alive list."""

    __slots__ = ("state", "device", "stream", "keep")

    def __init__(self, state):
        self.state = state
        self.device = state.index
        self.stream = state.handle
        self.keep = []


def stage_leaves(leaves, launch: Launch):
    """Make every leaf readable by a kernel on launch.device: host slices are copied to
    the device (asynchronously, on the segment stream).  Returns per-leaf pointers (0 for
    index leaves)."""
    from .runtime import await_pending

    await_pending(launch.state, [lf.handle for lf in leaves if lf.kind == "array" and lf.handle is not None])
    # leaves on other GPUs are read over NVLink: order this launch after the work already
    # enqueued on their devices (an asynchronous scan may still be writing them)
    waited = set()
    for lf in leaves:
        if lf.kind == "array" and lf.handle is not None and lf.device != launch.device and lf.device not in waited:
            waited.add(lf.device)
            launch.state.stream.wait_event(lf.handle.runtime.device_state(lf.device).compute_event())
    ptrs = []
    for lf in leaves:
        if lf.kind == "array":
            ptrs.append(lf.ptr())
        elif lf.kind == "host":
            from .runtime import torch

            t = torch()
            arr = np.ascontiguousarray(lf.host)
            with t.cuda.stream(launch.state.stream):
                dev = t.from_numpy(arr).to(launch.state.device, non_blocking=False)
            launch.keep.append(dev)
            ptrs.append(dev.data_ptr())
        else:
            ptrs.append(0)
    return ptrs


def _is_leaf(node, leaves, kind="array"):
    return node.op == "leaf" and leaves[node.value].kind == kind


def _uniform(node, dtype):
    """All loop dtypes of node equal dtype."""
    return node.loop is not None and all(d == dtype for d in node.loop)


def _scalar_arg(value, dtype):
    return _lib.scalar_buffer(value, dtype)


# ----------------------------------------------------------------------------------------
# map


def match_map(node, leaves, out_dtype):
    """Catalogue entry for `out <- node` or None.  Returns (fn_name, arg_builder)."""
    T = np.dtype(out_dtype)
    if T not in _lib.DTYPE_CODE:
        return None
    code = _lib.DTYPE_CODE[T]
    if node.op == "const":
        return ("drk_fill", lambda out, n, ptrs, L: (code, out, n, _keep(L, _scalar_arg(node.value, T))))
    if node.op == "leaf":
        lf = leaves[node.value]
        if lf.kind == "index":
            return ("drk_iota", lambda out, n, ptrs, L: (code, out, n, lf.base))
        if lf.dtype == T:
            k = node.value
            return ("drk_copy", lambda out, n, ptrs, L: (code, out, ptrs[k], n))
        return None
    if node.dtype != T:
        return None
    if node.op == "multiply" and _uniform(node, T):
        a, b = node.args
        if a.op == "const" and _is_leaf(b, leaves):
            a, b = b, a
        if b.op == "const" and _is_leaf(a, leaves):
            k, alpha = a.value, b.value
            return ("drk_scale", lambda out, n, ptrs, L: (code, out, ptrs[k], n, _keep(L, _scalar_arg(alpha, T))))
    if node.op == "add" and _uniform(node, T):
        a, b = node.args
        if _is_leaf(a, leaves) and _is_leaf(b, leaves):
            ka, kb = a.value, b.value
            return ("drk_add", lambda out, n, ptrs, L: (code, out, ptrs[ka], ptrs[kb], n))
        # b + alpha*c (either operand order; IEEE add and multiply commute bit-exactly)
        for x, y in ((a, b), (b, a)):
            if _is_leaf(x, leaves) and y.op == "multiply" and _uniform(y, T):
                p, q = y.args
                if p.op == "const" and _is_leaf(q, leaves):
                    p, q = q, p
                if q.op == "const" and _is_leaf(p, leaves):
                    kb, kc, alpha = x.value, p.value, q.value
                    return ("drk_triad", lambda out, n, ptrs, L: (
                        code, out, ptrs[kb], ptrs[kc], n, _keep(L, _scalar_arg(alpha, T))))
    if node.op in ("call:black_scholes", "call:black_scholes_fast") and T.kind == "f" and all(
            _is_leaf(a, leaves) and a.dtype == T for a in node.args):
        ks = [a.value for a in node.args]
        flags = _lib.BS_FAST if node.op == "call:black_scholes_fast" else 0
        return ("drk_black_scholes_ex", lambda out, n, ptrs, L: (code, flags, out, *[ptrs[k] for k in ks], n))
    return None


def _keep(launch, buf):
    launch.keep.append(buf)
    return buf


def run_map(writes, leaves, n, launch: Launch):
    """Write each (Target, node) of `writes` for n elements on launch's device."""
    if n == 0 or not writes:
        return
    from .runtime import await_pending

    await_pending(launch.state, [t.handle for t, _ in writes if t.handle is not None])
    leaves = _dealias(writes, leaves, n, launch)
    ptrs = stage_leaves(leaves, launch)
    if len(writes) == 1:
        tgt, node = writes[0]
        m = match_map(node, leaves, tgt.dtype)
        if m is not None:
            name, build = m
            launch_kernel(name, launch, n, *build(tgt.ptr(), n, ptrs, launch))
            _release_peers(leaves, launch)
            return
    from . import codegen

    codegen.run_map(writes, leaves, ptrs, n, launch)
    _release_peers(leaves, launch)


class BoundMap:
    """One map launch with every argument fixed (a plan's lowered segment on its own GPU):
    re-issued as a single entry-point call.  Used by cached for_each / copy plans; profiled
    runs and launches that need per-call work (host slices, peer reads, aliasing
    snapshots) take run_map instead."""

    __slots__ = ("fn", "args", "name", "handles", "keep", "state")

    def __call__(self):
        for h in self.handles:
            if h._pending:
                from .runtime import await_pending

                await_pending(self.state, self.handles)
                break
        rc = self.fn(*self.args)
        if rc:
            _lib.check(rc, self.name)


class BoundGraph:
    """Several BoundMaps on one stream captured into one CUDA graph (drk_graph_*): a cached
    plan over many segments of one GPU replays with a single launch."""

    __slots__ = ("exec", "state", "handles", "keep", "__weakref__")

    def __call__(self):
        for h in self.handles:
            if h._pending:
                from .runtime import await_pending

                await_pending(self.state, self.handles)
                break
        rc = _lib.fn("drk_graph_launch")(self.exec, self.state.index, self.state.handle)
        if rc:
            _lib.check(rc, "drk_graph_launch")

    def __del__(self):
        try:
            if self.exec:
                _lib.fn("drk_graph_destroy")(self.exec)
        except Exception:  # pragma: no cover - interpreter teardown
            pass


def capture(bounds):
    """A BoundGraph replaying `bounds` (several BoundMaps of one device state), or None when
    they do not share a stream or the capture fails (the caller keeps the BoundMaps)."""
    if len(bounds) < 2 or any(b.state is not bounds[0].state for b in bounds):
        return None
    st = bounds[0].state
    for b in bounds:  # settle pending transfers outside the capture
        for h in b.handles:
            if h._pending:
                from .runtime import await_pending

                await_pending(st, b.handles)
                break
    if _lib.fn("drk_graph_begin")(st.index, st.handle):
        return None
    ok = True
    for b in bounds:
        if b.fn(*b.args):
            ok = False
            break
    ex = ctypes.c_void_p()
    rc = _lib.fn("drk_graph_end")(st.index, st.handle, ctypes.byref(ex))
    if not ok or rc or not ex.value:
        if ex.value:
            _lib.fn("drk_graph_destroy")(ex)
        return None
    g = BoundGraph()
    g.exec = ex.value
    g.state = st
    g.handles = [h for b in bounds for h in b.handles]
    g.keep = [b.keep for b in bounds]
    return g


def bind_map(writes, leaves, n, state):
    """A BoundMap for run_map(writes, leaves, n) on `state`'s GPU, or None when the launch
    needs per-call work."""
    if n == 0 or not writes:
        return None
    for lf in leaves:
        if lf.kind == "host" or (lf.kind == "array" and lf.device != state.index):
            return None
    for tgt, _ in writes:
        if tgt.handle is None:
            return None
        for lf in leaves:
            if lf.kind == "array" and lf.handle is tgt.handle and lf.start != tgt.start:
                return None  # an aliasing snapshot per call
    launch = Launch(state)
    ptrs = [lf.ptr() if lf.kind == "array" else 0 for lf in leaves]
    b = BoundMap()
    b.state = state
    b.handles = [t.handle for t, _ in writes] + [lf.handle for lf in leaves if lf.kind == "array" and lf.handle is not None]
    m = match_map(writes[0][1], leaves, writes[0][0].dtype) if len(writes) == 1 else None
    if m is not None:
        name, build = m
        b.name = name
        b.fn = _lib.fn(name)
        b.args = (*build(writes[0][0].ptr(), n, ptrs, launch), state.index, state.handle)
    else:
        from . import codegen

        mod, kernel, grid, buf, nbytes = codegen.map_launch(writes, leaves, ptrs, n, state.index)
        b.name = "drk_jit_launch"
        b.fn = _lib.fn("drk_jit_launch")
        b.args = (mod.handle, kernel.encode(), grid, codegen.BLOCK, 0, buf, nbytes, state.index, state.handle)
        launch.keep.append(buf)
    b.keep = launch.keep
    return b


def _release_peers(leaves, launch: Launch):
    """After a kernel that reads other GPUs' memory over NVLink: their streams wait for it, so
    nothing they run later (a write, or the reuse of freed memory) overtakes the read."""
    done = set()
    for lf in leaves:
        if lf.kind == "array" and lf.handle is not None and lf.device != launch.device and lf.device not in done:
            done.add(lf.device)
            lf.handle.runtime.device_state(lf.device).stream.wait_event(launch.state.compute_event())


def _dealias(writes, leaves, n, launch):
    """Leaves that overlap a written range at a different offset are snapshotted first
    (the reference computes the whole right-hand side before storing, views.py:176)."""
    out = list(leaves)
    for i, lf in enumerate(leaves):
        if lf.kind != "array":
            continue
        for tgt, _ in writes:
            if lf.handle is tgt.handle and lf.start != tgt.start:
                lo, hi = lf.start, lf.start + n
                if lo < tgt.start + n and tgt.start < hi:
                    from .runtime import torch

                    t = torch()
                    with t.cuda.stream(launch.state.stream):
                        snap = t.empty(n, dtype=lf.handle.span().dtype, device=launch.state.device)
                    _lib.call("drk_memcpy_async", snap.data_ptr(), lf.ptr(), n * lf.dtype.itemsize,
                              launch.device, launch.stream)
                    launch.keep.append(snap)
                    out[i] = _TensorLeaf(snap, lf.dtype, n)
                    break
    return out


class _TensorLeaf(Leaf):
    __slots__ = ("tensor",)

    def __init__(self, tensor, dtype, n):
        super().__init__("array", n, dtype)
        self.tensor = tensor

    def ptr(self):
        return self.tensor.data_ptr()


# ----------------------------------------------------------------------------------------
# reduce


def catalogue_reduce(node, leaves, opcode, device):
    """The batched form of run_reduce's catalogue match for a segment whose leaves are plain
    device arrays on `device`: ("reduce", dtype code, ptr) or ("dot", code, ptr_x, ptr_y),
    else None."""
    T = node.dtype
    if opcode is None or T not in _lib.DTYPE_CODE:
        return None
    code = _lib.DTYPE_CODE[T]

    def arr(k):
        lf = leaves[k]
        return lf.kind == "array" and lf.handle is not None and lf.device == device

    if node.op == "leaf" and arr(node.value):
        return ("reduce", code, leaves[node.value].ptr())
    if (opcode == _lib.ADD and node.op == "multiply" and _uniform(node, T)
            and all(_is_leaf(a, leaves) and arr(a.value) for a in node.args)):
        a, b = node.args
        return ("dot", code, leaves[a.value].ptr(), leaves[b.value].ptr())
    return None


def run_reduce(node, leaves, n, opcode, combiner, launch: Launch, slot: int, *, ptrs=None, result_ptr=None):
    """Reduce `node` over n elements into host result slot `slot` of launch.state (value in
    drk_acc_dtype(node.dtype, op) for catalogue ops; read with fetch_host_results), or into
    the device address result_ptr.  ptrs: the leaves' pointers if already staged."""
    if ptrs is None:
        ptrs = stage_leaves(leaves, launch)
    st = launch.state
    # stored straight into mapped pinned memory unless a device slot is given
    res = result_ptr if result_ptr is not None else st.host_result_dev_ptr(slot)
    T = node.dtype
    if opcode is not None and T in _lib.DTYPE_CODE:
        code = _lib.DTYPE_CODE[T]
        if node.op == "leaf" and leaves[node.value].kind == "array":
            launch_kernel("drk_reduce", launch, n, code, opcode, ptrs[node.value], n, res,
                                st.reduce_scratch.data_ptr())
            return
        if (opcode == _lib.ADD and node.op == "multiply" and _uniform(node, T)
                and all(_is_leaf(a, leaves) for a in node.args)):
            a, b = node.args
            launch_kernel("drk_dot", launch, n, code, ptrs[a.value], ptrs[b.value], n, res,
                                st.reduce_scratch.data_ptr())
            return
    from . import codegen

    codegen.run_reduce(node, leaves, ptrs, n, opcode, combiner, launch, slot, result_ptr=result_ptr)


# ----------------------------------------------------------------------------------------
# scan


_SCAN_SCRATCH_BYTES = {}


def run_scan(dtype, opcode, exclusive, in_ptr, out_ptr, n, lctx: Launch, *, init=None, carry_value=None,
             carry_dev=None, seg_total_slot=None, carry_out_slot=None, chained=False, scratch_index=0):
    """One drk_scan over a plain device buffer (the caller materialises views first).

    chained: this scan continues a chain of segment scans on the stream (its carry_dev is
    written by the scan enqueued just before; drk_scan_ex DRK_SCAN_CHAINED), and
    scratch_index alternates the scratch buffer between consecutive scans of the chain."""
    T = np.dtype(dtype)
    code = _lib.dtype_code(T)
    A = _lib.acc_dtype(T, opcode)
    st = lctx.state
    nbytes = _scan_scratch_bytes(code, opcode, n)
    scratch = st.scan_scratch(nbytes, scratch_index)
    init_buf = _keep(lctx, _scalar_arg(init, A)) if init is not None else None
    carry_buf = _keep(lctx, _scalar_arg(carry_value, A)) if carry_value is not None else None
    launch_kernel(
        "drk_scan_ex", lctx, n, code, opcode, 1 if exclusive else 0, _lib.SCAN_CHAINED if chained else 0,
        in_ptr, out_ptr, n,
        ctypes.addressof(init_buf) if init_buf is not None else None,
        ctypes.addressof(carry_buf) if carry_buf is not None else None,
        carry_dev,
        st.result_dev_ptr(seg_total_slot) if seg_total_slot is not None else None,
        st.result_dev_ptr(carry_out_slot) if carry_out_slot is not None else None,
        scratch.data_ptr(), scratch.numel(),
    )


# ----------------------------------------------------------------------------------------
# scan of a fused view


class ScanView:
    """What a fused segment scan reads: `node` (already cast to the output dtype) over
    `leaves`, whose device pointers are `ptrs` (kernels.stage_leaves)."""

    __slots__ = ("node", "leaves", "ptrs", "n")

    def __init__(self, node, leaves, ptrs, n):
        self.node = node
        self.leaves = leaves
        self.ptrs = ptrs
        self.n = n

    def vec_ok(self) -> bool:
        return all(self.ptrs[k] % 16 == 0 for k in _array_slots(self.node, self.leaves))


def _array_slots(node, leaves):
    from . import expr

    return sorted(k for k in expr.leaves_used(node) if leaves[k].kind in ("array", "host"))


def match_scan_view(node, leaves, opcode, T):
    """AOT fused-scan loader for `node` (dtype T) with add: (kind, words) or None.
    PRODUCT x*y (zip|transform dot shape); AFFINE alpha*x, alpha*x + beta, x + beta, x - beta
    — exactly numpy's roundings (one per operation, no FMA)."""
    T = np.dtype(T)
    if opcode != _lib.ADD or T not in _lib.DTYPE_CODE or node.dtype != T or not _uniform(node, T):
        return None
    from .codegen import const_bits

    if node.op == "multiply":
        a, b = node.args
        if _is_leaf(a, leaves) and _is_leaf(b, leaves):
            return _lib.VIEW_PRODUCT, ("leaf", a.value), ("leaf", b.value)
        if b.op == "const" and _is_leaf(a, leaves):
            a, b = b, a
        if a.op == "const" and _is_leaf(b, leaves):
            return _lib.VIEW_AFFINE, ("leaf", b.value), const_bits(a.value, T), 0, 0
        return None
    if node.op in ("add", "subtract"):
        x, c = node.args
        if node.op == "add" and x.op == "const":
            x, c = c, x
        if c.op != "const":
            return None
        beta = c.value if node.op == "add" else -np.asarray(c.value, dtype=T)
        if _is_leaf(x, leaves):
            return _lib.VIEW_AFFINE, ("leaf", x.value), const_bits(1, T), const_bits(beta, T), 1
        if x.op == "multiply" and _uniform(x, T):
            p, q = x.args
            if q.op == "const" and _is_leaf(p, leaves):
                p, q = q, p
            if p.op == "const" and _is_leaf(q, leaves):
                return _lib.VIEW_AFFINE, ("leaf", q.value), const_bits(p.value, T), const_bits(beta, T), 1
    return None


def run_scan_view(T, opcode, exclusive, view: ScanView, out_ptr, n, lctx: Launch, *, combiner=None, init=None,
                  carry_value=None, carry_dev=None, seg_total_slot=None, carry_out_slot=None, chained=False,
                  scratch_index=0):
    """One fused scan of a view segment: out = scan(view) with the view's values computed from
    its leaves inside the scan kernel (AOT drk_scan_view for product / affine views with add,
    an NVRTC module otherwise) — no intermediate array."""
    T = np.dtype(T)
    st = lctx.state
    A = _lib.acc_dtype(T, opcode) if opcode is not None else T
    init_buf = _keep(lctx, _scalar_arg(init, A)) if init is not None else None
    carry_buf = _keep(lctx, _scalar_arg(carry_value, A)) if carry_value is not None else None
    tail = (
        1 if exclusive else 0,
    )
    common = (out_ptr, n,
              ctypes.addressof(init_buf) if init_buf is not None else None,
              ctypes.addressof(carry_buf) if carry_buf is not None else None,
              carry_dev,
              st.result_dev_ptr(seg_total_slot) if seg_total_slot is not None else None,
              st.result_dev_ptr(carry_out_slot) if carry_out_slot is not None else None)
    flags = _lib.SCAN_CHAINED if chained else 0
    m = match_scan_view(view.node, view.leaves, opcode, T) if combiner is None else None
    if m is not None:
        kind, *parts = m
        words = [view.ptrs[x[1]] if isinstance(x, tuple) else x for x in parts]
        wbuf = _keep(lctx, (ctypes.c_uint64 * len(words))(*[w & 0xFFFFFFFFFFFFFFFF for w in words]))
        code = _lib.dtype_code(T)
        nbytes = _scan_scratch_bytes(code, opcode, n)
        scratch = st.scan_scratch(nbytes, scratch_index)
        launch_kernel("drk_scan_view_ex", lctx, n, kind, code, opcode, *tail, flags, wbuf, len(words),
                      1 if view.vec_ok() else 0, *common, scratch.data_ptr(), scratch.numel(),
                      key="drk_scan_view:" + ("product" if kind == _lib.VIEW_PRODUCT else "affine"))
        return
    from . import codegen

    mod, words, geom = codegen.scan_view_plan(view, T, opcode, combiner)
    wbuf = _keep(lctx, (ctypes.c_uint64 * len(words))(*[w & 0xFFFFFFFFFFFFFFFF for w in words]))
    nbytes = int(_lib.load().drk_jit_scan_scratch_bytes(n, 256 * geom[4]))
    scratch = st.scan_scratch(nbytes, scratch_index)
    args = (mod.handle, T.itemsize, A.itemsize, *geom, *tail, flags, wbuf, len(words), 1 if view.vec_ok() else 0,
            *common, scratch.data_ptr(), scratch.numel(), st.index, st.handle)
    if _PROFILE is None:
        _lib.call("drk_jit_scan_view", *args)
        return
    from .runtime import torch

    t = torch()
    s_, e_ = t.cuda.Event(enable_timing=True), t.cuda.Event(enable_timing=True)
    s_.record(st.stream)
    _lib.call("drk_jit_scan_view", *args)
    e_.record(st.stream)
    _PROFILE.setdefault("drk_scan_view:jit", []).append((s_, e_, n))


def _scan_scratch_bytes(code, opcode, n):
    key = (code, opcode, n)
    nbytes = _SCAN_SCRATCH_BYTES.get(key)
    if nbytes is None:
        nbytes = _SCAN_SCRATCH_BYTES[key] = int(_lib.load().drk_scan_scratch_bytes(code, opcode, n))
    return nbytes

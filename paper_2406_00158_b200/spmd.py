"""One process per GPU: the cross-rank combine steps over torch.distributed (NCCL).

The shp runtime combines per-segment results on its driver (reference
algorithms.py:146-149 for reduce, :256-262 for the scan carry).  When the segments of a
vector are spread over processes — one process per B200, launched by torchrun — those
two driver steps become collectives:

  reduce:  each rank folds its own segments' device partials, then one NCCL all-gather
           of (has, partial) pairs and the reference's ascending fold from init on every
           rank (so the result does not depend on NCCL's reduction order).
  scan:    each rank computes its segment total on the device, one NCCL all-gather of
           (has, total) pairs, then rank r folds the totals of ranks < r into its carry
           and runs the single-pass device scan with that carry.  This is the
           reduce-then-scan schedule: 3n element touches at P > 1 against 2n on one GPU.

Element-wise work (STREAM, Black-Scholes, copy of aligned data) needs no exchange.
The same functions run over gloo with CPU tensors, which is how the exchange logic is
tested on hosts without GPUs.
"""

from __future__ import annotations

import operator
import os

import numpy as np

from . import _lib

_NP_TO_TORCH = None


def _torch():
    import torch

    return torch


def _dist():
    import torch.distributed as dist

    return dist


class Group:
    """A torch.distributed process group (default: the world)."""

    def __init__(self, group=None, combine=None):
        dist = _dist()
        if not dist.is_initialized():
            raise RuntimeError("torch.distributed is not initialised (launch with torchrun)")
        self.group = group
        self.rank = dist.get_rank(group)
        self.size = dist.get_world_size(group)
        self.backend = dist.get_backend(group)
        # how the reduce / scan exchange of (has, value) pairs runs: "collective" — an
        # all-gather of the backend (NCCL on the rank's stream); "ipc" — the library's own
        # kernel over peer memory (every rank's mailbox mapped with CUDA IPC, no NCCL call)
        # "auto" (the default) uses "ipc" when every rank can map every other rank's mailbox
        # and a trial exchange returns every rank's pair, else "collective" — decided
        # collectively on first use (_decide)
        combine = combine or os.environ.get("DRK_SPMD_COMBINE", "auto")
        if combine not in ("collective", "ipc", "auto"):
            raise ValueError(f"unknown combine {combine!r} (collective, ipc or auto)")
        if combine == "ipc" and self.size > _lib.COMM_MAX_RANKS:
            raise ValueError(f"combine='ipc' supports up to {_lib.COMM_MAX_RANKS} ranks")
        if combine == "auto" and self.size > _lib.COMM_MAX_RANKS:
            combine = "collective"
        self._combine = combine
        self._mailbox = None

    @property
    def combine(self):
        return self._combine

    def decide(self, state):
        """Resolve combine="auto" (collective: every rank must call it at the same point)."""
        if self._combine != "auto":
            return self._combine
        dist = _dist()
        mb, ok = None, True
        try:
            mb = _Mailbox(self, state)
            ok = mb.trial()
        except Exception:  # no IPC / peer access between these GPUs: the backend's collective
            ok = False
        flags = [None] * self.size
        dist.all_gather_object(flags, ok, group=self.group)
        if all(flags):
            self._mailbox, self._combine = mb, "ipc"
        else:
            self._combine = "collective"
            del mb
        return self._combine

    def exchange_buffers(self, state):
        """Persistent buffers of gather_pairs on the rank's GPU (reused call after call: every
        exchange is complete, and read back, before the next one starts)."""
        bufs = getattr(self, "_xbufs", None)
        if bufs is None:
            bufs = self._xbufs = _ExchangeBuffers(self, state)
        return bufs

    def scan_buffers(self, state):
        """Persistent device buffers of the scan's carry exchange on the rank's GPU."""
        b = getattr(self, "_sbufs", None)
        if b is None:
            b = self._sbufs = _ScanBuffers(self, state)
        return b

    def mailbox(self, state):
        """The rank's peer-memory mailbox (created collectively on first use)."""
        if self._mailbox is None:
            self._mailbox = _Mailbox(self, state)
        return self._mailbox

    def device(self):
        t = _torch()
        if self.backend == "nccl":
            return t.device("cuda", t.cuda.current_device())
        return t.device("cpu")


class _ExchangeBuffers:
    """The (has, value) pair in mapped pinned memory (host-written, kernel-read), its device
    copy for NCCL, the gathered pairs + a status word on the device, and their host copy."""

    def __init__(self, group: Group, state):
        import ctypes

        t = _torch()
        n = 2 * group.size + 1
        self.pair_host = t.zeros(2, dtype=t.int64, pin_memory=True)
        self.pair_np = self.pair_host.numpy()
        self.pair_host_ptr = self.pair_host.data_ptr()
        dev = ctypes.c_void_p()
        _lib.call("drk_mapped_ptr", self.pair_host_ptr, ctypes.byref(dev))
        self.pair_dev = _Ptr(int(dev.value))
        with t.cuda.stream(state.stream):
            self.buf = t.zeros(2, dtype=t.int64, device=state.device)
            self.out = t.zeros(n, dtype=t.int64, device=state.device)
        self.status = self.out[2 * group.size:]
        self.status_ptr = self.status.data_ptr()
        self.host = t.zeros(n, dtype=t.int64, pin_memory=True)
        self.host_np = self.host.numpy()


class _ScanBuffers:
    """pair (has, total), gathered pairs followed by the exchange status word, and the carry."""

    def __init__(self, group: Group, state):
        t = _torch()
        with t.cuda.stream(state.stream):
            self.pair = t.zeros(2, dtype=t.int64, device=state.device)
            g = t.zeros(2 * group.size + 1, dtype=t.int64, device=state.device)
            self.carry = t.zeros(1, dtype=t.int64, device=state.device)
        self.gathered = g
        self.status = g[2 * group.size:]
        self.one = np.array([1], dtype=np.int64)


class _Ptr:
    """A raw device address with the data_ptr() of a tensor."""

    __slots__ = ("p",)

    def __init__(self, p):
        self.p = p

    def data_ptr(self):
        return self.p


class _Mailbox:
    """Every rank's mailbox mapped into this rank (drk_ipc_*), for drk_mailbox_allgather: the
    all-gather of one (has, value) pair per rank as one kernel over NVLink peer memory."""

    TIMEOUT_NS = 120 * 10**9  # a rank that never arrives: an error after two minutes, not a hang

    def __init__(self, group: Group, state):
        import ctypes

        dist = _dist()
        self.group, self.state = group, state
        own = ctypes.c_void_p()
        _lib.call("drk_ipc_alloc", 2 * group.size * 32, state.index, ctypes.byref(own))
        self.own = own.value
        handle = ctypes.create_string_buffer(64)
        _lib.call("drk_ipc_handle", self.own, handle)
        handles = [None] * group.size
        dist.all_gather_object(handles, handle.raw, group=group.group)
        peers, self.opened = [], []
        for j, h in enumerate(handles):
            if j == group.rank:
                peers.append(self.own)
                continue
            p = ctypes.c_void_p()
            _lib.call("drk_ipc_open", ctypes.create_string_buffer(h, 64), state.index, ctypes.byref(p))
            peers.append(p.value)
            self.opened.append(p.value)
        self.peers = (ctypes.c_void_p * group.size)(*peers)
        self.epoch = 0
        dist.barrier(group=group.group)  # every mailbox mapped before anyone writes

    def trial(self, timeout_ns=10 * 10**9) -> bool:
        """One exchange of (1, rank): True when every rank's pair arrived in place."""
        t = _torch()
        st, g = self.state, self.group
        with t.cuda.stream(st.stream):
            pair = t.tensor([1, g.rank], dtype=t.int64).to(st.device)
            out = t.zeros(2 * g.size + 1, dtype=t.int64, device=st.device)
        self.epoch += 1
        _lib.call("drk_mailbox_allgather", pair.data_ptr(), self.peers, g.size, g.rank, self.own, self.epoch,
                  timeout_ns, out.data_ptr(), out.data_ptr() + 16 * g.size, st.index, st.handle)
        st.synchronize()
        got = out.cpu().numpy()
        want = np.array([[1, j] for j in range(g.size)], dtype=np.int64).ravel()
        return bool(np.array_equal(got[: 2 * g.size], want) and (got[2 * g.size] & 0xFFFFFFFF) == 0)

    def allgather(self, pair, gathered, status):
        """Enqueue the exchange on the rank's stream (pair: 16 device bytes; gathered: world x
        16 device bytes; status: a device int32 that becomes 1 if a rank did not arrive)."""
        self.epoch += 1
        st, g = self.state, self.group
        _lib.call("drk_mailbox_allgather", pair.data_ptr(), self.peers, g.size, g.rank, self.own, self.epoch,
                  self.TIMEOUT_NS, gathered.data_ptr(), status.data_ptr(), st.index, st.handle)

    def __del__(self):
        try:
            for p in self.opened:
                _lib.call("drk_ipc_close", p)
            _lib.call("drk_ipc_free", self.own)
        except Exception:  # pragma: no cover - interpreter teardown
            pass


_REDUCE_OPS = {"add": "SUM", "multiply": "PRODUCT", "minimum": "MIN", "maximum": "MAX"}
_PYOPS = {"add": operator.add, "multiply": operator.mul, "minimum": min, "maximum": max}


def _identity(opname, dtype):
    dtype = np.dtype(dtype)
    if opname == "add":
        return dtype.type(0)
    if opname == "multiply":
        return dtype.type(1)
    if dtype.kind == "f":
        return dtype.type(np.inf if opname == "minimum" else -np.inf)
    info = np.iinfo(dtype)
    return dtype.type(info.max if opname == "minimum" else info.min)


def _encode(value, A):
    """An accumulator/partial value as 8 raw bytes (float64 for floats, int64 for ints:
    exact for every partial dtype of the device kernels)."""
    wide = np.float64 if np.dtype(A).kind == "f" else np.int64
    return np.array([value], dtype=wide).view(np.int64)[0]


def _decode(bits, A):
    wide = np.float64 if np.dtype(A).kind == "f" else np.int64
    return np.asarray(np.array([bits], dtype=np.int64).view(wide)[0]).astype(A)[()]


# dtypes a gathered value can carry; the pair's has-word is 1 + the sender's dtype index, so
# every rank decodes every value in its sender's dtype (a rank without elements does not
# know the dtype of the others' partials)
_PAIR_DTYPES = [np.dtype(d) for d in (np.float32, np.float64, np.int32, np.int64, np.uint32, np.uint64,
                                      np.int16, np.int8, np.uint16, np.uint8, np.float16, np.bool_)]


def gather_pairs(value, acc_dtype, group: Group, state=None) -> list:
    """All-gather of one optional value per rank -> list indexed by rank (None = that rank
    had no elements).  With NCCL the (has, value) pair is written by a kernel, gathered on
    the rank's compute stream and read back by a kernel into mapped pinned memory: no
    copy engine is involved, so the exchange never queues behind bulk PCIe transfers."""
    t = _torch()
    dist = _dist()
    A = np.dtype(acc_dtype)
    pair = np.zeros(2, dtype=np.int64)
    if value is not None:
        pair[0], pair[1] = 1 + _PAIR_DTYPES.index(A), _encode(value, A)
    ipc = state is not None and group.decide(state) == "ipc"
    if (group.backend == "nccl" or ipc) and state is not None:
        x = group.exchange_buffers(state)
        if ipc:
            # the pair goes straight from the host into mapped memory, which the exchange
            # kernel reads as device memory: one kernel, one readback, one wait
            x.pair_np[:] = pair
            _lib.call("drk_memset_async", x.status_ptr, 0, 8, state.index, state.handle)
            group.mailbox(state).allgather(x.pair_dev, x.out, x.status)
        else:
            x.pair_np[:] = pair
            # a kernel copy from mapped memory (a copy-engine transfer could queue behind bulk
            # PCIe traffic on another stream)
            _lib.call("drk_copy", _lib.I64, x.buf.data_ptr(), x.pair_dev.p, 2, state.index, state.handle)
            with t.cuda.device(state.index), t.cuda.stream(state.stream):
                dist.all_gather_into_tensor(x.out[: 2 * group.size], x.buf, group=group.group)
        _lib.call("drk_readback", x.host.data_ptr(), x.out.data_ptr(), 8 * (2 * group.size + 1), state.index,
                  state.handle)
        state.synchronize()
        h = x.host_np
        if ipc and h[2 * group.size] & 0xFFFFFFFF:
            raise RuntimeError("spmd: a rank did not reach the peer-memory exchange in time")
        got = h[: 2 * group.size].reshape(group.size, 2)
    else:
        x = t.from_numpy(pair).to(group.device())
        outs = t.empty(2 * group.size, dtype=t.int64, device=x.device)
        dist.all_gather_into_tensor(outs, x, group=group.group)
        got = outs.cpu().numpy().reshape(group.size, 2)
    return [_decode(v, _PAIR_DTYPES[h - 1]) if h else None for h, v in got]


def allreduce_partial(partial, opname: str, acc_dtype, group: Group, state=None):
    """Combine one partial per rank (None = rank had no elements), folded in rank order
    like the reference's driver fold of segment partials (algorithms.py:147-149), so the
    result does not depend on the collective's reduction order."""
    fold = _PYOPS[opname]
    acc = None
    for q in gather_pairs(partial, acc_dtype, group, state):
        if q is not None:
            acc = q if acc is None else fold(acc, q)
    return acc


def gather_totals(total, acc_dtype, group: Group, state=None) -> list:
    """All-gather of per-rank (has, total) -> list indexed by rank (None = no elements)."""
    return gather_pairs(total, acc_dtype, group, state)


def exclusive_carry(total, opname: str, acc_dtype, group: Group, state=None):
    """Fold of the totals of ranks before this one (None if all of them were empty)."""
    totals = gather_totals(total, acc_dtype, group, state)
    fold = _PYOPS[opname]
    carry = None
    for r in range(group.rank):
        q = totals[r]
        if q is not None:
            carry = q if carry is None else fold(carry, q)
    return carry


# ----------------------------------------------------------------------------------------
# distributed algorithms over a rank-local vector that is block r of a global vector


def reduce(local, init, op, group: Group):
    """Global reduce of the concatenation of every rank's `local` range: the rank's device
    partial, an all-gather of one partial per rank, then the reference's ascending driver
    fold from `init` (algorithms.py:146-149) — bit-identical to the one-process result
    when every rank holds one segment."""
    from . import algorithms as A

    op = A.as_binary_op(op)
    opname = getattr(op.ufunc, "__name__", None)
    if opname not in _REDUCE_OPS:
        raise TypeError("distributed reduce needs add/multiply/minimum/maximum")
    from . import plans

    rt = A.runtime_of(local)
    opk = A._op_key(op)
    key, dvs, plan = plans.lookup("spmd_reduce", local, opk) if opk is not None else (None, None, None)
    if plan is None:  # the rank's lowered pieces, memoised like algorithms.reduce (False: none)
        pieces = A._pieces(local)
        plan = plans.store(key, dvs, A._ReducePlan(rt, pieces, op) if pieces else False)
    partial = None
    vdt = None
    if plan:
        parts = plan.run()
        vdt = np.asarray(parts[0]).dtype
        for p in parts:
            partial = p if partial is None else op.fn(partial, p)
    code_dt = vdt if vdt is not None else _value_dtype(local)
    L = A._partial_dtype(op, code_dt) if code_dt in _lib.DTYPE_CODE else code_dt
    acc = init
    for q in gather_pairs(partial, L, group, _state_of(rt, local)):
        if q is not None:
            acc = op.fn(acc, q)
    return acc.item() if isinstance(acc, np.generic) else acc


def _value_dtype(local):
    """Element dtype of a rank-local range that may hold no elements: the vector's dtype, or
    for a view the dtype of its lowered (empty) segment expression — so an empty rank decodes
    and folds the gathered partials in the same dtype as the ranks that have elements."""
    dt = getattr(local, "dtype", None)
    if dt is not None:
        return np.dtype(dt)
    from . import algorithms as A
    from .views import lower

    for seg in A.segments_of(local):
        try:
            value = lower(seg).value
        except Exception:  # pragma: no cover - a view that cannot lower has no device dtype
            continue
        if not isinstance(value, tuple):
            return np.dtype(value.dtype)
    return np.dtype(np.float64)


def _state_of(rt, local):
    """The device state of the rank's (first) segment, if the runtime has devices."""
    if rt is None or getattr(rt, "backend", None) != "cuda":
        return None
    from . import algorithms as A

    segs = A.segments_of(local)
    rank = next((s.rank for s in segs if getattr(s, "rank", None) is not None), 0)
    return rt.state_of(rank)


def inclusive_scan(local, out, group: Group, op=None):
    return _scan(local, out, group, op, exclusive=False, init=None)


def exclusive_scan(local, out, init, group: Group, op=None):
    return _scan(local, out, group, op, exclusive=True, init=init)


def _scan(local, out, group, op, exclusive, init):
    from . import algorithms as A

    op = A.as_binary_op(op if op is not None else A.add)
    opname = getattr(op.ufunc, "__name__", None)
    if opname not in _REDUCE_OPS:
        raise TypeError("distributed scan needs add/multiply/minimum/maximum")
    T = np.dtype(out.dtype)
    opcode = A.OPCODES[opname]
    acc = _lib.acc_dtype(T, opcode)
    pieces = A._pieces(local)
    st = _state_of(A.runtime_of(local), local)  # every rank, so the collective choices agree
    if pieces and st is not None and (group.backend == "nccl" or group.decide(st) == "ipc") \
            and group.size <= _lib.CARRY_MAX:
        # device path: local totals -> (has, total) pair -> all-gather -> carry, all on the
        # rank's stream; the host only checks the int32 carry range after the scan
        A._scan_impl(local, out, op, exclusive, init, want_partials=False,
                     carry_hook=_device_carry_hook(group, _lib.dtype_code(T), opcode, opname, acc))
        return None
    total = None
    if pieces:
        rt = A.runtime_of(local)
        for p in A._segment_partials(rt, pieces, op):
            total = p if total is None else op.fn(total, p)
    carry = exclusive_carry(None if total is None else acc.type(total), opname, acc, group, st)
    A._scan_impl(local, out, op, exclusive, init, carry=carry, want_partials=False)
    return None


def _device_carry_hook(group: Group, code: int, opcode: int, opname: str, acc):
    """carry_hook for algorithms._scan_impl: between the scan's two passes, fold the rank's
    segment totals into a (has, total) pair (drk_carry_fold), all-gather the pairs with NCCL
    on the rank's stream, and fold the totals of lower ranks into the carry (drk_carry_fold
    again) — no host round trip.  Returns (carry device pointer or None, host-value function)."""
    import ctypes

    t = _torch()
    dist = _dist()
    A = np.dtype(acc)

    def hook(total_ptrs, st):
        ipc = group.decide(st) == "ipc"
        # persistent per (group, GPU): consecutive scans use them in stream order
        b = group.scan_buffers(st)
        pair, gathered, carry, status = b.pair, b.gathered, b.carry, b.status
        _lib.call("drk_fill", _lib.I64, pair.data_ptr(), 1, b.one.ctypes.data, st.index, st.handle)
        if ipc:
            _lib.call("drk_memset_async", status.data_ptr(), 0, 8, st.index, st.handle)
        vals = (ctypes.c_void_p * len(total_ptrs))(*total_ptrs)
        _lib.call("drk_carry_fold", code, opcode, vals, None, len(total_ptrs), None, None, pair.data_ptr() + 8,
                  st.index, st.handle)
        if ipc:
            group.mailbox(st).allgather(pair, gathered, status)
        else:
            with t.cuda.device(st.index), t.cuda.stream(st.stream):
                dist.all_gather_into_tensor(gathered[: 2 * group.size], pair, group=group.group)
        r = group.rank
        carry_ptr = None
        if r > 0:
            g = gathered.data_ptr()
            vals = (ctypes.c_void_p * r)(*[g + 16 * j + 8 for j in range(r)])
            has = (ctypes.c_void_p * r)(*[g + 16 * j for j in range(r)])
            _lib.call("drk_carry_fold", code, opcode, vals, has, r, None, None, carry.data_ptr(), st.index,
                      st.handle)
            carry_ptr = carry.data_ptr()

        def host_value():
            """The carry as the host path computes it (after the scan has completed)."""
            host = t.empty(2 * group.size + 1, dtype=t.int64, pin_memory=True)
            _lib.call("drk_readback", host.data_ptr(), gathered.data_ptr(), 8 * (2 * group.size + 1), st.index,
                      st.handle)
            st.synchronize()
            if ipc and int(host.numpy()[2 * group.size]) & 0xFFFFFFFF:
                raise RuntimeError("spmd: a rank did not reach the peer-memory exchange in time")
            raw = host.numpy().tobytes()
            fold = _PYOPS[opname]
            c = None
            for j in range(r):
                if np.frombuffer(raw[16 * j: 16 * j + 8], dtype=np.int64)[0]:
                    v = np.frombuffer(raw[16 * j + 8: 16 * j + 8 + A.itemsize], dtype=A)[0]
                    c = v if c is None else fold(c, v)
            _keep = (pair, gathered, carry, status)  # noqa: F841 - alive until the scan has run
            return c

        return carry_ptr, host_value

    return hook


# ----------------------------------------------------------------------------------------
# distributed sample sort, one process per GPU (reference algorithms.py:315-432)


def _exchange(send, sizes_out, sizes_in, group: Group, st):
    """all-to-all-v of a 1-D device tensor's bytes: sizes_out[j] bytes (consecutive) to rank
    j, sizes_in[j] from rank j, in rank order.  NCCL runs on the rank's stream (NVLink);
    gloo (the shared-GPU test mode) stages through host memory."""
    t = _torch()
    dist = _dist()
    total_in = int(sum(sizes_in))
    src = send.view(t.uint8) if send.numel() else send.new_empty(0, dtype=t.uint8)
    if group.backend == "nccl":
        with t.cuda.device(st.index), t.cuda.stream(st.stream):
            out = t.empty(total_in, dtype=t.uint8, device=st.device)
            dist.all_to_all_single(out, src, [int(s) for s in sizes_in], [int(s) for s in sizes_out],
                                   group=group.group)
        return out
    st.synchronize()
    host_in = src.cpu()
    host_out = t.empty(total_in, dtype=t.uint8)
    dist.all_to_all_single(host_out, host_in, [int(s) for s in sizes_in], [int(s) for s in sizes_out],
                           group=group.group)
    with t.cuda.stream(st.stream):
        return host_out.to(st.device, non_blocking=False)


def sort(local, group: Group, key=None) -> None:
    """Sort the global vector whose block r is rank r's `local` DistributedVector, in place,
    ascending (by key if given, stably): after the call rank r's block holds sorted positions
    [offset_r, offset_r + len(local)) — the reference's sample sort with one segment per rank:
      1. the rank's elements sorted on its GPU (the library's radix sort; key functions run on
         the device and the elements follow a stable pair sort);
      2. P-1 evenly spaced samples per rank, all-gathered; splitters picked from the pool like
         the reference's driver (algorithms.py:358-367);
      3. counts of the rank's run per destination (drk_sort_bounds) all-gathered;
      4. one all-to-all-v moves the runs (NCCL over NVLink), a stable sort of the received
         chunk (runs arrive in rank order, so ties keep their global order);
      5. a second all-to-all-v restores every rank's length (the reference's sweep back).
    Every rank must call it (a collective)."""
    from . import _sort as S
    from . import algorithms as A
    from . import kernels
    from .runtime import await_pending, torch_dtype

    t = _torch()
    dist = _dist()
    P, r = group.size, group.rank
    rt = A.runtime_of(local)
    segs = A.segments_of(local)
    for s in segs:
        if not hasattr(s, "handle"):
            raise TypeError("sort needs raw writable storage segments")
    live = [s for s in segs if len(s)]
    T = np.dtype(local.dtype)
    vcode = _lib.sort_dtype_code(T)
    states = {rt.state_of(s.rank).index for s in segs}
    if len(states) > 1:
        raise ValueError("spmd.sort: a rank's segments must live on one GPU")
    st = rt.state_of(segs[0].rank)
    for s in live:
        await_pending(st, [s.handle])
    n_r = sum(len(s) for s in segs)
    # the rank's block as one device buffer
    with t.cuda.stream(st.stream):
        vals = t.empty(n_r, dtype=torch_dtype(T), device=st.device)
    pos = 0
    for s in live:
        _lib.call("drk_memcpy_async", vals.data_ptr() + pos * T.itemsize,
                  s.handle.data_ptr() + s.start * T.itemsize, len(s) * T.itemsize, st.index, st.handle)
        pos += len(s)
    node, K = (S._key_node(key, T) if key is not None else (None, T))
    kcode = _lib.sort_dtype_code(K)
    keep = []

    def keys_of(v, m):
        """Device keys of the m elements of v (the values themselves without a key)."""
        if node is None:
            return v
        from .algorithms import _DeviceTarget

        with t.cuda.stream(st.stream):
            k = t.empty(m, dtype=torch_dtype(K), device=st.device)
        if m:
            kernels.run_map([(_DeviceTarget(k, K, st.index), node)], [kernels._TensorLeaf(v, T, m)], m,
                            kernels.Launch(st))
        return k

    def local_sort(v, m):
        k = keys_of(v, m)
        if m > 1:
            keep.extend(S._sort_buffer(st, kcode, k, m, None if node is None else v, vcode))
        return k

    # 1. local sort
    keys = local_sort(vals, n_r)
    # 2. samples -> splitters
    spos = S._sorted_positions(n_r, P)
    if spos:
        with t.cuda.stream(st.stream):
            idx = t.tensor(spos, dtype=t.int64).to(st.device)
            smp = keys[idx]
        st.synchronize()
        samples = smp.cpu().numpy()
    else:
        samples = np.empty(0, dtype=K)
    pools = [None] * P
    dist.all_gather_object(pools, samples, group=group.group)
    pool = np.concatenate([p for p in pools if len(p)]) if any(len(p) for p in pools) else np.empty(0, dtype=K)
    pool = pool[np.argsort(pool, kind="stable")]
    m = len(pool)
    split = np.ascontiguousarray(pool[[(j + 1) * m // P for j in range(P - 1)]]) if m else np.empty(0, dtype=K)
    # 3. counts of this run per destination
    if P > 1 and n_r and len(split) == P - 1:
        with t.cuda.stream(st.stream):
            split_d = t.from_numpy(split).to(st.device, non_blocking=False)
            bnd = t.empty(P - 1, dtype=t.int64, device=st.device)
        _lib.call("drk_sort_bounds", kcode, keys.data_ptr(), n_r, split_d.data_ptr(), P - 1, bnd.data_ptr(),
                  st.index, st.handle)
        st.synchronize()
        counts = np.diff(np.concatenate(([0], bnd.cpu().numpy(), [n_r])))
    else:
        counts = np.zeros(P, dtype=np.int64)
        counts[min(r, P - 1) if not len(split) else 0] = n_r
    table = [None] * P
    dist.all_gather_object(table, (n_r, counts.astype(np.int64)), group=group.group)
    lens = np.array([x[0] for x in table], dtype=np.int64)
    cmat = np.stack([x[1] for x in table])          # cmat[k][j]: rank k's elements for chunk j
    # 4. the runs to their chunks, then a stable chunk sort
    chunk = _exchange(vals, counts * T.itemsize, cmat[:, r] * T.itemsize, group, st).view(torch_dtype(T))
    S_r = int(cmat[:, r].sum())
    local_sort(chunk, S_r)
    # 5. back to every rank's own length: chunk r covers global [C_r, C_r + S_r)
    sizes = cmat.sum(axis=0)
    C = np.concatenate(([0], np.cumsum(sizes)))
    off = np.concatenate(([0], np.cumsum(lens)))
    send = [max(0, min(C[r + 1], off[q + 1]) - max(C[r], off[q])) for q in range(P)]
    recv = [max(0, min(C[q + 1], off[r + 1]) - max(C[q], off[r])) for q in range(P)]
    result = _exchange(chunk, np.array(send) * T.itemsize, np.array(recv) * T.itemsize, group, st)
    pos = 0
    for s in live:
        _lib.call("drk_memcpy_async", s.handle.data_ptr() + s.start * T.itemsize,
                  result.data_ptr() + pos * T.itemsize, len(s) * T.itemsize, st.index, st.handle)
        pos += len(s)
    st.synchronize()
    del keep

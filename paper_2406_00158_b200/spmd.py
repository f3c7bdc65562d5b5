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

    def __init__(self, group=None):
        dist = _dist()
        if not dist.is_initialized():
            raise RuntimeError("torch.distributed is not initialised (launch with torchrun)")
        self.group = group
        self.rank = dist.get_rank(group)
        self.size = dist.get_world_size(group)
        self.backend = dist.get_backend(group)

    def device(self):
        t = _torch()
        if self.backend == "nccl":
            return t.device("cuda", t.cuda.current_device())
        return t.device("cpu")


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
    if group.backend == "nccl" and state is not None:
        with t.cuda.stream(state.stream):
            buf = t.empty(2, dtype=t.int64, device=state.device)
            out = t.empty(2 * group.size, dtype=t.int64, device=state.device)
        for k in range(2):
            w = np.array([pair[k]], dtype=np.int64)
            _lib.call("drk_fill", _lib.I64, buf.data_ptr() + 8 * k, 1, w.ctypes.data, state.index, state.handle)
        with t.cuda.device(state.index), t.cuda.stream(state.stream):
            dist.all_gather_into_tensor(out, buf, group=group.group)
        host = t.empty(2 * group.size, dtype=t.int64, pin_memory=True)
        _lib.call("drk_readback", host.data_ptr(), out.data_ptr(), 16 * group.size, state.index, state.handle)
        state.synchronize()
        got = host.numpy().reshape(group.size, 2)
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
    pieces = A._pieces(local)
    rt = A.runtime_of(local)
    partial = None
    vdt = None
    if pieces:
        parts = A._segment_partials(rt, pieces, op)
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
    st = _state_of(A.runtime_of(local), local) if pieces else None
    if pieces and st is not None and group.backend == "nccl" and group.size <= _lib.CARRY_MAX:
        # device path: local totals -> (has, total) pair -> all-gather -> carry, all on the
        # rank's stream; the host only checks the int32 carry range after the scan
        return A._scan_impl(local, out, op, exclusive, init,
                            carry_hook=_device_carry_hook(group, _lib.dtype_code(T), opcode, opname, acc))
    total = None
    if pieces:
        rt = A.runtime_of(local)
        for p in A._segment_partials(rt, pieces, op):
            total = p if total is None else op.fn(total, p)
    carry = exclusive_carry(None if total is None else acc.type(total), opname, acc, group, st)
    return A._scan_impl(local, out, op, exclusive, init, carry=carry)


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
        with t.cuda.stream(st.stream):
            pair = t.zeros(2, dtype=t.int64, device=st.device)
            gathered = t.empty(2 * group.size, dtype=t.int64, device=st.device)
            carry = t.zeros(1, dtype=t.int64, device=st.device)
        one = np.array([1], dtype=np.int64)
        _lib.call("drk_fill", _lib.I64, pair.data_ptr(), 1, one.ctypes.data, st.index, st.handle)
        vals = (ctypes.c_void_p * len(total_ptrs))(*total_ptrs)
        _lib.call("drk_carry_fold", code, opcode, vals, None, len(total_ptrs), None, None, pair.data_ptr() + 8,
                  st.index, st.handle)
        with t.cuda.device(st.index), t.cuda.stream(st.stream):
            dist.all_gather_into_tensor(gathered, pair, group=group.group)
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
            host = t.empty(2 * group.size, dtype=t.int64, pin_memory=True)
            _lib.call("drk_readback", host.data_ptr(), gathered.data_ptr(), 16 * group.size, st.index, st.handle)
            st.synchronize()
            raw = host.numpy().tobytes()
            fold = _PYOPS[opname]
            c = None
            for j in range(r):
                if np.frombuffer(raw[16 * j: 16 * j + 8], dtype=np.int64)[0]:
                    v = np.frombuffer(raw[16 * j + 8: 16 * j + 8 + A.itemsize], dtype=A)[0]
                    c = v if c is None else fold(c, v)
            _keep = (pair, gathered, carry)  # noqa: F841 - alive until the scan has run
            return c

        return carry_ptr, host_value

    return hook

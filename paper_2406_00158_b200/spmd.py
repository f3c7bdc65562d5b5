"""One process per GPU: the cross-rank combine steps over torch.distributed (NCCL).

The shp runtime combines per-segment results on its driver (reference
algorithms.py:146-149 for reduce, :256-262 for the scan carry).  When the segments of a
vector are spread over processes — one process per B200, launched by torchrun — those
two driver steps become collectives:

  reduce:  each rank folds its own segments' device partials, then one NCCL all-reduce
           of a single accumulator-typed element (float32 sums travel as float64,
           int32 sums as int64, exactly like the device accumulators).
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


def allreduce_partial(partial, opname: str, acc_dtype, group: Group):
    """Combine one accumulator-typed partial per rank (None = rank had no elements)."""
    t = _torch()
    dist = _dist()
    A = np.dtype(acc_dtype)
    val = _identity(opname, A) if partial is None else A.type(partial)
    x = t.from_numpy(np.array([val], dtype=A)).to(group.device())
    has = t.tensor([0 if partial is None else 1], dtype=t.int64, device=group.device())
    dist.all_reduce(x, op=getattr(dist.ReduceOp, _REDUCE_OPS[opname]), group=group.group)
    dist.all_reduce(has, op=dist.ReduceOp.SUM, group=group.group)
    if int(has.item()) == 0:
        return None
    return x.cpu().numpy()[0]


def gather_totals(total, acc_dtype, group: Group) -> list:
    """All-gather of per-rank (has, total) -> list indexed by rank (None = no elements)."""
    t = _torch()
    dist = _dist()
    A = np.dtype(acc_dtype)
    pair = np.zeros(2, dtype=np.float64 if A.kind == "f" else np.int64)
    if total is not None:
        pair[0], pair[1] = 1, total
    x = t.from_numpy(pair).to(group.device())
    out = [t.empty_like(x) for _ in range(group.size)]
    dist.all_gather(out, x, group=group.group)
    res = []
    for o in out:
        h, v = o.cpu().numpy()
        res.append(A.type(v) if h else None)
    return res


def exclusive_carry(total, opname: str, acc_dtype, group: Group):
    """Fold of the totals of ranks before this one (None if all of them were empty)."""
    totals = gather_totals(total, acc_dtype, group)
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
    """Global reduce of the concatenation of every rank's `local` range."""
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
    code_dt = vdt if vdt is not None else np.dtype(getattr(local, "dtype", np.float64))
    acc = _lib.acc_dtype(code_dt, A.OPCODES[opname]) if code_dt in _lib.DTYPE_CODE else code_dt
    total = allreduce_partial(partial, opname, acc, group)
    if total is None:
        return init.item() if isinstance(init, np.generic) else init
    L = A._partial_dtype(op, code_dt)
    r = op.fn(init, np.asarray(total).astype(L)[()])
    return r.item() if isinstance(r, np.generic) else r


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
    acc = _lib.acc_dtype(T, A.OPCODES[opname])
    pieces = A._pieces(local)
    total = None
    if pieces:
        rt = A.runtime_of(local)
        for p in A._segment_partials(rt, pieces, op):
            total = p if total is None else op.fn(total, p)
    carry = exclusive_carry(None if total is None else acc.type(total), opname, acc, group)
    return A._scan_impl(local, out, op, exclusive, init, carry=carry)

"""ORACLE — CPU restatement of the reference's hot path (test infrastructure only).

This module is the parity checker and the CPU baseline, never the product: only
tests/, __graft_entry__.smoke() and bench.py (its `cpu_baseline` leg and
`--impl reference`) may import it.  The shipped package (paper_2406_00158_b200) has no
host compute path.

It restates, in numpy, exactly what the reference package `segrange`
(/root/reference/pkg/src/segrange, pure Python + numpy + scipy) does on the
distributed-vector path, with the same numpy calls so that results are bit-identical to
the reference on the same inputs:

  block partition          core.py:108-130      Distribution.block
  splitmix64 / unit_doubles repro.py:21-40
  CRC-32 checksum          repro.py:43-53
  reduce                   algorithms.py:135-162  per-segment ufunc.reduce, ascending fold
  dot_product              bench.py:87-90         zip|transform(t[0]*t[1])|reduce
  stream_triad             bench.py:93-99         a = b + alpha*c (numpy, two roundings)
  inclusive/exclusive scan algorithms.py:169-308  local accumulate, driver prefix, offset/seed
  black_scholes_call       bench.py:102-116       (scipy.special.erf, fp64 internals)
  sort                     algorithms.py:315-432  sample sort (local sort, splitters, chunks)

Pinning: tests/test_oracle.py checks every function here against golden vectors produced
by the real reference (tests/golden/make_golden.py imports /root/reference and writes
tests/golden/*.npz + golden.json), and against the reference's own known-answer tests
(dot [1,2,3].[4,5,6] = 32, scan [1,2,3,4] -> [1,3,6,10] with partials [3,7], ...).

Third-party arithmetic: numpy (ufunc reduce = pairwise sum, accumulate = sequential) and
scipy.special.erf, unpinned by the reference (pyproject: numpy>=1.24, scipy>=1.10); the
fixtures were generated with numpy 2.3.5 / scipy 1.18.1 (NEP 50 promotion).
"""

from __future__ import annotations

import math
import os
import zlib
from concurrent.futures import ThreadPoolExecutor

import numpy as np

# ---------------------------------------------------------------------------------------
# data generation (repro.py:21-53)

_G = np.uint64(0x9E3779B97F4A7C15)
_M1 = np.uint64(0xBF58476D1CE4E5B9)
_M2 = np.uint64(0x94D049BB133111EB)


def splitmix64(seed, start, count):
    i = np.arange(start + 1, start + count + 1, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = np.uint64(seed & 0xFFFFFFFFFFFFFFFF) + i * _G
        z = (z ^ (z >> np.uint64(30))) * _M1
        z = (z ^ (z >> np.uint64(27))) * _M2
        return z ^ (z >> np.uint64(31))


def unit_doubles(seed, start, count):
    return (splitmix64(seed, start, count) >> np.uint64(11)).astype(np.float64) * (2.0 ** -53)


def uniform_doubles(seed, start, count, lo, hi):
    return lo + (hi - lo) * unit_doubles(seed, start, count)


def mod_ints(seed, start, count, modulus, offset):
    """(splitmix64 % modulus).astype(int64) + offset — the acceptance tests' integer data
    (test_acceptance.py:70-74 uses modulus 2001, offset -1000)."""
    return (splitmix64(seed, start, count) % np.uint64(modulus)).astype(np.int64) + offset


def checksum(arr) -> str:
    if np.isscalar(arr) or (isinstance(arr, np.ndarray) and arr.ndim == 0):
        arr = np.asarray([arr])
    a = np.ascontiguousarray(np.asarray(arr))
    return format(zlib.crc32(a.astype(a.dtype.newbyteorder("<"), copy=False).tobytes()) & 0xFFFFFFFF, "08x")


def generate(desc: dict, dtype) -> np.ndarray:
    """Inputs described by a golden-fixture record."""
    kind = desc["kind"]
    if kind == "unit":
        x = unit_doubles(desc["seed"], desc["start"], desc["n"])
    elif kind == "uniform":
        x = uniform_doubles(desc["seed"], desc["start"], desc["n"], desc["lo"], desc["hi"])
    elif kind == "mod":
        x = mod_ints(desc["seed"], desc["start"], desc["n"], desc["modulus"], desc["offset"])
    elif kind == "arange":
        x = np.arange(desc["start"], desc["start"] + desc["n"])
    else:
        raise ValueError(kind)
    return x.astype(dtype)


# ---------------------------------------------------------------------------------------
# partition (core.py:108-130)


def block_lengths(n, p):
    if n == 0:
        return []
    s = -(-n // p)
    return [min(s, max(0, n - i * s)) for i in range(p)]


def block_segments(x, p, lengths=None):
    lengths = block_lengths(len(x), p) if lengths is None else list(lengths)
    out, off = [], 0
    for ln in lengths:
        out.append(x[off : off + ln])
        off += ln
    return out


# ---------------------------------------------------------------------------------------
# a thread-per-segment executor, like the reference Runtime (runtime.py:130-245)

def _run(tasks, threads):
    if threads <= 1 or len(tasks) <= 1:
        return [t() for t in tasks]
    with ThreadPoolExecutor(max_workers=threads) as ex:
        futs = [ex.submit(t) for t in tasks]
        return [f.result() for f in futs]


# ---------------------------------------------------------------------------------------
# algorithms


def reduce(x, p, init=0, ufunc=np.add, threads=1, lengths=None):
    """algorithms.py:135-162: ufunc.reduce per non-empty segment, fold ascending on init."""
    segs = [s for s in block_segments(x, p, lengths) if len(s)]
    partials = _run([lambda s=s: ufunc.reduce(s) for s in segs], threads)
    acc, fold = init, _pyop(ufunc)  # BinaryOp.fn: operator.add / operator.mul / min / max
    for q in partials:
        acc = fold(acc, q)
    return acc.item() if isinstance(acc, np.generic) else acc


def dot(x, y, p, threads=1):
    """bench.py:87-90 via algorithms.reduce: np.add.reduce(x*y) per segment, 0.0 + ..."""
    xs, ys = block_segments(x, p), block_segments(y, p)
    pairs = [(a, b) for a, b in zip(xs, ys) if len(a)]
    partials = _run([lambda a=a, b=b: np.add.reduce(a * b) for a, b in pairs], threads)
    acc = 0.0
    for q in partials:
        acc = acc + q
    return acc.item() if isinstance(acc, np.generic) else acc


def triad(b, c, alpha=3.0, p=1, threads=1):
    """bench.py:93-99: a = b + alpha * c with numpy's weak-scalar promotion."""
    bs, cs = block_segments(b, p), block_segments(c, p)
    parts = _run([lambda u=u, v=v: u + alpha * v for u, v in zip(bs, cs) if len(u)], threads)
    return np.concatenate(parts) if parts else np.empty(0, dtype=b.dtype)


def scan(x, p, out_dtype=None, exclusive=False, init=None, ufunc=np.add, threads=1, lengths=None):
    """algorithms.py:234-308 on aligned input/output.  Returns (out, partials)."""
    out_dtype = np.dtype(out_dtype or x.dtype)
    segs = block_segments(x, p, lengths)
    lens = [len(s) for s in segs]
    out_segs = [np.zeros(len(s), dtype=out_dtype) for s in segs]
    live = [k for k, s in enumerate(segs) if len(s)]

    def local(k):  # _local_scan_task, algorithms.py:277-289
        inc = ufunc.accumulate(np.asarray(segs[k]))
        if exclusive:
            sh = np.empty_like(inc)
            sh[0] = inc[0]
            sh[1:] = inc[:-1]
            out_segs[k][...] = sh
        else:
            out_segs[k][...] = inc
        return inc[-1].item()

    res = _run([lambda k=k: local(k) for k in live], threads)
    partials = [None] * len(segs)
    for k, q in zip(live, res):
        partials[k] = q
    offsets, prefix = [], None
    for q in partials:  # driver loop, algorithms.py:256-262 (op.fn = operator.add etc.)
        offsets.append(prefix)
        if q is not None:
            prefix = q if prefix is None else _pyop(ufunc)(prefix, q)

    def fix(k):  # _offset_task / _seed_task, algorithms.py:292-308
        off = offsets[k]
        if exclusive:
            seed = init if off is None else _pyop(ufunc)(init, off)
            vals = out_segs[k]
            new = np.empty_like(vals)
            new[0] = seed
            if len(vals) > 1:
                new[1:] = ufunc(seed, vals[1:])
            out_segs[k][...] = new
        elif off is not None:
            out_segs[k][...] = ufunc(off, out_segs[k])

    _run([lambda k=k: fix(k) for k in live if exclusive or offsets[k] is not None], threads)
    out = np.concatenate(out_segs) if out_segs else np.empty(0, dtype=out_dtype)
    return out, partials


def trimmed_lengths(lengths, f, l):
    """views.py:271-292 trim_segments on segment lengths: window [f, l), no empty pieces."""
    out, pos = [], 0
    for n in lengths:
        lo, hi = max(f, pos), min(l, pos + n)
        if hi > lo:
            out.append(hi - lo)
        pos += n
    return out


def realigned_lengths(*length_lists):
    """views.py:444-477 realign_segments: chunk lengths at the union of all boundaries."""
    cuts = set()
    for lst in length_lists:
        cuts.update(np.cumsum([0] + list(lst)).tolist())
    cuts = sorted(cuts)
    return [b - a for a, b in zip(cuts, cuts[1:]) if b > a]


def sample_sort(x, p, key=None, lengths=None):
    """algorithms.py:315-432 (paper Alg. 5): local sort of every segment, n-1 evenly spaced
    samples per segment, splitters from the pooled samples, redistribution into chunks by
    searchsorted(splitters, key, side="left"), chunk sort, chunks swept back in order.
    Returns the sorted copy of x (the reference sorts in place)."""
    segs = [np.array(sg) for sg in block_segments(x, p, lengths)]
    n_chunks = len(segs)
    if len(x) <= 1 or n_chunks == 0:
        return np.array(x)

    def kv(a):
        return a if key is None else key(a)

    def local_sort(a):
        if key is None:
            a.sort()
        else:
            a[...] = a[np.argsort(kv(a), kind="stable")]

    live = [sg for sg in segs if len(sg)]
    for sg in live:
        local_sort(sg)
    if n_chunks == 1:
        return segs[0]
    samples = []
    for sg in live:
        m = len(sg)
        samples.append(sg.copy() if m < n_chunks - 1 else sg[[(j + 1) * m // n_chunks for j in range(n_chunks - 1)]])
    pool = np.concatenate(samples)
    pool = pool[np.argsort(kv(pool), kind="stable")]
    m = len(pool)
    split_keys = kv(pool[[(j + 1) * m // n_chunks for j in range(n_chunks - 1)]])
    chunks = [[] for _ in range(n_chunks)]
    for sg in live:
        idx = np.searchsorted(split_keys, kv(sg), side="left")
        for j in range(n_chunks):
            chunks[j].append(sg[idx == j])
    out = []
    for parts in chunks:
        c = np.concatenate(parts) if parts else np.empty(0, dtype=x.dtype)
        local_sort(c)
        out.append(c)
    return np.concatenate(out)


def _pyop(ufunc):
    import operator

    return {np.add: operator.add, np.multiply: operator.mul, np.minimum: min, np.maximum: max}[ufunc]


def black_scholes(spot, strike, rate, volatility, expiry):
    """bench.py:102-116 (fp64 internals from np.asarray(spot, float64); scipy erf)."""
    from scipy.special import erf

    spot = np.asarray(spot, dtype=np.float64)
    vol = volatility * np.sqrt(expiry)
    discount = np.exp(-rate * expiry)
    with np.errstate(divide="ignore", invalid="ignore"):
        d1 = (np.log(spot / strike) + (rate + 0.5 * volatility**2) * expiry) / vol
        d2 = d1 - vol
        cdf = lambda v: 0.5 * (1.0 + erf(v / np.sqrt(2.0)))
        price = spot * cdf(d1) - strike * discount * cdf(d2)
    return np.where(vol > 0, price, np.maximum(spot - strike * discount, 0.0))


def black_scholes_prices(cols, out_dtype, p=1, threads=1):
    """bench.py:119-126: price per segment, stored in the out dtype."""
    n = len(cols[0])
    segs = [block_segments(c, p) for c in cols]
    parts = _run([lambda k=k: black_scholes(*[s[k] for s in segs]).astype(out_dtype)
                  for k in range(len(segs[0])) if len(segs[0][k])], threads)
    return np.concatenate(parts) if parts else np.empty(0, dtype=out_dtype)


def cpu_threads() -> int:
    """The reference's default locale count: host cores capped at 16 (runtime.py:46-58)."""
    try:
        hw = len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        hw = os.cpu_count() or 1
    return max(1, min(hw, 16))

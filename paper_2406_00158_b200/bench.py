"""Benchmark kernels of the distributed-ranges paper on the device runtime.

Same kernels and harness as the reference's bench module
(/root/reference/pkg/src/segrange/bench.py): dot_product = zip|transform|reduce
(:87-90), stream_triad (:93-99), Black-Scholes (:102-126), BenchSpec / run_spec / CSV
(:50-80, 348-386); plus the other STREAM kernels (copy, scale, add) named by the north
star.  Each kernel here is the *same view pipeline* as the reference, lowered to one
fused sm_100a kernel per segment.  GEMM and sort are outside this runtime's scope.
"""

from __future__ import annotations

import math
import time
from dataclasses import dataclass, field

import numpy as np

from . import _lib, algorithms, expr, repro, views
from .algorithms import add
from .containers import DistributedVector
from .runtime import Runtime
from .views import get_zip_mode, set_zip_mode

BENCH_NAMES = ("dot", "reduce", "inclusive_scan", "black_scholes", "stream", "sort")
DEFAULT_SIZES = {name: 10**7 for name in BENCH_NAMES}
REL_TOL = 1e-12
STREAM_ALPHA = 3.0

# Strike below spot keeps prices O(10), so relative tolerances are meaningful (bench.py:39-47).
BS_RANGES = {
    "spot": (90.0, 110.0),
    "strike": (70.0, 90.0),
    "rate": (0.0, 0.05),
    "volatility": (0.1, 0.4),
    "expiry": (0.25, 2.0),
}


@dataclass(frozen=True)
class BenchSpec:
    name: str
    size: int
    locales: int
    reps: int = 3
    seed: int = 1
    check: bool = False
    mode: str = "relaxed"
    dtype: str = "float64"

    def __post_init__(self):
        if self.name not in BENCH_NAMES:
            raise ValueError(f"unknown bench {self.name!r}; one of {BENCH_NAMES}")
        if self.reps < 1:
            raise ValueError("reps must be at least 1")
        if self.size < 0:
            raise ValueError("size must be non-negative")


@dataclass
class BenchResult:
    spec: BenchSpec
    seconds: list = field(default_factory=list)
    checksum: str = ""
    verified: bool | None = None
    extra: dict = field(default_factory=dict)

    @property
    def median_seconds(self) -> float:
        s = sorted(self.seconds)
        return s[len(s) // 2] if s else float("nan")


# ----------------------------------------------------------------------------------------
# kernels (the same view pipelines as the reference)


def dot_product(x, y):
    """zip | transform(t[0]*t[1]) | reduce(add) — one fused kernel per segment."""
    z = views.transform(views.zip(x, y), lambda t: t[0] * t[1])
    return algorithms.reduce(z, 0.0, add)


def stream_triad(a, b, c, alpha=STREAM_ALPHA):
    """a[i] = b[i] + alpha * c[i]."""
    algorithms.for_each(views.zip(a, b, c), lambda t: (t[1] + alpha * t[2], None, None), vectorized=True)


def stream_copy(c, a):
    """c[i] = a[i]."""
    algorithms.copy(a, c)


def stream_scale(b, c, alpha=STREAM_ALPHA):
    """b[i] = alpha * c[i]."""
    algorithms.for_each(views.zip(b, c), lambda t: (alpha * t[1], None), vectorized=True)


def stream_add(c, a, b):
    """c[i] = a[i] + b[i]."""
    algorithms.for_each(views.zip(c, a, b), lambda t: (t[1] + t[2], None, None), vectorized=True)


def _bs_result_dtype(dts):
    return np.float32 if all(np.dtype(d) == np.float32 for d in dts) else np.float64


def _bs_host(spot, strike, rate, volatility, expiry):
    """black_scholes_call on plain scalars/arrays: evaluated by the device kernel."""
    from .runtime import torch

    args = [np.atleast_1d(np.asarray(a, dtype=np.float64)) for a in (spot, strike, rate, volatility, expiry)]
    shape = np.broadcast_shapes(*[a.shape for a in args])
    args = [np.ascontiguousarray(np.broadcast_to(a, shape)).ravel() for a in args]
    t = torch()
    if not t.cuda.is_available():
        raise RuntimeError("black_scholes_call needs a CUDA device (no CPU fallback)")
    dev = t.device("cuda", t.cuda.current_device())
    d_in = [t.from_numpy(a).to(dev) for a in args]
    d_out = t.empty(args[0].size, dtype=t.float64, device=dev)
    stream = t.cuda.current_stream(dev)
    _lib.call("drk_black_scholes", _lib.F64, d_out.data_ptr(), *[x.data_ptr() for x in d_in], args[0].size,
              dev.index, stream.cuda_stream)
    stream.synchronize()
    out = d_out.cpu().numpy().reshape(shape)
    return out if np.ndim(spot) else out.reshape(np.shape(spot) if np.ndim(spot) else ())


black_scholes_call = expr.DeviceFunction("black_scholes", 5, _bs_result_dtype, _bs_host)
black_scholes_call.__doc__ = """European call price C = S*Phi(d1) - K*exp(-rT)*Phi(d2); vol = sigma*sqrt(T) <= 0
gives the discounted intrinsic value (reference bench.py:106-116).  Priced in fp64 and rounded
once to the result dtype, like the reference prices fp32 columns in float64 (bench.py:109).
Inside a traced element function it becomes the fused drk_black_scholes kernel."""

black_scholes_call_fast = expr.DeviceFunction("black_scholes_fast", 5, _bs_result_dtype, _bs_host)
black_scholes_call_fast.__doc__ = """black_scholes_call with fp32 columns priced in fp32 (SFU
exp2/log2/rcp, one erfc fit for Phi: rel <= 1e-5 against the fp64 formula): the fast tier,
HBM-bound on B200 (drk_black_scholes_ex DRK_BS_FAST).  fp64 columns are priced in fp64."""

BS_PRECISIONS = ("reference", "fast")


def norm_cdf(x):
    from scipy.special import erf

    return 0.5 * (1.0 + erf(x / np.sqrt(2.0)))


def black_scholes_prices(out, spot, strike, rate, volatility, expiry, precision="reference"):
    """out[i] = call price of option i, element-wise over the zipped inputs (reference
    bench.py:119-126).  precision "reference" prices in fp64 like the reference; "fast"
    prices fp32 columns in fp32 (black_scholes_call_fast)."""
    if precision not in BS_PRECISIONS:
        raise ValueError(f"precision must be one of {BS_PRECISIONS}, got {precision!r}")
    if precision == "fast":
        fn = lambda t: (black_scholes_call_fast(t[1], t[2], t[3], t[4], t[5]), None, None, None, None, None)  # noqa: E731
    else:
        fn = lambda t: (black_scholes_call(t[1], t[2], t[3], t[4], t[5]), None, None, None, None, None)  # noqa: E731
    algorithms.for_each(views.zip(out, spot, strike, rate, volatility, expiry), fn, vectorized=True)


# ----------------------------------------------------------------------------------------
# sequential oracles for --check (plain loops on host copies; verification only)


def _oracle_dot(xs, ys) -> float:
    total = 0.0
    for a, b in zip(xs.tolist(), ys.tolist()):
        total += a * b
    return total


def _oracle_bs(S, K, r, v, T) -> float:
    vol = v * math.sqrt(T)
    disc = math.exp(-r * T)
    if vol <= 0.0:
        return max(S - K * disc, 0.0)
    d1 = (math.log(S / K) + (r + 0.5 * v * v) * T) / vol
    d2 = d1 - vol
    phi = lambda x: 0.5 * (1.0 + math.erf(x / math.sqrt(2.0)))
    return S * phi(d1) - K * disc * phi(d2)


def rel_close(actual, expected, tol) -> bool:
    return bool(np.isclose(np.asarray(actual), np.asarray(expected), rtol=tol, atol=0.0).all())


def _timed(reps, kernel, rt, reset=None):
    """Per rep: wall seconds from the call until every device stream has drained (the
    algorithms may return once their kernels are enqueued), and device seconds from CUDA
    events recorded on every device stream around the call (max over devices)."""
    from .runtime import torch

    t = torch()
    seconds, device_seconds, result = [], [], None
    states = rt.device_states
    for _ in range(reps):
        if reset is not None:
            reset()
            rt.synchronize()
        evs = []
        for st in states:
            e0, e1 = t.cuda.Event(enable_timing=True), t.cuda.Event(enable_timing=True)
            e0.record(st.stream)
            evs.append((e0, e1, st))
        t0 = time.perf_counter()
        result = kernel()
        for e0, e1, st in evs:
            e1.record(st.stream)
        rt.synchronize()
        seconds.append(time.perf_counter() - t0)
        device_seconds.append(max(e0.elapsed_time(e1) for e0, e1, _ in evs) / 1e3)
    return seconds, device_seconds, result


def _gpu_extra(res, rt, device_seconds, bytes_per_elem):
    """GPU columns of the CSV: device time, algorithmic GB/s and elements/s, fraction of the
    aggregate HBM roofline of the GPUs the locales occupy."""
    res.extra["device_seconds"] = list(device_seconds)
    res.extra["bytes_per_element"] = bytes_per_elem
    res.extra["devices"] = len(rt.device_states)


def _dt(spec):
    return np.dtype(spec.dtype)


def _dt(spec):
    return np.dtype(spec.dtype)


def bench_dot(spec: BenchSpec, rt: Runtime) -> BenchResult:
    n, dt = spec.size, _dt(spec)
    xs = repro.unit_doubles(spec.seed, 0, n).astype(dt)
    ys = repro.unit_doubles(spec.seed, n, n).astype(dt)
    x = DistributedVector.from_numpy(rt, xs)
    y = DistributedVector.from_numpy(rt, ys)
    seconds, dsec, value = _timed(spec.reps, lambda: dot_product(x, y), rt)
    res = BenchResult(spec, seconds, repro.checksum(np.float64(value)))
    _gpu_extra(res, rt, dsec, 2 * dt.itemsize)
    if spec.check:
        tol = REL_TOL if dt == np.float64 else 1e-5
        res.verified = rel_close(value, _oracle_dot(xs, ys), tol) if n else value == 0.0
    return res


def bench_reduce(spec: BenchSpec, rt: Runtime) -> BenchResult:
    n = spec.size
    v = DistributedVector(rt, n, dtype=np.int64)
    if n:
        algorithms.copy(views.iota(n), v)
    seconds, dsec, value = _timed(spec.reps, lambda: algorithms.reduce(v, 0, add), rt)
    res = BenchResult(spec, seconds, repro.checksum(np.int64(value)))
    _gpu_extra(res, rt, dsec, 8)
    if spec.check:
        res.verified = value == n * (n - 1) // 2
    return res


def bench_inclusive_scan(spec: BenchSpec, rt: Runtime) -> BenchResult:
    n = spec.size
    v = DistributedVector(rt, n, dtype=np.int64)
    if n:
        algorithms.copy(views.iota(n), v)
    out = DistributedVector(rt, n, init=0, dtype=np.int64)
    seconds, dsec, _ = _timed(spec.reps, lambda: algorithms.inclusive_scan(v, out, add), rt)
    data = out.to_numpy()
    res = BenchResult(spec, seconds, repro.checksum(data))
    _gpu_extra(res, rt, dsec, 16)
    if spec.check:
        i = np.arange(n, dtype=np.int64)
        res.verified = bool(np.array_equal(data, i * (i + 1) // 2))
    return res


def bench_black_scholes(spec: BenchSpec, rt: Runtime) -> BenchResult:
    n, dt = spec.size, _dt(spec)
    cols = {name: repro.uniform_doubles(spec.seed, k * n, n, lo, hi).astype(dt)
            for k, (name, (lo, hi)) in enumerate(BS_RANGES.items())}
    vecs = {k: DistributedVector.from_numpy(rt, v) for k, v in cols.items()}
    out = DistributedVector(rt, n, dtype=dt)
    seconds, dsec, _ = _timed(spec.reps, lambda: black_scholes_prices(
        out, vecs["spot"], vecs["strike"], vecs["rate"], vecs["volatility"], vecs["expiry"]), rt)
    data = out.to_numpy()
    res = BenchResult(spec, seconds, repro.checksum(data))
    _gpu_extra(res, rt, dsec, 6 * dt.itemsize)
    if spec.check:
        exp = np.array([_oracle_bs(*(float(cols[k][i]) for k in BS_RANGES)) for i in range(n)])
        res.verified = rel_close(data, exp, REL_TOL if dt == np.float64 else 1e-5)
    return res


def bench_stream(spec: BenchSpec, rt: Runtime) -> BenchResult:
    n, dt = spec.size, _dt(spec)
    bs = repro.unit_doubles(spec.seed, 0, n).astype(dt)
    cs = repro.unit_doubles(spec.seed, n, n).astype(dt)
    a = DistributedVector(rt, n, dtype=dt)
    b = DistributedVector.from_numpy(rt, bs)
    c = DistributedVector.from_numpy(rt, cs)
    seconds, dsec, _ = _timed(spec.reps, lambda: stream_triad(a, b, c), rt)
    data = a.to_numpy()
    res = BenchResult(spec, seconds, repro.checksum(data))
    _gpu_extra(res, rt, dsec, 3 * dt.itemsize)
    med = sorted(seconds)[len(seconds) // 2]
    res.extra["bytes_per_second"] = 3.0 * dt.itemsize * n / med if med > 0 else float("inf")
    if spec.check:
        alpha = dt.type(STREAM_ALPHA)
        res.verified = bool(np.array_equal(data, bs + alpha * cs))
    return res


def bench_sort(spec: BenchSpec, rt: Runtime) -> BenchResult:
    """Reference bench.py:332-345: sort splitmix64 uint64 keys, reset before every rep."""
    n = spec.size
    keys = repro.splitmix64(spec.seed, 0, n)
    v = DistributedVector(rt, n, dtype=np.uint64)

    def reset():
        algorithms.copy(keys, v)

    seconds, dsec, _ = _timed(spec.reps, lambda: algorithms.sort(v), rt, reset=reset)
    data = v.to_numpy()
    res = BenchResult(spec, seconds, repro.checksum(data))
    _gpu_extra(res, rt, dsec, None)  # a sort has no single algorithmic byte count
    if spec.check:
        res.verified = bool(np.array_equal(data, np.sort(keys)))
    return res


BENCHES = {
    "sort": bench_sort,
    "dot": bench_dot,
    "reduce": bench_reduce,
    "inclusive_scan": bench_inclusive_scan,
    "black_scholes": bench_black_scholes,
    "stream": bench_stream,
}


def run_spec(spec: BenchSpec) -> BenchResult:
    previous = get_zip_mode()
    set_zip_mode(spec.mode)
    try:
        with Runtime(spec.locales) as rt:
            return BENCHES[spec.name](spec, rt)
    finally:
        set_zip_mode(previous)


CSV_HEADER = "bench,size,locales,rep,seconds,checksum,verified"
# appended after the reference's columns (drbench --gpu-columns), so the first seven fields
# keep the reference schema (bench.py:369-386)
GPU_COLUMNS = "device_seconds,gbps,elements_per_second,roofline_frac,devices"


def hbm_peak_gbs() -> float:
    """Per-GPU HBM roofline: MEASURED_PEAKS.json hbm_gbs (driver-written), else the
    B200_PROFILING.md fallback."""
    import json
    import os

    path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")
    try:
        with open(path) as fh:
            return float(json.load(fh)["hbm_gbs"])
    except Exception:
        return 6650.0


def csv_rows(results, gpu_columns: bool = False) -> list:
    rows = [CSV_HEADER + ("," + GPU_COLUMNS if gpu_columns else "")]
    peak = hbm_peak_gbs() if gpu_columns else None
    for r in results:
        dsec = r.extra.get("device_seconds", [])
        bpe = r.extra.get("bytes_per_element")
        ndev = r.extra.get("devices", 1)
        for i, sec in enumerate(r.seconds):
            verified = "" if r.verified is None else ("true" if r.verified else "false")
            row = f"{r.spec.name},{r.spec.size},{r.spec.locales},{i},{sec:.9f},{r.checksum},{verified}"
            if gpu_columns:
                d = dsec[i] if i < len(dsec) else float("nan")
                if bpe is not None and d > 0:
                    gbps = bpe * r.spec.size / d / 1e9
                    row += f",{d:.9f},{gbps:.3f},{r.spec.size / d:.6e},{gbps / (peak * ndev):.4f},{ndev}"
                else:
                    eps = r.spec.size / d if d > 0 else float("nan")
                    row += f",{d:.9f},,{eps:.6e},,{ndev}"
            rows.append(row)
    return rows


def emit_csv(results, path, gpu_columns: bool = False) -> None:
    with open(path, "w", encoding="ascii") as fh:
        fh.write("\n".join(csv_rows(results, gpu_columns)) + "\n")

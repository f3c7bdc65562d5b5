"""Generate golden vectors by running the REAL reference (segrange) in this container.

    python tests/golden/make_golden.py            # needs /root/reference (read-only source)

The reference is pure Python; it is imported from a temporary copy of
/root/reference/pkg/src (nothing is copied into this repository).  Inputs are described
by splitmix64 generator records (reference repro.py:21-40) so they can be regenerated
anywhere; outputs are stored as exact scalars (float.hex / int), CRC-32 checksums of the
output bytes (reference repro.py:43-53), and, for small n, the full output arrays
(golden.npz).  The GPU box never reads /root/reference: tests use these fixtures.
"""

from __future__ import annotations

import json
import os
import shutil
import sys
import tempfile

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REF = "/root/reference/pkg/src"
ARRAY_MAX = 4099


def import_reference():
    tmp = tempfile.mkdtemp(prefix="segref_")
    shutil.copytree(REF, os.path.join(tmp, "src"))
    sys.path.insert(0, os.path.join(tmp, "src"))
    import segrange  # noqa: F401

    return segrange


def enc(v):
    if isinstance(v, np.generic):
        v = v.item()
    if isinstance(v, float):
        return {"f": v.hex()}
    if isinstance(v, bool):
        return {"b": v}
    if isinstance(v, int):
        return {"i": str(v)}
    if v is None:
        return None
    raise TypeError(type(v))


def main():
    sr = import_reference()
    from segrange import algorithms as A
    from segrange import bench as B
    from segrange import repro as R
    from segrange import DistributedVector, Runtime, views

    rts = {p: Runtime(p) for p in (1, 2, 3, 4, 7)}
    cases, arrays = [], {}

    def gen(desc, dtype):
        k = desc["kind"]
        if k == "unit":
            x = R.unit_doubles(desc["seed"], desc["start"], desc["n"])
        elif k == "uniform":
            x = R.uniform_doubles(desc["seed"], desc["start"], desc["n"], desc["lo"], desc["hi"])
        elif k == "mod":
            x = (R.splitmix64(desc["seed"], desc["start"], desc["n"]) % np.uint64(desc["modulus"])).astype(
                np.int64) + desc["offset"]
        elif k == "arange":
            x = np.arange(desc["start"], desc["start"] + desc["n"])
        return x.astype(dtype)

    def add_case(case, out_array=None):
        case["id"] = f"{case['op']}-{case['dtype']}-n{case['n']}-p{case['p']}-{len(cases)}"
        if out_array is not None:
            case["checksum"] = R.checksum(out_array)
            if case["n"] <= ARRAY_MAX:
                arrays[case["id"]] = out_array
                case["array"] = True
        cases.append(case)

    small = (0, 1, 2, 3, 5, 8, 17, 1000, 4099)
    P = (1, 2, 3, 4, 7)

    # dot_product (bench.py:87-90)
    for dt in ("float32", "float64"):
        for n in small + (65536,):
            for p in P:
                dx = {"kind": "unit", "seed": 1, "start": 0, "n": n}
                dy = {"kind": "unit", "seed": 1, "start": n, "n": n}
                x, y = gen(dx, dt), gen(dy, dt)
                rt = rts[p]
                v = B.dot_product(DistributedVector.from_numpy(rt, x), DistributedVector.from_numpy(rt, y))
                add_case({"op": "dot", "dtype": dt, "n": n, "p": p, "inputs": [dx, dy], "result": enc(v),
                          "input_checksums": [R.checksum(x), R.checksum(y)]})

    # reduce (algorithms.py:135-162)
    for dt, kind in (("int32", "mod"), ("int64", "mod"), ("float32", "unit"), ("float64", "unit")):
        for opname, init in (("add", 0), ("minimum", 10**9), ("maximum", -(10**9)), ("multiply", 1)):
            for n in small + (65536,):
                for p in (1, 3, 7):
                    if opname == "multiply" and n > 17:
                        continue
                    d = ({"kind": "mod", "seed": 1, "start": 0, "n": n, "modulus": 2001, "offset": -1000}
                         if kind == "mod" else {"kind": "unit", "seed": 1, "start": 0, "n": n})
                    if opname == "multiply":
                        d = {"kind": "mod", "seed": 2, "start": 0, "n": n, "modulus": 5, "offset": -2}
                    x = gen(d, dt)
                    init_v = init if dt.startswith("int") else float(init)
                    v = A.reduce(DistributedVector.from_numpy(rts[p], x), init_v, getattr(A, opname))
                    add_case({"op": "reduce", "ufunc": opname, "init": enc(init_v), "dtype": dt, "n": n, "p": p,
                              "inputs": [d], "result": enc(v)})

    # stream triad (bench.py:93-99)
    for dt in ("float32", "float64"):
        for n in small + (65536,):
            for p in (1, 4, 7):
                db = {"kind": "unit", "seed": 1, "start": 0, "n": n}
                dc = {"kind": "unit", "seed": 1, "start": n, "n": n}
                b, c = gen(db, dt), gen(dc, dt)
                rt = rts[p]
                a = DistributedVector(rt, n, dtype=np.dtype(dt))
                B.stream_triad(a, DistributedVector.from_numpy(rt, b), DistributedVector.from_numpy(rt, c))
                add_case({"op": "triad", "dtype": dt, "n": n, "p": p, "alpha": 3.0, "inputs": [db, dc]},
                         a.to_numpy())

    # scans (algorithms.py:169-308) incl. the white-box partials of _scan_aligned
    scan_inputs = {
        "int32": {"kind": "mod", "seed": 1, "start": 0, "modulus": 2001, "offset": -1000},
        "int64": {"kind": "mod", "seed": 1, "start": 0, "modulus": 2001, "offset": -1000},
        "float32": {"kind": "mod", "seed": 1, "start": 0, "modulus": 3, "offset": -1},   # exact tier
        "float64": {"kind": "unit", "seed": 1, "start": 0},
    }
    for dt, base in scan_inputs.items():
        for exclusive in (False, True):
            for n in small + (65536,):
                for p in P:
                    d = dict(base, n=n)
                    x = gen(d, dt)
                    rt = rts[p]
                    v = DistributedVector.from_numpy(rt, x)
                    out = DistributedVector(rt, n, init=0, dtype=np.dtype(dt))
                    init = (5 if dt.startswith("int") else 0.5) if exclusive else None
                    parts = A._scan_aligned(v, out, A.add, exclusive=exclusive, init=init)
                    add_case({"op": "exclusive_scan" if exclusive else "inclusive_scan", "dtype": dt, "n": n,
                              "p": p, "init": enc(init), "inputs": [d], "partials": [enc(q) for q in parts]},
                             out.to_numpy())
    # fp32 accuracy tier at moderate n (reference still accurate)
    for n in (1000, 65536):
        for p in (1, 4):
            d = {"kind": "unit", "seed": 3, "start": 0, "n": n}
            x = gen(d, "float32")
            v = DistributedVector.from_numpy(rts[p], x)
            out = DistributedVector(rts[p], n, init=0, dtype=np.float32)
            parts = A._scan_aligned(v, out, A.add, exclusive=False, init=None)
            add_case({"op": "inclusive_scan", "dtype": "float32", "tier": "accuracy", "n": n, "p": p, "init": None,
                      "inputs": [d], "partials": [enc(q) for q in parts]}, out.to_numpy())
    # scan min/max (ops without identity)
    for opname in ("minimum", "maximum"):
        for dt in ("int32", "float64"):
            for n in (17, 1000):
                for p in (1, 3):
                    d = ({"kind": "mod", "seed": 4, "start": 0, "n": n, "modulus": 2001, "offset": -1000}
                         if dt == "int32" else {"kind": "unit", "seed": 4, "start": 0, "n": n})
                    x = gen(d, dt)
                    v = DistributedVector.from_numpy(rts[p], x)
                    out = DistributedVector(rts[p], n, init=0, dtype=np.dtype(dt))
                    parts = A._scan_aligned(v, out, getattr(A, opname), exclusive=False, init=None)
                    add_case({"op": "inclusive_scan", "ufunc": opname, "dtype": dt, "n": n, "p": p, "init": None,
                              "inputs": [d], "partials": [enc(q) for q in parts]}, out.to_numpy())
    # exclusive scans with minimum / maximum (init takes part in every prefix)
    for opname, dt, init in (("minimum", "int32", 0), ("maximum", "float64", 0.25), ("minimum", "float32", 0.5)):
        for n in (17, 1000, 4099):
            for p in (1, 3, 7):
                d = ({"kind": "mod", "seed": 10, "start": 0, "n": n, "modulus": 2001, "offset": -1000}
                     if dt == "int32" else {"kind": "unit", "seed": 10, "start": 0, "n": n})
                x = gen(d, dt)
                v = DistributedVector.from_numpy(rts[p], x)
                out = DistributedVector(rts[p], n, init=0, dtype=np.dtype(dt))
                parts = A._scan_aligned(v, out, getattr(A, opname), exclusive=True, init=init)
                add_case({"op": "exclusive_scan", "ufunc": opname, "dtype": dt, "n": n, "p": p, "init": enc(init),
                          "inputs": [d], "partials": [enc(q) for q in parts]}, out.to_numpy())

    # int32 carry overflow raises (algorithms.py:292-296 -> np.add(off, int32) OverflowError)
    n = 4096
    d = {"kind": "mod", "seed": 1, "start": 0, "n": n, "modulus": 1, "offset": 1_000_000}
    x = gen(d, "int32")
    try:
        v = DistributedVector.from_numpy(rts[4], x)
        A.inclusive_scan(v, DistributedVector(rts[4], n, init=0, dtype=np.int32))
        raised = None
    except Exception as exc:  # AggregateTaskError wrapping OverflowError
        raised = type(exc).__name__ + ":" + ",".join(type(e).__name__ for _, e in getattr(exc, "failures", []))
    add_case({"op": "inclusive_scan", "dtype": "int32", "n": n, "p": 4, "init": None, "inputs": [d],
              "raises": raised})

    # Black-Scholes (bench.py:102-126)
    for dt in ("float32", "float64"):
        for n in (1, 5, 257, 4099):
            for p in (1, 3):
                descs = [{"kind": "uniform", "seed": 1, "start": k * n, "n": n, "lo": lo, "hi": hi}
                         for k, (lo, hi) in enumerate(B.BS_RANGES.values())]
                cols = [gen(dd, dt) for dd in descs]
                rt = rts[p]
                vecs = [DistributedVector.from_numpy(rt, c) for c in cols]
                out = DistributedVector(rt, n, dtype=np.dtype(dt))
                B.black_scholes_prices(out, *vecs)
                add_case({"op": "black_scholes", "dtype": dt, "n": n, "p": p, "inputs": descs}, out.to_numpy())

    # copy between different partitions (algorithms.py:468-503)
    for dt in ("float32", "int64"):
        n = 23
        d = {"kind": "arange", "start": 0, "n": n}
        x = gen(d, dt)
        v3 = DistributedVector.from_numpy(rts[3], x)
        v4 = DistributedVector(rts[4], n, dtype=np.dtype(dt))
        A.copy(v3, v4)
        add_case({"op": "copy", "dtype": dt, "n": n, "p": 4, "inputs": [d]}, v4.to_numpy())

    # sort (algorithms.py:315-432): sample sort, optionally by a key function (stable)
    sort_keys = {"none": None, "abs": np.abs, "neg": np.negative}
    for dt in ("int32", "int64", "float32", "float64"):
        for n in (0, 1, 2, 3, 5, 17, 1000, 4099):
            for p in P:
                for kname in ("none", "abs", "neg"):
                    if kname != "none" and n not in (17, 4099):
                        continue
                    # ties on purpose (mod 41 around zero) so a key sort's stability shows
                    d = ({"kind": "mod", "seed": 5, "start": 0, "n": n, "modulus": 41, "offset": -20}
                         if kname != "none" or dt.startswith("int") else {"kind": "unit", "seed": 5, "start": 0, "n": n})
                    x = gen(d, dt)
                    v = DistributedVector.from_numpy(rts[p], x)
                    A.sort(v, key=sort_keys[kname])
                    add_case({"op": "sort", "dtype": dt, "n": n, "p": p, "key": kname, "inputs": [d]}, v.to_numpy())

    # view pipelines (views.py:271-556): reduce over drop|take, dot over a non-aligned zip,
    # scan of a transform view, copy of a transform view
    for dt, kind in (("int32", "mod"), ("float32", "unit"), ("float64", "unit")):
        for n in (17, 1000, 4099):
            for p in (1, 3, 4, 7):
                for dr, tk in ((0, n), (3, n - 5), (n // 3, n // 2), (n - 1, 1)):
                    d = ({"kind": "mod", "seed": 6, "start": 0, "n": n, "modulus": 2001, "offset": -1000}
                         if kind == "mod" else {"kind": "unit", "seed": 6, "start": 0, "n": n})
                    x = gen(d, dt)
                    v = DistributedVector.from_numpy(rts[p], x)
                    r = A.reduce(views.take(views.drop(v, dr), tk), 0, A.add)
                    add_case({"op": "reduce_view", "dtype": dt, "n": n, "p": p, "drop": dr, "take": tk,
                              "inputs": [d], "result": enc(r)})
    for dt in ("float32", "float64"):
        n = 1000
        for pa, pb in (([500, 500], [300, 300, 400]), ([0, 1000], [999, 1]), ([250, 250, 250, 250], [1000])):
            dx = {"kind": "unit", "seed": 7, "start": 0, "n": n}
            dy = {"kind": "unit", "seed": 7, "start": n, "n": n}
            x, y = gen(dx, dt), gen(dy, dt)
            rt = rts[max(len(pa), len(pb))]
            vx = DistributedVector.from_numpy(rt, x, partition=pa)
            vy = DistributedVector.from_numpy(rt, y, partition=pb)
            r = A.reduce(views.transform(views.zip(vx, vy), lambda t: t[0] * t[1]), 0.0, A.add)
            add_case({"op": "dot_nonaligned", "dtype": dt, "n": n, "p": len(pa), "parts": [pa, pb],
                      "inputs": [dx, dy], "result": enc(r)})
    for n in (17, 1000, 4099):
        for p in (1, 3, 7):
            d = {"kind": "mod", "seed": 8, "start": 0, "n": n, "modulus": 2001, "offset": -1000}
            x = gen(d, "int32")
            v = DistributedVector.from_numpy(rts[p], x)
            out = DistributedVector(rts[p], n, init=0, dtype=np.int32)
            A.inclusive_scan(views.transform(v, lambda e: e * 3 - 1), out)
            add_case({"op": "scan_view", "dtype": "int32", "n": n, "p": p, "inputs": [d]}, out.to_numpy())
    for dt in ("float32", "float64", "int64"):
        for n in (17, 4099):
            for p in (1, 4):
                d = ({"kind": "mod", "seed": 9, "start": 0, "n": n, "modulus": 2001, "offset": -1000}
                     if dt == "int64" else {"kind": "unit", "seed": 9, "start": 0, "n": n})
                x = gen(d, dt)
                v = DistributedVector.from_numpy(rts[p], x)
                out = DistributedVector(rts[p], n, init=0, dtype=np.dtype(dt))
                A.copy(views.transform(v, lambda e: e * 2.5 + 1), out) if dt != "int64" else \
                    A.copy(views.transform(v, lambda e: e * 7 - 3), out)
                add_case({"op": "copy_transform", "dtype": dt, "n": n, "p": p, "inputs": [d]}, out.to_numpy())

    # reference known-answer tests (tests/test_bench.py, tests/test_algorithms.py)
    kat = {
        "dot_123_456": B.dot_product(DistributedVector.from_numpy(rts[3], np.array([1.0, 2.0, 3.0])),
                                     DistributedVector.from_numpy(rts[3], np.array([4.0, 5.0, 6.0]))),
        "bs_atm": float(B.black_scholes_call(100.0, 100.0, 0.0, 0.2, 1.0)),
        "bs_sigma0_itm": float(B.black_scholes_call(110.0, 100.0, 0.0, 0.0, 1.0)),
        "bs_sigma0_otm": float(B.black_scholes_call(90.0, 100.0, 0.0, 0.0, 1.0)),
        "splitmix_seed42_first5": [str(int(v)) for v in R.splitmix64(42, 0, 5)],
        "checksum_15_m225": R.checksum(np.array([1.5, -2.25])),
    }
    for rt in rts.values():
        rt.close()

    meta = {"numpy": np.__version__, "generator": "tests/golden/make_golden.py",
            "reference": "/root/reference/pkg/src/segrange (segrange 0.1.0)", "cases": cases,
            "kat": {k: (enc(v) if not isinstance(v, (list, str)) else v) for k, v in kat.items()}}
    import scipy

    meta["scipy"] = scipy.__version__
    with open(os.path.join(HERE, "golden.json"), "w") as fh:
        json.dump(meta, fh, indent=0, sort_keys=True)
    np.savez_compressed(os.path.join(HERE, "golden.npz"), **arrays)
    print(f"{len(cases)} cases, {len(arrays)} arrays")


if __name__ == "__main__":
    main()

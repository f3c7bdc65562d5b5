"""Kernel micro-benchmark: time libdrk entry points directly (CUDA events, L2-cold
inputs of 2^log2n elements) and check them.  Used to tune kernels; bench.py is the
end-to-end number.

    python tools/kbench.py [--log2n 30] [--reps 20] [--only scan,triad,...]
"""
import argparse
import ctypes
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
from paper_2406_00158_b200 import _lib  # noqa: E402


def timeit(fn, reps):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    fn()
    torch.cuda.synchronize()
    times = []
    for _ in range(reps):
        s.record()
        fn()
        e.record()
        e.synchronize()
        times.append(s.elapsed_time(e))
    return float(np.median(times)), float(np.min(times))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--log2n", type=int, default=30)
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--tune", default="", help="name=value,... passed to drk_tune")
    ap.add_argument("--only", default="copy,triad,dot,reduce,scan_f32,scan_i32,scan_f64,scan_excl_i32,bs")
    args = ap.parse_args()
    n = 1 << args.log2n
    dev = torch.device("cuda", 0)
    stream = torch.cuda.current_stream().cuda_stream
    peak = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists(
        os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
    lib = _lib.load()
    for kv in filter(None, args.tune.split(",")):
        k, v = kv.split("=")
        lib.drk_tune(k.encode(), int(v))
    a = torch.empty(n, dtype=torch.float32, device=dev)
    b = torch.rand(n, dtype=torch.float32, device=dev)
    c = torch.rand(n, dtype=torch.float32, device=dev)
    red_scratch = torch.zeros(lib.drk_reduce_scratch_bytes(), dtype=torch.uint8, device=dev)
    res = torch.zeros(4, dtype=torch.float64, device=dev)
    alpha = _lib.scalar_buffer(3.0, np.float32)
    out = {}

    def report(name, nbytes, t, extra=None):
        med, best = t
        gbs = nbytes / (med / 1e3) / 1e9
        out[name] = {"ms": round(med, 4), "best_ms": round(best, 4), "GB/s": round(gbs, 1), "frac": round(gbs / peak, 4)}
        if extra:
            out[name].update(extra)
        print(name, out[name], flush=True)

    only = args.only.split(",")
    if "copy" in only:
        report("copy", 8 * n, timeit(lambda: _lib.call("drk_copy", _lib.F32, a.data_ptr(), b.data_ptr(), n, 0, stream), args.reps))
    if "triad" in only:
        report("triad", 12 * n, timeit(lambda: _lib.call("drk_triad", _lib.F32, a.data_ptr(), b.data_ptr(), c.data_ptr(), n, alpha, 0, stream), args.reps))
        ok = torch.equal(a[:1 << 20], b[:1 << 20] + 3.0 * c[:1 << 20])
        out["triad"]["exact_sample"] = bool(ok)
    if "dot" in only:
        report("dot", 8 * n, timeit(lambda: _lib.call("drk_dot", _lib.F32, b.data_ptr(), c.data_ptr(), n, res.data_ptr(), red_scratch.data_ptr(), 0, stream), args.reps))
        ref = torch.dot(b.double(), c.double()).item()
        out["dot"]["rel_err"] = abs(res[0].item() - ref) / ref
    if "reduce" in only:
        report("reduce", 4 * n, timeit(lambda: _lib.call("drk_reduce", _lib.F32, _lib.ADD, b.data_ptr(), n, res.data_ptr(), red_scratch.data_ptr(), 0, stream), args.reps))
    for name, dt, code in (("scan_f32", torch.float32, _lib.F32), ("scan_i32", torch.int32, _lib.I32),
                           ("scan_f64", torch.float64, _lib.F64), ("scan_excl_i32", torch.int32, _lib.I32)):
        if name not in only:
            continue
        excl = name.startswith("scan_excl")
        m = n if dt != torch.float64 else n // 2
        if dt == torch.int32:
            x = torch.randint(-1000, 1001, (m,), dtype=torch.int32, device=dev)
        else:
            x = torch.rand(m, dtype=dt, device=dev)
        y = torch.empty_like(x)
        sb = lib.drk_scan_scratch_bytes(code, _lib.ADD, m)
        scratch = torch.zeros(sb + 4096, dtype=torch.uint8, device=dev)
        acc = _lib.acc_dtype(np.dtype(str(x.dtype).replace("torch.", "")), _lib.ADD)
        init = _lib.scalar_buffer(0, acc)
        tot = torch.zeros(2, dtype=torch.float64, device=dev)
        f = lambda: _lib.call("drk_scan", code, _lib.ADD, 1 if excl else 0, x.data_ptr(), y.data_ptr(), m,
                              ctypes.addressof(init) if excl else None, None, None, tot.data_ptr(), None,
                              scratch.data_ptr(), scratch.numel(), 0, stream)
        report(name, 2 * x.element_size() * m, timeit(f, args.reps))
        if dt == torch.int32:
            ref = torch.cumsum(x.long(), 0).int()
            if excl:
                ref = torch.cat([torch.zeros(1, dtype=torch.int32, device=dev), ref[:-1]])
            out[name]["exact"] = bool(torch.equal(ref, y))
        else:
            ref = torch.cumsum(x.double(), 0)
            out[name]["max_rel_err"] = float(((y.double() - ref).abs() / ref.abs().clamp_min(1e-30)).max().item())
        del x, y, scratch
    if "bs" in only:
        m = n // 4
        cols = [torch.rand(m, dtype=torch.float32, device=dev) * (hi - lo) + lo for lo, hi in
                ((90, 110), (70, 90), (0, 0.05), (0.1, 0.4), (0.25, 2.0))]
        o = torch.empty(m, dtype=torch.float32, device=dev)
        report("black_scholes", 24 * m, timeit(lambda: _lib.call("drk_black_scholes", _lib.F32, o.data_ptr(), *[q.data_ptr() for q in cols], m, 0, stream), args.reps))
    print(json.dumps(out))


if __name__ == "__main__":
    main()

"""Scan kernel time by size (one GPU): plain inclusive scans (fp32 / int32 / fp64) and fused
view scans (affine, product) through the public API, kernel time from CUDA events on the
launch stream (kernels.profile), back-to-back reps (median).  GB/s on algorithmic bytes
(8 B/elem fp32 scan, 12 for the product view) and the fraction of MEASURED_PEAKS hbm_gbs.

    python tools/scan_sizes.py [--sizes 20,22,...] [--reps 20] [--tune name=value,...]
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_2406_00158_b200 as sr  # noqa: E402
from paper_2406_00158_b200 import _lib, algorithms as A, kernels, repro, views  # noqa: E402


def peak():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"])
    except Exception:
        return 6650.0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="20,22,23,24,25,26,27,28,30")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--kinds", default="f32,i32,f64,affine_f32,product_f32",
                    help="f32, i32, f64, affine_f32, product_f32, copy_f32 (the copy kernel, for reference)")
    ap.add_argument("--tune", default="")
    ap.add_argument("--queue", type=float, default=0.0,
                    help="ms of GPU sleep enqueued before the reps (0: host-paced launches)")
    args = ap.parse_args()
    lib = _lib.load()
    for kv in filter(None, args.tune.split(",")):
        k, v = kv.split("=")
        lib.drk_tune(k.encode(), int(v))
    pk = peak()
    rt = sr.Runtime(1)
    rows = []
    for lg in [int(x) for x in args.sizes.split(",")]:
        n = 1 << lg
        for kind in args.kinds.split(","):
            dt = {"f32": np.float32, "i32": np.int32, "f64": np.float64}[kind.split("_")[-1]]
            x = sr.DistributedVector(rt, n, dtype=dt)
            repro.fill_mod(x, 1, 0, 3, -1)
            y = sr.DistributedVector(rt, n, dtype=dt)
            out = sr.DistributedVector(rt, n, dtype=dt)
            repro.fill_mod(y, 2, 0, 3, -1)
            if kind.startswith("affine"):
                src, nbytes = views.transform(x, lambda v: 2.5 * v + 1.0), 2 * dt().itemsize
            elif kind.startswith("product"):
                src, nbytes = views.transform(views.zip(x, y), lambda t: t[0] * t[1]), 3 * dt().itemsize
            else:
                src, nbytes = x, 2 * dt().itemsize
            run = (lambda: A.copy(x, out)) if kind.startswith("copy") else (lambda: A.inclusive_scan(src, out))
            for _ in range(3):
                run()
            rt.synchronize()
            with kernels.profile() as prof:
                if args.queue:
                    # keep the GPU busy while the host enqueues the reps, so the events
                    # bracket kernel time only (no host launch gaps inside them)
                    with torch.cuda.stream(rt.device_states[0].stream):
                        torch.cuda._sleep(int(args.queue * 2e6))
                for _ in range(args.reps):
                    run()
                rt.synchronize()
            times = sorted(s.elapsed_time(e) for recs in prof.records.values() for s, e, _ in recs)
            ms = times[len(times) // 2]
            gbs = nbytes * n / (ms / 1e3) / 1e9
            rows.append({"log2n": lg, "kind": kind, "ms": round(ms, 4), "GB/s": round(gbs, 1),
                         "frac": round(gbs / pk, 3), "kernels": sorted(prof.records)})
            print(json.dumps(rows[-1]), flush=True)
            del x, y, out
    print(json.dumps({"peak": pk, "rows": len(rows)}))


if __name__ == "__main__":
    main()

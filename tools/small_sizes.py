"""Small / mid sizes on one GPU: device time per call of reduce, inclusive scan (fp32, int32)
and copy (the HBM ceiling at that size) measured as R back-to-back calls between ONE pair of
CUDA events, with the queue kept full by a GPU sleep enqueued first (so neither host launch
cost nor per-launch event records are inside the figure; inter-kernel gaps are).

    python tools/small_sizes.py [--sizes 20,21,...] [--reps 200] [--tune name=value,...]
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
from paper_2406_00158_b200 import _lib, algorithms as A, repro  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sizes", default="20,21,22,23,24,25,26")
    ap.add_argument("--reps", type=int, default=200)
    ap.add_argument("--kinds", default="copy_f32,reduce_f32,scan_f32,scan_i32")
    ap.add_argument("--tune", default="")
    args = ap.parse_args()
    lib = _lib.load()
    for kv in filter(None, args.tune.split(",")):
        k, v = kv.split("=")
        lib.drk_tune(k.encode(), int(v))
    pk = float(json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"])
    rt = sr.Runtime(1)
    st = rt.device_states[0]
    for lg in [int(s) for s in args.sizes.split(",")]:
        n = 1 << lg
        for kind in args.kinds.split(","):
            op, dts = kind.split("_")
            dt = {"f32": np.float32, "i32": np.int32}[dts]
            x = sr.DistributedVector(rt, n, dtype=dt)
            out = sr.DistributedVector(rt, n, dtype=dt)
            repro.fill_mod(x, 1, 0, 3, -1)
            if op in ("reduce", "reducedev"):
                plan = A._ReducePlan(rt, A._pieces(x), A.add)
                dres = torch.zeros(16, dtype=torch.float64, device=st.device)
                run = plan.batch.launch if op == "reduce" else (lambda: plan.batch.launch(result_ptr=dres.data_ptr()))
                nbytes = n * x.dtype.itemsize
            elif op == "scan":
                run, nbytes = (lambda: A.inclusive_scan(x, out)), 2 * n * x.dtype.itemsize
            else:
                run, nbytes = (lambda: A.copy(x, out)), 2 * n * x.dtype.itemsize
            for _ in range(5):
                run()
            rt.synchronize()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            with torch.cuda.stream(st.stream):
                torch.cuda._sleep(int(20e6))
                s.record()
            for _ in range(args.reps):
                run()
            with torch.cuda.stream(st.stream):
                e.record()
            rt.synchronize()
            us = s.elapsed_time(e) * 1e3 / args.reps
            gbs = nbytes / (us * 1e-6) / 1e9
            print(json.dumps({"log2n": lg, "kind": kind, "us": round(us, 2), "GB/s": round(gbs, 1),
                              "frac": round(gbs / pk, 3)}), flush=True)
            del x, out


if __name__ == "__main__":
    main()

"""C5 at small n on one GPU: API time per call (back-to-back, the host path) against the
kernel's device time (CUDA events with the GPU queue kept full) for reduce, transform,
inclusive_scan and dot on fp32 vectors of 2^20 and 2^22 elements."""
import json, os, sys, time
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2406_00158_b200 as sr  # noqa: E402
from paper_2406_00158_b200 import algorithms as A, bench as B, kernels, repro  # noqa: E402


def api(f, reps=2000):
    for _ in range(50):
        f()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        f()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) / reps * 1e6


rt = sr.Runtime(1)
st = rt.device_states[0]
for lg in (20, 22):
    n = 1 << lg
    x = sr.DistributedVector(rt, n, dtype=np.float32)
    y = sr.DistributedVector(rt, n, dtype=np.float32)
    repro.fill_unit(x, 1, 0)
    ops = {"reduce": lambda: A.reduce(x, 0.0), "transform": lambda: A.transform(x, y, lambda v: v * 2.0 + 1.0),
           "scan": lambda: A.inclusive_scan(x, y), "dot": lambda: B.dot_product(x, y)}
    for name, f in ops.items():
        a = api(f)
        f()
        torch.cuda.synchronize()
        with kernels.profile() as prof:
            with torch.cuda.stream(st.stream):
                torch.cuda._sleep(int(2e6))
            for _ in range(50):
                f()
            rt.synchronize()
        ts = sorted(s.elapsed_time(e) for recs in prof.records.values() for s, e, _ in recs)
        k = ts[len(ts) // 2] * 1e3 if ts else float("nan")
        print(json.dumps({"log2n": lg, "op": name, "api_us": round(a, 1), "kernel_us": round(k, 1),
                          "ratio": round(a / k, 2), "kernels": sorted(prof.records)}), flush=True)
